"""Config-4 diagnostics, part 2: variable-length attention backends for the
16 ragged per-stream token subsets (heads 16, head dim 72, bf16):
flash-attention 2 varlen (flash_attn), torch varlen_attn (default and with
the FA4 implementation activated), flashinfer fmha_varlen and its cuDNN
batch prefill.  ms per call and max |diff| to flash-attention 2."""
import torch

from flash_attn import flash_attn_varlen_func

torch.manual_seed(0)
dev = "cuda"
H, HD, B = 16, 72, 16
lens = [1024, 543, 480, 600, 1024, 300, 512, 700, 450, 520, 610, 1024, 390, 560, 505, 640]
T = sum(lens)
off = torch.tensor([0] + list(torch.cumsum(torch.tensor(lens), 0)), dtype=torch.int32, device=dev)
qkv = torch.randn(T, 3 * H * HD, device=dev, dtype=torch.bfloat16)
q, k, v = (t.unflatten(-1, (H, HD)) for t in qkv.split(H * HD, dim=-1))


def timeit(fn, n=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


R = flash_attn_varlen_func(q, k, v, off, off, 1024, 1024)
res = {"fa2": timeit(lambda: flash_attn_varlen_func(q, k, v, off, off, 1024, 1024))}


def trial(name, fn):
    try:
        o = fn()
        if isinstance(o, tuple):
            o = o[0]
        res[name] = timeit(fn)
        res[name + "_err"] = float((o.reshape(R.shape).float() - R.float()).abs().max())
    except Exception as ex:  # noqa: BLE001
        res[name] = f"{type(ex).__name__}: {str(ex)[:120]}"


from torch.nn.attention.varlen import varlen_attn
qc, kc, vc = q.contiguous(), k.contiguous(), v.contiguous()
trial("torch_varlen_default", lambda: varlen_attn(qc, kc, vc, off, off, 1024, 1024))
import torch.nn.attention as A
for impl in ("FA4", "FA3"):
    try:
        A.activate_flash_attention_impl(impl)
        trial(f"torch_varlen_{impl}", lambda: varlen_attn(qc, kc, vc, off, off, 1024, 1024))
        A.restore_flash_attention_impl()
    except Exception as ex:  # noqa: BLE001
        res[f"torch_varlen_{impl}"] = f"{type(ex).__name__}: {str(ex)[:120]}"
try:
    import flashinfer.prefill as P
    trial("flashinfer_fmha_varlen", lambda: P.fmha_varlen(qc, kc, vc, off, off, max_qo_len=1024))
    ws = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    lq = (off[1:] - off[:-1]).to(torch.int32).view(-1, 1, 1, 1)
    bo = (off.to(torch.int64) * H * HD).to(torch.int32).view(-1, 1, 1, 1)   # B + 1 ragged offsets
    trial("flashinfer_cudnn", lambda: P.cudnn_batch_prefill_with_kv_cache(
        qc, kc, vc, HD ** -0.5, ws, max_token_per_sequence=1024, max_sequence_kv=1024,
        actual_seq_lens_q=lq, actual_seq_lens_kv=lq, causal=False, return_lse=False,
        batch_offsets_q=bo, batch_offsets_o=bo, batch_offsets_k=bo, batch_offsets_v=bo)[0])
except Exception as ex:  # noqa: BLE001
    res["flashinfer"] = f"{type(ex).__name__}: {str(ex)[:120]}"
print(res)

# strided q / k / v (views of the fused QKV rows) and CUDA-graph capture of
# the cuDNN ragged prefill
res2 = {}
try:
    import flashinfer.prefill as P
    ws = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    lq = (off[1:] - off[:-1]).to(torch.int32).view(-1, 1, 1, 1)
    bo3 = (off.to(torch.int64) * 3 * H * HD).to(torch.int32).view(-1, 1, 1, 1)
    bo1 = (off.to(torch.int64) * H * HD).to(torch.int32).view(-1, 1, 1, 1)

    def strided():
        return P.cudnn_batch_prefill_with_kv_cache(
            q, k, v, HD ** -0.5, ws, max_token_per_sequence=1024, max_sequence_kv=1024,
            actual_seq_lens_q=lq, actual_seq_lens_kv=lq, causal=False, return_lse=False,
            batch_offsets_q=bo3, batch_offsets_o=bo1, batch_offsets_k=bo3, batch_offsets_v=bo3,
            is_cuda_graph_compatible=True)[0]
    o = strided()
    res2["cudnn_strided"] = timeit(strided)
    res2["cudnn_strided_err"] = float((o.reshape(R.shape).float() - R.float()).abs().max())
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        strided()
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g):
        og = strided()
    g.replay()
    torch.cuda.synchronize()
    res2["cudnn_graph_err"] = float((og.reshape(R.shape).float() - R.float()).abs().max())
    res2["cudnn_graph_ms"] = timeit(g.replay)
except Exception as ex:  # noqa: BLE001
    import traceback
    res2["error"] = f"{type(ex).__name__}: {str(ex)[:300]}"
print(res2)
