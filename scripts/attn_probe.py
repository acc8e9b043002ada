"""Config-4 diagnostics: attention over 16 ragged per-stream token subsets
(heads 16, head dim 72, bf16) — flash-attention varlen (contiguous or
strided q/k/v), SDPA over a padded batch with a key-padding mask, SDPA per
stream.  Prints ms per call (CUDA events) and the max difference to the
per-stream reference."""
import sys

import torch
import torch.nn.functional as F

try:
    from flash_attn import flash_attn_varlen_func
except Exception:  # noqa: BLE001
    flash_attn_varlen_func = None

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


def ref():
    outs = []
    for i in range(B):
        s, e = int(off[i]), int(off[i + 1])
        o = F.scaled_dot_product_attention(*(t[s:e].transpose(0, 1)[None] for t in (q, k, v)))
        outs.append(o[0].transpose(0, 1))
    return torch.cat(outs)


R = ref()
res = {"per_stream_sdpa": timeit(ref)}
if flash_attn_varlen_func is not None:
    fa_c = lambda: flash_attn_varlen_func(q.contiguous(), k.contiguous(), v.contiguous(), off, off, 1024, 1024)
    fa_s = lambda: flash_attn_varlen_func(q, k, v, off, off, 1024, 1024)
    res["fa2_varlen_contig"] = timeit(fa_c)
    res["fa2_varlen_strided"] = timeit(fa_s)
    res["fa2_err"] = float((fa_s() - R).abs().max())
L = max(lens)
pad = torch.zeros(B, L, 3, H, HD, device=dev, dtype=torch.bfloat16)
mask = torch.zeros(B, 1, 1, L, dtype=torch.bool, device=dev)
for i in range(B):
    s, e = int(off[i]), int(off[i + 1])
    pad[i, : e - s] = qkv[s:e].view(e - s, 3, H, HD)
    mask[i, ..., : e - s] = True
qp, kp, vp = (pad[:, :, j].transpose(1, 2) for j in range(3))
dense_mask = lambda: F.scaled_dot_product_attention(qp, kp, vp, attn_mask=mask)
res["padded_mask_sdpa"] = timeit(dense_mask)
dense_nomask = lambda: F.scaled_dot_product_attention(qp, kp, vp)
res["padded_nomask_sdpa(wrong, speed only)"] = timeit(dense_nomask)
from torch.nn.attention import SDPBackend, sdpa_kernel
for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.EFFICIENT_ATTENTION, SDPBackend.FLASH_ATTENTION):
    try:
        with sdpa_kernel(be):
            res[f"padded_mask_{be.name}"] = timeit(dense_mask)
    except Exception as ex:  # noqa: BLE001
        res[f"padded_mask_{be.name}"] = str(ex)[:80]
flops = sum(4 * l * l * H * HD for l in lens)
res["tflops_at_per_stream"] = flops / res["per_stream_sdpa"] / 1e9
print(res)

# the padded layout of CachedEncoder's graphed subset path: [B L + 1, 3, H, hdp]
hdp = 80
padb = torch.zeros(B * L + 1, 3, H, hdp, device=dev, dtype=torch.bfloat16)
dense = padb[:-1].unflatten(0, (B, -1))
qq, kk, vv = (dense[:, :, j].transpose(1, 2) for j in range(3))
res2 = {}
res2["padded80_strided_default"] = timeit(lambda: F.scaled_dot_product_attention(qq, kk, vv, scale=HD ** -0.5))
for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.EFFICIENT_ATTENTION, SDPBackend.FLASH_ATTENTION):
    try:
        with sdpa_kernel(be):
            res2[f"padded80_strided_{be.name}"] = timeit(lambda: F.scaled_dot_product_attention(qq, kk, vv, scale=HD ** -0.5))
    except Exception as ex:  # noqa: BLE001
        res2[f"padded80_strided_{be.name}"] = str(ex)[:60]
qc, kc, vc = (t.contiguous() for t in (qq, kk, vv))
res2["padded80_contig_default"] = timeit(lambda: F.scaled_dot_product_attention(qc, kc, vc, scale=HD ** -0.5))
q72 = torch.randn(B, H, L, 72, device=dev, dtype=torch.bfloat16)
res2["dense72_contig_default"] = timeit(lambda: F.scaled_dot_product_attention(q72, q72, q72))
print(res2)

# jagged nested tensors through SDPA (which backend torch picks for them)
offs64 = off.to(torch.int64)
nj = lambda t: torch.nested.nested_tensor_from_jagged(t, offs64).transpose(1, 2)
res3 = {}
try:
    qn, kn, vn = nj(q), nj(k), nj(v)
    res3["njt_default"] = timeit(lambda: F.scaled_dot_product_attention(qn, kn, vn))
    for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.EFFICIENT_ATTENTION, SDPBackend.FLASH_ATTENTION):
        try:
            with sdpa_kernel(be):
                res3[f"njt_{be.name}"] = timeit(lambda: F.scaled_dot_product_attention(qn, kn, vn))
        except Exception as ex:  # noqa: BLE001
            res3[f"njt_{be.name}"] = str(ex)[:60]
except Exception as ex:  # noqa: BLE001
    res3["njt"] = str(ex)[:100]
try:
    import flashinfer
    res3["flashinfer"] = flashinfer.__version__
except Exception as ex:  # noqa: BLE001
    res3["flashinfer"] = str(ex)[:60]
print(res3)
