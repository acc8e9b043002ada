"""Probe: variable-length attention options on this GPU (timing only)."""
import torch, torch.nn.functional as F
dev = "cuda"
B, H, d = 16, 16, 72
torch.manual_seed(0)
lens = torch.randint(400, 1024, (B,))
T = int(lens.sum())
off = torch.zeros(B + 1, dtype=torch.int32)
off[1:] = torch.cumsum(lens, 0)
off = off.to(dev)
q = torch.randn(T, H, d, device=dev, dtype=torch.bfloat16)
k, v = torch.randn_like(q), torch.randn_like(q)


def bench(fn, n=20):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


qd = torch.randn(B, H, 1024, d, device=dev, dtype=torch.bfloat16)
print("dense 16x1024 sdpa ms", bench(lambda: F.scaled_dot_product_attention(qd, qd, qd)))
try:
    from flash_attn import flash_attn_varlen_func
    mx = int(lens.max())
    o = flash_attn_varlen_func(q, k, v, off, off, mx, mx)
    print("flash_attn varlen ok", o.shape, "ms", bench(lambda: flash_attn_varlen_func(q, k, v, off, off, mx, mx)))
except Exception as e:  # noqa: BLE001
    print("flash_attn varlen failed:", type(e).__name__, str(e)[:200])
try:
    from torch.nn.attention import sdpa_kernel, SDPBackend
    offl = off.long()
    def njt():
        qn = torch.nested.nested_tensor_from_jagged(q, offl).transpose(1, 2)
        return F.scaled_dot_product_attention(qn, qn, qn)
    with sdpa_kernel(SDPBackend.FLASH_ATTENTION):
        print("njt flash ms", bench(njt))
except Exception as e:  # noqa: BLE001
    print("njt flash failed:", type(e).__name__, str(e)[:200])
try:
    import flashinfer
    print("flashinfer", flashinfer.__version__)
except Exception as e:  # noqa: BLE001
    print("flashinfer import failed", e)
try:
    import torch.nn.attention as A
    print("flash impls", A.list_flash_attention_impls(), "current", A.current_flash_attention_impl())
except Exception as e:  # noqa: BLE001
    print("impl list failed", e)
try:
    from torch.nn.attention.varlen import varlen_attn
    mx = int(lens.max())
    print("torch varlen ms", bench(lambda: varlen_attn(q, k, v, off, off, mx, mx)))
except Exception as e:  # noqa: BLE001
    print("torch varlen failed:", type(e).__name__, str(e)[:300])
try:
    import torch.nn.attention as A
    A.activate_flash_attention_impl("FA4")
    print("FA4 active", A.current_flash_attention_impl())
    print("dense sdpa FA4 ms", bench(lambda: F.scaled_dot_product_attention(qd, qd, qd)))
    from torch.nn.attention.varlen import varlen_attn
    print("torch varlen FA4 ms", bench(lambda: varlen_attn(q, k, v, off, off, mx, mx)))
except Exception as e:  # noqa: BLE001
    print("FA4 failed:", type(e).__name__, str(e)[:300])
