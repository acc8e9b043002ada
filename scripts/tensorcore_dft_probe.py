"""Data for DESIGN §2 "why CUDA cores": the row transform of the bench's 512
frames as a dense DFT on the tensor cores (cuBLAS GEMMs — library kernels,
measurement only), in one TF32 pass and in split-precision 3xTF32, against
this repo's K_A (which does the packed row FFT plus luma, block-DCT energies
and the T1 store in 0.30 ms).  Prints one JSON object: time per step and the
normwise error of the half spectrum against fp64.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

S, H, W = 512, 448, 448
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
x = torch.rand((S * H, W), generator=g, device=dev)             # gray rows in [0, 1]
k = torch.arange(W // 2 + 1, device=dev, dtype=torch.float64)
n = torch.arange(W, device=dev, dtype=torch.float64)
ang = 2 * torch.pi * torch.outer(n, k) / W
w64 = torch.cat([torch.cos(ang), -torch.sin(ang)], dim=1)       # [W, 2 * 225]: real | imag
w = w64.float()


def split(t):
    hi = (t.view(torch.int32) & ~0x1FFF).view(torch.float32)     # tf32-representable part
    return hi, t - hi


def run_1pass():
    return x @ w


xh, xl = split(x)
wh, wl = split(w)


def run_3pass():
    return xh @ wh + (xh @ wl + xl @ wh)


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


torch.backends.cuda.matmul.allow_tf32 = True
ref = (x[:4096].double() @ w64)
res = {"workload": f"row DFT of {S} frames {H}x{W} (M={S * H}, K={W}, N={2 * (W // 2 + 1)}), fp32 in/out",
       "flops_per_pass": 2 * S * H * W * 2 * (W // 2 + 1)}
for name, fn in (("tf32_1pass", run_1pass), ("tf32_3pass", run_3pass)):
    ms = timeit(fn)
    y = fn()[:4096].double()
    err = float((y - ref).abs().max() / ref.abs().max())
    res[name] = {"ms_per_step": ms, "normwise_err": err}
torch.backends.cuda.matmul.allow_tf32 = False
ms = timeit(run_1pass)
y = run_1pass()[:4096].double()
res["fp32_simt"] = {"ms_per_step": ms, "normwise_err": float((y - ref).abs().max() / ref.abs().max())}
res["this_repo_K_A_ms"] = 0.303
print(json.dumps(res))
