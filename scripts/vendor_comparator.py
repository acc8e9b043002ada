"""Vendor comparator: the same per-step selection + splice composed
from library calls — cuFFT through torch.fft.rfft2 / irfft2, torch
elementwise, reductions, sort and gather — on the same config-5 workload as
bench.py (512 streams of 448x448x3 fp32, P = 14, N = 1024, 1024x1152 bf16
hidden states).  Time only: it approximates the paper's "cuFFT + SIMT"
implementation and is NOT the product (no tie rules, no failure semantics).

Prints one JSON object: ms per step of the torch composition and of this
repo's path (fc_select + in-place splice, serial launch order, the splice
copier at its standalone sizing, FC_SPLICE_BULK_CTAS=2), same inputs.
"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import math

import torch

os.environ.setdefault("FC_SPLICE_BULK_CTAS", "2")   # serial order: the splice runs alone
import paper_2604_24391_b200 as fc  # noqa: E402
from paper_2604_24391_b200.synth import torch_stream_frames  # noqa: E402

S, H, P, D, R = int(os.environ.get("S", 512)), 448, 14, 1152, 4
G = H // P
N = G * G


def dct_matrix(p, device):
    u = torch.arange(p, dtype=torch.float64, device=device)[:, None]
    x = torch.arange(p, dtype=torch.float64, device=device)[None, :]
    c = torch.cos(math.pi * u * (2 * x + 1) / (2 * p)) * math.sqrt(2.0 / p)
    c[0] *= math.sqrt(0.5)
    return c


class TorchSelect:
    """decide() for a batch, composed from torch / cuFFT calls."""

    def __init__(self, device):
        self.c = dct_matrix(P, device)
        self.prev = None
        w = torch.full((H // 2 + 1,), 2.0, device=device)
        w[0] = 1.0
        w[-1] = 1.0
        self.w = w  # Hermitian weights of the half spectrum

    def __call__(self, rgb, alpha_min=0.08, alpha_max=0.5, tau=0.12, lam=0.25):
        gray64 = (0.299 * rgb[..., 0].double() + 0.587 * rgb[..., 1].double()) + 0.114 * rgb[..., 2].double()
        spec = torch.fft.rfft2(gray64.float())                       # cuFFT, complex64 [B, H, H/2+1]
        # block-DCT high-pass energy per patch (fp64, as the reference)
        # Parseval form (as this repo's kernel): E = sum X^2 - sum_{u,v<3} Y[u][v]^2
        blocks = gray64.reshape(S, G, P, G, P).permute(0, 1, 3, 2, 4)  # [B, gi, gj, x, y]
        c3 = self.c[:3]
        y = torch.einsum("ux,bijxy,vy->bijuv", c3, blocks, c3)
        energy = ((blocks * blocks).sum((-2, -1)) - (y * y).sum((-2, -1))).clamp(min=0).reshape(S, N)
        mu = energy.mean(1, keepdim=True)
        sd = energy.std(1, unbiased=False, keepdim=True)
        fresh = energy > mu + lam * sd
        pc = spec.real ** 2 + spec.imag ** 2
        if self.prev is None:
            self.prev = spec
            return None
        pp = self.prev.real ** 2 + self.prev.imag ** 2
        # global amplitude cosine (Hermitian-weighted), entropy, budget
        sim = ((pp * pc).sqrt() * self.w).sum((1, 2)) / ((pp * self.w).sum((1, 2)).sqrt()
                                                         * (pc * self.w).sum((1, 2)).sqrt())
        tot = (pc * self.w).sum((1, 2))
        plogp = (torch.xlogy(pc, pc) * self.w).sum((1, 2))
        psi = (torch.log(tot) - plogp / tot) / math.log(H * H)
        alpha = alpha_min + (alpha_max - alpha_min) * torch.exp(-psi)
        k_reuse = torch.floor(alpha * N).long()
        # phase correlation
        cross = self.prev * spec.conj()
        cross = cross / (cross.abs() + 1e-12)
        r = torch.fft.irfft2(cross, s=(H, H))
        pos = r.reshape(S, -1).argmax(1)
        di = (-(pos // H)) % H
        dj = (-(pos % H)) % H
        di = torch.where(2 * di >= H, di - H, di)
        dj = torch.where(2 * dj >= H, dj - H, dj)
        dip = torch.sign(di) * ((2 * di.abs() + P - 1) // (2 * P))
        djp = torch.sign(dj) * ((2 * dj.abs() + P - 1) // (2 * P))
        ii = torch.arange(N, device=rgb.device) // G
        jj = torch.arange(N, device=rgb.device) % G
        si, sj = ii[None] - dip[:, None], jj[None] - djp[:, None]
        aligned = (si >= 0) & (si < G) & (sj >= 0) & (sj < G)
        flush = (sim < tau) | (torch.maximum(dip.abs(), djp.abs()) > 1)
        cand = aligned & ~fresh & ~flush[:, None]
        key = torch.where(cand, energy, torch.full_like(energy, float("inf")))
        order = torch.sort(key, dim=1, stable=True).indices            # ascending (E, index)
        kf = torch.minimum(k_reuse, cand.sum(1))
        reuse = torch.zeros((S, N), dtype=torch.bool, device=rgb.device)
        rank = torch.arange(N, device=rgb.device)[None].expand(S, N)
        reuse.scatter_(1, order, rank < kf[:, None])
        src = torch.where(reuse, si * G + sj, torch.full_like(si, -1)).int()
        self.prev = spec
        return src


def torch_splice(src, cache, fresh):
    idx = src.clamp(min=0).long()
    gathered = torch.gather(cache, 1, idx[..., None].expand(-1, -1, D))
    return torch.where((src >= 0)[..., None], gathered, fresh)


def timeit(fn, n=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn(0)
    torch.cuda.synchronize()
    e0.record()
    for i in range(n):
        fn(i + 1)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def main():
    dev = torch.device("cuda")
    frames = torch.empty((R, S, H, H, 3), dtype=torch.float32, device=dev)
    for c0 in range(0, S, 64):
        frames[:, c0:c0 + 64] = torch_stream_frames(min(64, S - c0), R, H, H, seed=5000 + c0, device=dev)
    g = torch.Generator(device=dev).manual_seed(3000)
    cache = torch.empty((2, S, N, D), dtype=torch.bfloat16, device=dev)
    cache[0].normal_(generator=g)
    fresh = torch.empty((S, N, D), dtype=torch.bfloat16, device=dev).normal_(generator=g)
    ages = torch.zeros((2, S, N), dtype=torch.int64, device=dev)

    ts = TorchSelect(dev)
    ts(frames[0])
    state = {"cache": cache[0].clone()}

    def vendor_step(i):
        src = ts(frames[i % R])
        state["cache"] = torch_splice(src, state["cache"], fresh)

    vendor_ms = timeit(vendor_step)

    eng = fc.FreqCacheEngine(S, H, H, P, fmt="rgb", device=dev)
    spl = fc.SpliceState(cache, ages)
    cfg = fc.CacheConfig(patch_size=P)
    eng.select(frames[0], cfg, refresh_shift=1)

    def ours_step(i):
        out = eng.select(frames[i % R], cfg, refresh_shift=1)
        spl.step(out.src_map, fresh)

    ours_ms = timeit(ours_step)
    line = {"workload": "config 5 per GPU: 512 streams, 448x448x3 fp32, P=14, select + bf16 splice (D=1152)",
            "vendor_path": "torch.fft.rfft2/irfft2 (cuFFT) + torch einsum low-corner DCT (fp64, Parseval), reductions, sort, gather",
            "vendor_ms_per_step": vendor_ms, "vendor_frames_per_s": S / (vendor_ms / 1e3),
            "ours_ms_per_step_serial": ours_ms, "ours_frames_per_s_serial": S / (ours_ms / 1e3),
            "speedup": vendor_ms / ours_ms, "streams": S}
    print(json.dumps(line), flush=True)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(line, f, indent=1)


if __name__ == "__main__":
    main()
