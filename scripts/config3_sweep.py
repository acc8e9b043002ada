"""BASELINE config 3 measurement: select + token splice at 256 streams with the
reuse ratio swept through BudgetConfig(r, r), r = 0.2 .. 0.8 (one B200).

Per r: achieved reuse (K_final / N, which is min(K_reuse, K_cand)), device
time of select + in-place splice per step (CUDA events, 20 steps after
warm-up, frames from a resident 4-step ring, serial launch order), frames/s,
and the splice's bytes moved and GB/s.  Prints one JSON object per r and a
summary list; `--out` writes the list.

Launch order is serial, so the splice runs alone: its copier is sized as
for a standalone splice (FC_SPLICE_BULK_CTAS=2, two CTAs per SM) unless the
environment says otherwise — the 1-CTA/SM default is sized to co-run with
the select kernels in the pipelined step.
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

os.environ.setdefault("FC_SPLICE_BULK_CTAS", "2")
import paper_2604_24391_b200 as fc  # noqa: E402
from paper_2604_24391_b200.synth import torch_stream_frames


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--streams", type=int, default=256)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    S, H, P, D, R = a.streams, 448, 14, 1152, 4
    dev = torch.device("cuda")
    frames = torch.empty((R, S, H, H, 3), dtype=torch.float32, device=dev)
    for c0 in range(0, S, 64):
        c1 = min(S, c0 + 64)
        frames[:, c0:c1] = torch_stream_frames(c1 - c0, R, H, H, seed=3000 + c0, device=dev)
    g = torch.Generator(device=dev).manual_seed(3000)
    cache = torch.empty((2, S, 1024, D), dtype=torch.bfloat16, device=dev)
    cache[0].normal_(generator=g)
    fresh = torch.empty((S, 1024, D), dtype=torch.bfloat16, device=dev).normal_(generator=g)
    ages = torch.zeros((2, S, 1024), dtype=torch.int64, device=dev)
    rows = []
    for r in (0.2, 0.35, 0.5, 0.65, 0.8):
        cfg = fc.CacheConfig(patch_size=P, budget=fc.BudgetConfig(r, r))
        eng = fc.FreqCacheEngine(S, H, H, P, fmt="rgb", device=dev)
        spl = fc.SpliceState(cache, ages)
        for t in range(3):
            out = eng.select(frames[t % R], cfg)
            spl.step(out.src_map, fresh)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for t in range(a.steps):
            out = eng.select(frames[(3 + t) % R], cfg)
            spl.step(out.src_map, fresh)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        res = out.host_results()
        N = eng.n_tokens
        k = res["k_final"]
        shifted = (k > 0) & ((res["di_patches"] != 0) | (res["dj_patches"] != 0))
        rows_moved = int(np.where(shifted, N, N - k).sum())
        moved = rows_moved * 2 * D * 2 + S * 20 * N
        # splice alone (same decisions), for its bandwidth
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.steps):
            spl.step(out.src_map, fresh)
        e1.record()
        torch.cuda.synchronize()
        spl_ms = e0.elapsed_time(e1) / a.steps
        row = {"target_reuse": r, "achieved_reuse_mean": float(k.mean() / N), "achieved_reuse_min": float(k.min() / N),
               "achieved_reuse_max": float(k.max() / N), "flush_rate": float(res["flushed"].mean()),
               "ms_per_step_select_plus_splice": ms, "frames_per_s": S / (ms / 1e3),
               "splice_ms": spl_ms, "splice_moved_bytes": moved, "splice_gbs": moved / (spl_ms / 1e3) / 1e9,
               "streams": S, "steps": a.steps}
        print(json.dumps(row), flush=True)
        rows.append(row)
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"config": "BASELINE config 3 (256 streams, 448x448x3, N=1024, D=1152 bf16, reuse sweep)",
                       "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
