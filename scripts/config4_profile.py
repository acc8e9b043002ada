"""Diagnostics for config 4: per-step device time of the full recompute
(graph), the layer1 cached step and its static tail alone, plus the top
kernels of each (torch.profiler)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2604_24391_b200 import CacheConfig
from paper_2604_24391_b200.synth import torch_stream_frames
from paper_2604_24391_b200.vit import CachedEncoder, GraphedViT, ViT, ViTConfig

S, T = 16, 12
dev = torch.device("cuda")
c = ViTConfig()
model = ViT(c).to(dev, torch.bfloat16).eval()
frames = torch_stream_frames(S, T, c.image, c.image, seed=1000, device=dev)
cfg = CacheConfig(patch_size=c.patch)
with torch.no_grad():
    gfull = GraphedViT(model, S)
    enc = CachedEncoder(model, S, mode="layer1")
    for t in range(4):
        enc.step(frames[t], cfg)
    torch.cuda.synchronize()

    def run_full():
        for t in range(4, T):
            gfull(frames[t])

    def run_l1():
        for t in range(4, T):
            enc.step(frames[t], cfg, next_frames=frames[t + 1] if t + 1 < T else None)

    def run_tail():
        for t in range(4, T):
            enc.tail_graphs[t & 1].replay()

    for name, fn in (("full-graph", run_full), ("layer1", run_l1), ("tail-graph", run_tail)):
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        print(name, "gpu ms/step", e0.elapsed_time(e1) / (T - 4), "wall ms/step",
              (time.perf_counter() - w0) * 1e3 / (T - 4), flush=True)
    import json
    dump = {}
    for name, fn in (("layer1", run_l1), ("full-graph", run_full)):
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            torch.cuda.synchronize()
        dump[name] = {e.key: [e.count, e.device_time_total] for e in prof.key_averages()}
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/config4_kernels.json", "w") as f:
        json.dump(dump, f, indent=1)
