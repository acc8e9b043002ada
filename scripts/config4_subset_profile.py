"""Diagnostics for config 4's subset mode: top kernels (torch.profiler) of
the full recompute (graph) and of the subset cached step, per step."""
import os
import sys

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
GRAPHS = os.environ.get("GRAPHS", "0") == "1"
with torch.no_grad():
    gfull = GraphedViT(model, S)
    enc = CachedEncoder(model, S, mode="subset", graphs=GRAPHS)
    for t in range(4):
        enc.step(frames[t], cfg)
    gfull(frames[0])
    torch.cuda.synchronize()
    for name, fn in (("full", lambda: [gfull(frames[t]) for t in range(4, T)]),
                     ("subset", lambda: [enc.step(frames[t], cfg, next_frames=frames[t + 1] if t + 1 < T else None)
                                         for t in range(4, T)])):
        fn()
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
            fn()
            torch.cuda.synchronize()
        print(f"===== {name} ({T - 4} steps)")
        print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30, max_name_column_width=70))
