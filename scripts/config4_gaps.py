"""Diagnostics: interleaved per-step device time of the full-recompute graph,
the layer1 tail graph alone and the layer1 step (clock drift cancels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2604_24391_b200 import CacheConfig
from paper_2604_24391_b200.synth import torch_stream_frames
from paper_2604_24391_b200.vit import CachedEncoder, GraphedViT, ViT, ViTConfig

S, T = 16, 24
dev = torch.device("cuda")
c = ViTConfig()
model = ViT(c).to(dev, torch.bfloat16).eval()
frames = torch_stream_frames(S, T, c.image, c.image, seed=1000, device=dev)
cfg = CacheConfig(patch_size=c.patch)
with torch.no_grad():
    gfull = GraphedViT(model, S)
    enc = CachedEncoder(model, S, mode="layer1")
    enc.step(frames[0], cfg, next_frames=frames[1])
    torch.cuda.synchronize()
    acc = {"full": [], "tail": [], "layer1": []}
    for t in range(1, T):
        for k, fn in (("full", lambda: gfull(frames[t])), ("tail", lambda: enc.tail_graphs[t & 1].replay()),
                      ("layer1", lambda: enc.step(frames[t], cfg, next_frames=frames[t + 1] if t + 1 < T else None))):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            acc[k].append((a, b))
    torch.cuda.synchronize()
    print(os.environ.get("FC_VIT_SELECT_MAIN", "0"), {k: round(sum(a.elapsed_time(b) for a, b in v[2:]) / len(v[2:]), 3)
                                                      for k, v in acc.items()})
    # where the layer1 step's time goes (events inside the step)
    enc.debug_marks = []
    import time
    h0 = time.perf_counter()
    for t in range(1, T):
        enc.step(frames[t], cfg, next_frames=frames[t + 1] if t + 1 < T else None)
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    h2 = time.perf_counter()
    m = enc.debug_marks[2:]
    print("block0 ms", sum(a.elapsed_time(b) for a, b, _ in m) / len(m), "tail ms",
          sum(b.elapsed_time(c) for _, b, c in m) / len(m),
          "gap to next step ms", sum(x[2].elapsed_time(y[0]) for x, y in zip(m, m[1:])) / (len(m) - 1),
          "host enqueue ms/step", (h1 - h0) * 1e3 / (T - 1), "drain ms", (h2 - h1) * 1e3)
