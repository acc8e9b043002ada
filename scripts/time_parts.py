"""Diagnostics: device time of select only / splice only / both (512 streams, 448^2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_24391_b200 import CacheConfig, FreqCacheEngine, splice
from paper_2604_24391_b200.synth import torch_stream_frames

S, H, P, D, R = int(os.environ.get("S", 512)), 448, 14, 1152, 4
dev = torch.device("cuda")
frames = torch.empty((R, S, H, H, 3), dtype=torch.float32, device=dev)
for c0 in range(0, S, 64):
    frames[:, c0:c0 + 64] = torch_stream_frames(min(64, S - c0), R, H, H, seed=7 + c0, device=dev)
cache = torch.randn((2, S, 1024, D), device=dev).to(torch.bfloat16)
fresh = torch.randn((S, 1024, D), device=dev).to(torch.bfloat16)
ages = torch.zeros((2, S, 1024), dtype=torch.int64, device=dev)
eng = FreqCacheEngine(S, H, H, P, fmt="rgb")
cfg = CacheConfig(patch_size=P)
for t in range(3):
    out = eng.select(frames[t % R], cfg, refresh_shift=1)
torch.cuda.synchronize()

def timeit(fn, n=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn(0); torch.cuda.synchronize()
    e0.record()
    for i in range(n):
        fn(i)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n

sel = timeit(lambda i: eng.select(frames[i % R], cfg, refresh_shift=1))
spl = timeit(lambda i: splice(out.src_map, cache[i & 1], ages[i & 1], fresh, cache[1 - (i & 1)], ages[1 - (i & 1)]))
both = timeit(lambda i: (eng.select(frames[i % R], cfg, refresh_shift=1),
                         splice(out.src_map, cache[i & 1], ages[i & 1], fresh, cache[1 - (i & 1)], ages[1 - (i & 1)])))
prof = []
eng.select(frames[0], cfg, refresh_shift=1, profile=prof)
print(f"S={S} chunk={os.environ.get('FC_CHUNK','def')} lanes={os.environ.get('FC_LANES','def')}: "
      f"select {sel:.3f} ms  splice {spl:.3f} ms  serial both {both:.3f} ms  | serial kernels {['%.3f' % x for x in prof]}")
