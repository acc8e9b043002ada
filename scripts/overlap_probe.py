"""Diagnostics: per-step device time of subsets of the pipelined step at a
given per-GPU batch (graph-captured phases, CUDA events): front only, back
only, front + back, splice only, all three.  Shows how much each branch
costs on its own and how well they overlap.

    S=64 python scripts/overlap_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2604_24391_b200 import CacheConfig, FreqCacheEngine, SpliceState, StepGraph
from paper_2604_24391_b200.synth import torch_stream_frames

S, H, P, D, R = int(os.environ.get("S", 64)), 448, 14, 1152, 8
dev = torch.device("cuda")
frames = torch.empty((R, S, H, H, 3), dtype=torch.float32, device=dev)
for c0 in range(0, S, 64):
    frames[:, c0:c0 + 64] = torch_stream_frames(min(64, S - c0), R, H, H, seed=7 + c0, device=dev)
N = 1024
cache = torch.randn((2, S, N, D), device=dev).to(torch.bfloat16)
fresh = torch.randn((S, N, D), device=dev).to(torch.bfloat16)
ages = torch.zeros((2, S, N), dtype=torch.int64, device=dev)
os.environ["FC_PROBE_BACK_PART"] = "all"   # the plan reads the per-call probe knob (deep variant)
eng = FreqCacheEngine(S, H, H, P, fmt="rgb")
del os.environ["FC_PROBE_BACK_PART"]
spl = SpliceState(cache, ages)
cfg = CacheConfig(patch_size=P)
outs = [eng.new_output(), eng.new_output()]
for t in range(4):
    eng.select(frames[t % R], cfg, out=outs[t & 1], refresh_shift=1)
eng.select_front(frames[0], cfg, outs[0], 0, refresh_shift=1)
eng.select_front(frames[1], cfg, outs[1], 1, refresh_shift=1)
torch.cuda.synchronize()
fs = torch.cuda.Stream()
side = torch.cuda.Stream(priority=-1)


bs2 = torch.cuda.Stream()


def make(t, front, back, splice, whole=False, deep=False):
    def fn():
        cur = torch.cuda.current_stream()
        fs.wait_stream(cur)
        side.wait_stream(cur)
        bs2.wait_stream(cur)
        if deep:
            # timing only: K_B of step t + 1 beside K_C + K_D of step t (the
            # probe env launches one half of the back; T2 / sums unordered)
            with torch.cuda.stream(bs2):
                os.environ["FC_PROBE_BACK_PART"] = "cols"
                eng.select_back(cfg, outs[(t + 1) & 1], (t + 1) & 1, refresh_shift=1)
            os.environ["FC_PROBE_BACK_PART"] = "tail"
            eng.select_back(cfg, outs[t & 1], t & 1, refresh_shift=1)
            del os.environ["FC_PROBE_BACK_PART"]
            cur.wait_stream(bs2)
        if whole:
            eng.select(frames[t % R], cfg, out=outs[t & 1], refresh_shift=1)
        if front:
            with torch.cuda.stream(fs):
                eng.select_front(frames[(t + 1) % R], cfg, outs[(t + 1) & 1], (t + 1) & 1, refresh_shift=1)
        if back:
            eng.select_back(cfg, outs[t & 1], t & 1, refresh_shift=1)
        if splice:
            with torch.cuda.stream(side):
                spl.step(outs[(t - 1) & 1].src_map, fresh)
        cur.wait_stream(fs)
        cur.wait_stream(side)
    return fn


ONLY = os.environ.get("PROBE_ONLY")


def timeit(label, front, back, splice, whole=False, n=64, deep=False):
    if ONLY and label.strip() != ONLY:
        return None
    base_k = spl.k
    graphs = []
    for p in range(R):
        spl.k = (base_k + p) & 1
        graphs.append(StepGraph(make(p + 1, front, back, splice, whole, deep)))
    spl.k = base_k
    for i in range(R):
        graphs[i].replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n):
        graphs[i % R].replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"S={S} {label:28s} {ms * 1e3:8.1f} us/step  {S / ms * 1e3:9.0f} frames/s", flush=True)
    return ms


timeit("front (K_A + K_D1)", True, False, False)
timeit("back (K_B + K_C + K_D)", False, True, False)
timeit("front + back", True, True, False)
timeit("splice", False, False, True)
timeit("front + back + splice", True, True, True)
timeit("deep: front+cols+tail+splice", True, False, True, deep=True)
timeit("deep: cols + tail", False, False, False, deep=True)
timeit("whole select", False, False, False, whole=True)
timeit("whole select + splice", False, False, True, whole=True)
prof = []
if ONLY:
    sys.exit(0)
eng.select(frames[0], cfg, refresh_shift=1, profile=prof)
print("serial kernels (rows_fwd, cols, rows_inv, K_D1+K_D):", ["%.1f" % (x * 1e3) for x in prof])
