#!/usr/bin/env python
"""FreqCache select + splice throughput on B200 (BASELINE config 5).

One step = one decision (fc_select: luma + block-DCT energy, 2-D FFT, phase
correlation, entropy budget, top-K) plus the bf16 hidden-state splice
(fc_splice_inplace, 1024 x 1152 per stream) for every stream of the job.

Workload (config 5 as written): 512 independent streams of 448x448x3 fp32
frames in total, sharded by stream across the ranks (512 / N per GPU, no
data-path collective; ``"scaling": "strong"``), P=14 (1024 tokens),
adaptive budget, config-2 refresh rule (flush when the patch shift exceeds
1), cache/fresh hidden states N(0,1) bf16.  ``--weak`` keeps 512 streams per
GPU instead.  Frames are synthetic (paper_2604_24391_b200.synth, torch draw
on the GPU, untimed) in a ring of 24 resident steps; each step reads
1.23 GB of frames (> L2).  Each pipelined step (select of step t beside the
splice of step t - 1) is one CUDA-graph launch.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

``--gpus N`` without torchrun re-launches itself under
``torch.distributed.run`` with N ranks (one per GPU, NCCL).  Prints ONE JSON
line on rank 0; at N > 1 it carries a weak-scaling leg (512 streams per
rank) beside the strong headline.

Environment (defaults are the measured best): FC_BENCH_SPLICE_BOOST
(extra copier CTAs joining each splice behind the back branch; 2 per SM above
128 streams per GPU, else 0), FC_BENCH_SPLICE_BOOST_ON=front, the stream
priorities FC_BENCH_{SIDE,FRONT,BACK}_PRIO, the library's FC_* kernel knobs;
FC_BENCH_DEVICE / FC_DIST_BACKEND=gloo run several ranks on one GPU (a
plumbing check, not a scaling number); FC_BENCH_PLUMBING=1 runs the
multi-rank reporting path without kernels (CPU tests).
"""

from __future__ import annotations

import argparse
import json

import numpy as np
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FreqCache select+splice frames/s & tokens/s at 1/2/4/8 B200; % of HBM/TC roofline"
UNIT = "frames/s"
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=128)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--streams", type=int, default=512,
                    help="streams of the whole job (config 5), sharded across the ranks; "
                         "with --weak: streams per rank")
    ap.add_argument("--weak", action="store_true", help="--streams per rank instead of in total")
    ap.add_argument("--size", type=int, default=448)
    ap.add_argument("--patch", type=int, default=14)
    ap.add_argument("--dim", type=int, default=1152)
    ap.add_argument("--ring", type=int, default=24, help="resident frame steps (even)")
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--sustained-s", type=float, default=1.5,
                    help="length of the sustained leg (0: skip)")
    ap.add_argument("--no-graph", action="store_true", help="launch every step eagerly")
    ap.add_argument("--graph-steps", type=int, default=1,
                    help="pipelined steps per CUDA graph without per-step joins (divides --ring; 1: per-step)")
    ap.add_argument("--no-pipeline", action="store_true",
                    help="whole select per step (no front/back overlap across steps)")
    ap.add_argument("--cpu-streams", type=int, default=64)
    ap.add_argument("--cpu-steps", type=int, default=6)
    ap.add_argument("--cpu-kind", default="auto", choices=["auto", "reference", "port"],
                    help="CPU baseline: the reference package (baseline/_ref) or the oracle port")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--refresh-shift", type=int, default=1)
    return ap.parse_args(argv)


def free_port():
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_command(argv, gpus, port):
    """torchrun command that re-runs this script with one rank per GPU."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *argv]


# ------------------------------------------------------------- CPU legs ----

def reference_available():
    """The unmodified reference package, installed into baseline/_ref."""
    if not os.path.isdir(os.path.join(REF_DIR, "freqcache")):
        return False
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import freqcache  # noqa: F401
        return os.path.abspath(freqcache.__file__).startswith(os.path.abspath(REF_DIR))
    except ImportError:
        return False


def _bf16_rows(rng, n, dim):
    """bf16 N(0,1) rows as their 16-bit patterns (bit copies everywhere)."""
    return (rng.standard_normal((n, dim), dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)


def _cpu_worker(args):
    """One host core: decide + splice for its streams, timed per step.

    kind "reference": the reference's own ``decide`` and ``step``
    (fusion.py:121-242, 462-512) from baseline/_ref — gray frames by its
    LUMA_WEIGHTS (frameio.py:26,85-88), hidden states as float64 tokens
    (bf16 values, exact), fresh rows fed to ``step`` through its token_fn in
    row-major recompute order, the config-2 shift rule applied on top.
    kind "port": the oracle restatement (oracle/freqcache_oracle.py)."""
    kind, streams, steps, warmup, size, patch, dim, refresh_shift, seed = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import dataclasses
    from paper_2604_24391_b200.synth import stream_frames
    n = (size // patch) ** 2
    total = warmup + steps + 1
    data = []
    for s in streams:
        fr = stream_frames(seed, s, total, size, size)
        rng = np.random.default_rng([3000, s])
        data.append((fr, _bf16_rows(rng, n, dim), _bf16_rows(rng, n, dim)))
    if kind == "reference":
        sys.path.insert(0, REF_DIR)
        import freqcache as ref
        from freqcache.frameio import LUMA_WEIGHTS
        cfg = ref.CacheConfig(patch_size=patch)
        rows = size // patch

        def gray(rgb):
            a = rgb.astype(np.float64)
            return LUMA_WEIGHTS[0] * a[..., 0] + LUMA_WEIGHTS[1] * a[..., 1] + LUMA_WEIGHTS[2] * a[..., 2]

        def bf16_f64(u16):
            return (u16.astype(np.uint32) << 16).view(np.float32).astype(np.float64)

        state = [ref.TokenCache(bf16_f64(c).reshape(rows, rows, dim), np.zeros((rows, rows), np.int64))
                 for _, c, _ in data]
        fresh64 = [bf16_f64(f) for _, _, f in data]

        def one(k, t):
            fr = data[k][0]
            d = ref.decide(gray(fr[t - 1]), gray(fr[t]), cfg, step=t)
            if (refresh_shift is not None and refresh_shift >= 0 and d.diagnostic is None and not d.flushed
                    and max(abs(d.displacement.di_patches), abs(d.displacement.dj_patches)) > refresh_shift):
                d = dataclasses.replace(d, flushed=True, k_candidate=0, k_final=0, reuse_set=(),
                                        recompute_set=tuple(range(n)))
            rec = iter(fresh64[k][list(d.recompute_set)] if not d.flushed else fresh64[k])
            state[k], _ = ref.step(state[k], d, gray(fr[t]), lambda patch_: next(rec))
    else:
        from oracle import freqcache_oracle as O
        cfg = O.OracleConfig(patch_size=patch, refresh_shift=refresh_shift)
        state = [(c, np.zeros(n, dtype=np.int64)) for _, c, _ in data]

        def one(k, t):
            fr, _, fresh = data[k]
            d = O.decide(fr[t - 1], fr[t], cfg, step=t)
            state[k] = O.splice(state[k][0], state[k][1], d, fresh[list(d.recompute_set)])
    t_timed = 0.0
    frames_done = 0
    for t in range(1, total):
        t0 = time.perf_counter()
        for k in range(len(data)):
            one(k, t)
        dt = time.perf_counter() - t0
        if t > warmup:
            t_timed += dt
            frames_done += len(data)
    return frames_done, t_timed


def cpu_run(kind, n_streams, steps, warmup, size, patch, dim, refresh_shift, seed=5000):
    """Whole-host CPU throughput (frames/s): one process per core, BLAS
    threads 1; returns (frames/s, cores, frames timed)."""
    import multiprocessing as mp
    cores = len(os.sched_getaffinity(0))
    workers = min(cores, n_streams)
    parts = [list(range(i, n_streams, workers)) for i in range(workers)]
    ctx = mp.get_context("spawn")
    env_keep = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")}
    for k in env_keep:
        os.environ[k] = "1"
    try:
        with ctx.Pool(workers) as pool:
            res = pool.map(_cpu_worker, [(kind, p, steps, warmup, size, patch, dim, refresh_shift, seed)
                                         for p in parts])
    finally:
        for k, v in env_keep.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    frames = sum(r[0] for r in res)
    wall = max(r[1] for r in res)
    return frames / wall if wall > 0 else 0.0, workers, frames


def cpu_kind(a):
    if a.cpu_kind == "port":
        return "port"
    ok = reference_available()
    if a.cpu_kind == "reference" and not ok:
        raise SystemExit("--cpu-kind reference: baseline/_ref/freqcache is not installed")
    return "reference" if ok else "port"


def cpu_sample_text(kind, streams, steps, warmup, frames):
    what = ("the reference's own decide + step (baseline/_ref freqcache, unmodified; luma by its "
            "LUMA_WEIGHTS, fresh rows through its token_fn, config-2 shift rule on top)"
            if kind == "reference" else "the oracle port (decide + splice)")
    return (f"{streams} streams x {steps} timed steps (+{warmup} warm-up) of {what}, {frames} frames, numpy "
            "draw of the same frozen generator, one process per core, BLAS threads 1")


def run_reference(a):
    """--impl reference: the reference's CPU path on all host cores (rank 0)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    t0 = time.time()
    kind = cpu_kind(a)
    v, cores, frames = cpu_run(kind, a.cpu_streams, a.steps, a.warmup, a.size, a.patch, a.dim, a.refresh_shift)
    line = {
        "metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * a.cpu_streams / v if v else None,
        "higher_is_better": True, "scaling": "weak" if a.weak else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (numpy draw of the frozen generator)",
        "config": {"workload": "config5 sample: decide+splice per frame, 448x448x3 fp32, P=14, N=1024, D=1152",
                   "streams": a.cpu_streams, "size": a.size, "patch": a.patch, "dim": a.dim,
                   "refresh_shift": a.refresh_shift},
        "tokens_per_s": v * (a.size // a.patch) ** 2,
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": cpu_sample_text(kind, a.cpu_streams, a.steps, a.warmup, frames)},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.time() - t0,
    }
    print(json.dumps(line), flush=True)


def run_plumbing(a):
    """FC_BENCH_PLUMBING=1 (CPU tests): the multi-rank launch and reporting
    path without kernels — gloo ranks, stream sharding, max-over-ranks
    timing, the counter all-reduce and the rank-0 line."""
    import torch
    import torch.distributed as dist
    from paper_2604_24391_b200.dist import gather_counters, max_over_ranks, shard
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    total = a.streams * world if a.weak else a.streams
    lo, hi = shard(total, world, rank)
    ms = max_over_ranks(1.0 + rank)
    n = (a.size // a.patch) ** 2
    cnt = gather_counters({"frames": (hi - lo) * a.steps, "tokens": (hi - lo) * a.steps * n,
                           "reused_tokens": 0, "flushes": 0, "cold": 0})
    spans = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    if world > 1:
        dist.all_gather(spans, torch.tensor([lo, hi], dtype=torch.int64))
    else:
        spans = [torch.tensor([lo, hi])]
    # the weak leg beside a strong headline: --streams per rank
    wlo, whi = (rank * a.streams, (rank + 1) * a.streams) if not a.weak else (lo, hi)
    wms = max_over_ranks(2.0 + rank)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "plumbing": True, "n_gpus": world, "ms_max": ms,
                          "weak_scaling": {"ms_max": wms, "span0": [wlo, whi],
                                           "streams_total": a.streams * world},
                          "streams_total": total, "streams_per_rank": [int(s[1] - s[0]) for s in spans],
                          "spans": [[int(s[0]), int(s[1])] for s in spans], "frames": cnt["frames"],
                          "scaling": "weak" if a.weak else "strong"}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ------------------------------------------------------------- GPU side ----

class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []          # (host time, csv line)
        self.window = None       # host-time bounds of the timed region

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi needs a moment before its first sample: wait for it
            # so the timed region (~0.1 s at the default size) is covered
            t_end = time.monotonic() + 5.0
            while not self.lines and time.monotonic() < t_end and self.proc.poll() is None:
                time.sleep(0.01)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def start(self):
        self.window = [time.monotonic(), None]

    def stop(self):
        # a sample is read shortly after it is taken: allow about one period
        time.sleep(0.03)
        self.window[1] = time.monotonic()
        return tuple(self.window)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, window=None):
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        window = window or self.window
        lo, hi = window if window and window[1] else (float("-inf"), float("inf"))
        for ts, ln in self.lines:
            if not (lo <= ts <= hi):
                continue
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sms.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sms)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


class Pipeline:
    """One rank's pipelined config-5 step on the GPU: resident frame ring,
    token caches, the engine and the in-place splice state, and the step
    replayed from CUDA graphs.  Step t = the front of select t + 1 (K_A,
    K_D1; workspace slot (t + 1) & 1) beside the back of select t (K_B, K_C,
    K_D; slot t & 1) beside the in-place splice of step t - 1, each on its
    own stream, joined at the end of the step.  Select outputs are
    double-buffered: the front of t + 1 writes only the energies of buffer
    (t + 1) & 1 while the splice of t - 1 reads that buffer's splice map.
    --no-pipeline: select(t) as one call beside the splice of t - 1.
    --graph-steps G > 1: chunks of G steps per graph without per-step joins
    (every branch waits only on the events of the work it depends on)."""

    def __init__(self, a, dev, S, lo, rank, R):
        import torch

        from paper_2604_24391_b200 import CacheConfig, FreqCacheEngine, SpliceState, StepGraph
        from paper_2604_24391_b200.synth import torch_stream_frames
        H, P, D = a.size, a.patch, a.dim
        N = (H // P) ** 2
        self.a, self.dev, self.R = a, dev, R
        self.cfg = cfg = CacheConfig(patch_size=P)
        # inputs, resident in HBM before timing (untimed generation); this
        # rank's streams are its contiguous block [lo, lo + S) of the job's
        self.frames = frames = torch.empty((R, S, H, H, 3), dtype=torch.float32, device=dev)
        for c0 in range(0, S, 64):
            c1 = min(S, c0 + 64)
            frames[:, c0:c1] = torch_stream_frames(c1 - c0, R, H, H, seed=5000 + lo + c0, device=dev)
        g = torch.Generator(device=dev).manual_seed(3000 + rank)
        cache = torch.empty((2, S, N, D), dtype=torch.bfloat16, device=dev)
        cache[0].normal_(generator=g)
        self.fresh = fresh = torch.empty((S, N, D), dtype=torch.bfloat16, device=dev).normal_(generator=g)
        ages = torch.zeros((2, S, N), dtype=torch.int64, device=dev)
        self.eng = eng = FreqCacheEngine(S, H, H, P, fmt="rgb", device=dev)
        self.spl = spl = SpliceState(cache, ages)   # in place where the displacement is zero, else ping-pong
        # run_sequence aggregates over the timed steps, accumulated by the
        # select kernel itself (frames, reused tokens, flushes, cold)
        self.counters = torch.zeros(4, dtype=torch.int64, device=dev)
        self.outs = outs = [eng.out, eng.new_output()]
        for o in outs:
            o.counters = self.counters
        torch.cuda.synchronize()
        self.launches = [0]
        self.per_phase = (eng.launches_per_select if a.no_pipeline else eng.launches_per_split_step) + 2
        self.n_spliced = n_spliced = [0]   # splices issued so far: SpliceState's ping-pong parity
        side = torch.cuda.Stream(dev, priority=int(os.environ.get("FC_BENCH_SIDE_PRIO", "-1")))
        fs = torch.cuda.Stream(dev, priority=int(os.environ.get("FC_BENCH_FRONT_PRIO", "0")))
        bs = torch.cuda.Stream(dev, priority=int(os.environ.get("FC_BENCH_BACK_PRIO", "0")))
        rs = a.refresh_shift

        # the splice of t - 1 gets 2 more copier CTAs per SM once the back of
        # t is done (they take only unclaimed rows): +0.7 % at 512 streams,
        # -1 % at 64, so on above 128 streams per GPU;
        # FC_BENCH_SPLICE_BOOST=c sets the CTA count (0: off)
        nsm = torch.cuda.get_device_properties(dev).multi_processor_count
        boost = int(os.environ.get("FC_BENCH_SPLICE_BOOST", str(2 * nsm if S > 128 else 0)))
        if boost > 0 and not a.no_pipeline:
            self.per_phase += 1          # the extra copier launch
        self.boost = boost if not a.no_pipeline else 0
        boost_on_front = os.environ.get("FC_BENCH_SPLICE_BOOST_ON", "back") == "front"

        def phase(t):
            cur = torch.cuda.current_stream(dev)
            side.wait_stream(cur)
            if a.no_pipeline:
                eng.select(frames[t % R], cfg, out=outs[t & 1], refresh_shift=rs)
            else:
                if t == 0:
                    eng.select_front(frames[0], cfg, outs[0], 0, refresh_shift=rs)
                fs.wait_stream(cur)
                with torch.cuda.stream(fs):
                    eng.select_front(frames[(t + 1) % R], cfg, outs[(t + 1) & 1], (t + 1) & 1, refresh_shift=rs)
                bs.wait_stream(cur)
                with torch.cuda.stream(bs):
                    eng.select_back(cfg, outs[t & 1], t & 1, refresh_shift=rs)
            if t > 0:
                with torch.cuda.stream(side):
                    spl.step(outs[(t - 1) & 1].src_map, fresh, boostable=boost > 0 and not a.no_pipeline)
                n_spliced[0] += 1
                if boost > 0 and not a.no_pipeline:
                    with torch.cuda.stream(fs if boost_on_front else bs):
                        spl.boost(boost)
                cur.wait_stream(side)
            if not a.no_pipeline:
                cur.wait_stream(bs)
                cur.wait_stream(fs)

        ev = {k: [torch.cuda.Event(), torch.cuda.Event()] for k in ("front", "back", "splice")}
        live = set()   # (kind, parity) recorded inside the current capture

        def wait(stream, kind, t):
            if t >= 0 and (kind, t & 1) in live:
                stream.wait_event(ev[kind][t & 1])

        def mark(stream, kind, t):
            ev[kind][t & 1].record(stream)
            live.add((kind, t & 1))

        def chunk(t0, n):
            cur = torch.cuda.current_stream(dev)
            live.clear()
            for st_ in (fs, bs, side):
                st_.wait_stream(cur)
            for t in range(t0, t0 + n):
                wait(fs, "back", t - 1)
                with torch.cuda.stream(fs):
                    eng.select_front(frames[(t + 1) % R], cfg, outs[(t + 1) & 1], (t + 1) & 1, refresh_shift=rs)
                mark(fs, "front", t + 1)
                wait(side, "back", t - 1)
                with torch.cuda.stream(side):
                    spl.step(outs[(t - 1) & 1].src_map, fresh)
                n_spliced[0] += 1
                mark(side, "splice", t - 1)
                wait(bs, "front", t)
                wait(bs, "splice", t - 2)
                with torch.cuda.stream(bs):
                    eng.select_back(cfg, outs[t & 1], t & 1, refresh_shift=rs)
                mark(bs, "back", t)
            for st_ in (fs, bs, side):
                cur.wait_stream(st_)

        self.phase = phase
        # CUDA graphs: one per ring phase (frames[t % R], outs[t & 1] and the
        # splice ping-pong parity repeat with period R), and one per chunk of
        # G phases starting at t = 1 (mod G), G dividing R
        self.graphs = self.chunk_graphs = None
        self.G = G = a.graph_steps if (a.graph_steps > 1 and R % a.graph_steps == 0 and not a.no_pipeline) else 1
        phase(0)                                   # step 0 establishes every stream's spectrum
        self.t_next = 1
        if not a.no_graph:
            base = n_spliced[0]
            self.graphs = []
            for p in range(R):
                t = self.t_next + p
                spl.k = (base + (t - 1)) & 1      # the parity splice(t - 1) has at replay
                self.graphs.append(StepGraph(lambda t=t: phase(t), device=dev))
            if G > 1:
                self.chunk_graphs = []
                for c0 in range(1, R + 1, G):
                    spl.k = (base + (c0 - 1)) & 1
                    self.chunk_graphs.append(StepGraph(lambda c0=c0: chunk(c0, G), device=dev))
            n_spliced[0] = base
            spl.k = base & 1
            torch.cuda.synchronize()

    def advance(self, n):
        """n pipelined steps from t_next (whole chunks where aligned)."""
        R, G = self.R, self.G
        while n > 0:
            t = self.t_next
            if self.chunk_graphs is not None and (t - 1) % G == 0 and n >= G:
                self.chunk_graphs[((t - 1) % R) // G].replay()
                k = G
            elif self.graphs is not None:
                self.graphs[(t - 1) % R].replay()
                k = 1
            else:
                self.phase(t)
                k = 1
            if self.graphs is not None:
                self.n_spliced[0] += k
                self.spl.k = self.n_spliced[0] & 1
            self.launches[0] += self.per_phase * k
            self.t_next += k
            n -= k


def run_ours(a):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # FC_BENCH_DEVICE / FC_DIST_BACKEND: plumbing checks of the multi-rank
    # path on a one-GPU box (ranks share the device over gloo; not a scaling
    # measurement — the driver's runs use one GPU per rank over NCCL)
    local = int(os.environ.get("FC_BENCH_DEVICE", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("FC_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    from paper_2604_24391_b200 import CacheConfig, FreqCacheEngine, SpliceState

    H, P, D, R = a.size, a.patch, a.dim, a.ring + (a.ring & 1)
    total_streams = a.streams * world if a.weak else a.streams
    N = (H // P) ** 2
    cfg = CacheConfig(patch_size=P)

    from paper_2604_24391_b200.dist import gather_counters, shard
    lo, hi = shard(total_streams, world, rank)
    S = hi - lo
    pl = Pipeline(a, dev, S, lo, rank, R)
    frames, eng, spl, outs, fresh, counters = pl.frames, pl.eng, pl.spl, pl.outs, pl.fresh, pl.counters
    n_spliced, launches, splice_bytes = pl.n_spliced, pl.launches, [0]

    def one_step(t, kernel_ms):
        """Serial select + splice with per-kernel timing (events between launches)."""
        fr = frames[t % R]
        prof = []
        out = eng.select(fr, cfg, refresh_shift=a.refresh_shift, profile=prof)
        for k in range(5):
            kernel_ms[k] += prof[k]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        spl.step(out.src_map, fresh)
        n_spliced[0] += 1
        e1.record()
        torch.cuda.synchronize()
        kernel_ms[5] += e0.elapsed_time(e1)
        # bytes the splice actually moves this step: in-place streams only
        # their recomputed rows, shifted streams every row
        r = out.host_results()
        moved = ((r["k_final"] > 0) & ((r["di_patches"] != 0) | (r["dj_patches"] != 0)))
        rows_moved = np.where(moved, N, N - r["k_final"]).sum()
        splice_bytes[0] += int(rows_moved) * 2 * D * 2 + S * 20 * N
        return out

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def advance(n):
        pl.advance(n)

    # clock sampling starts before the warm-up, so the GPU does not idle while
    # nvidia-smi starts; only samples inside the timed region are kept
    clocks = ClockSampler(local).__enter__()
    # ---- warm-up: step 0 (above) + W - 1 pipelined steps
    advance(max(0, a.warmup - 1))
    barrier()

    # ---- timed region: K pipelined steps (K selects beside K splices), CUDA
    # events on the launching stream, max over ranks
    stream = torch.cuda.current_stream(dev)
    counters.zero_()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches[0] = 0
    sustained = None
    try:
        barrier()
        clocks.start()
        ev0.record(stream)
        advance(a.steps)
        ev1.record(stream)
        barrier()
        win_main = clocks.stop()
        gpu_launches = launches[0]
        ms = ev0.elapsed_time(ev1)
        t_max = torch.tensor([ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t_max, op=dist.ReduceOp.MAX)   # every rank sizes the sustained leg alike
        ms = float(t_max.item())
        cnt_dev = counters.clone()
        # ---- sustained leg: the same steps for >= --sustained-s seconds, with
        # its own clock record (the short default region runs at burst clocks)
        if a.sustained_s > 0:
            # 1.25x margin: the sustained steps may run faster than the first K
            n_s = max(a.steps, int(1.25 * a.sustained_s * 1e3 / max(ms / a.steps, 1e-3)) + 1)
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier()
            clocks.start()
            s0.record(stream)
            advance(n_s)
            s1.record(stream)
            barrier()
            win_s = clocks.stop()
            sms = torch.tensor([s0.elapsed_time(s1)], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(sms, op=dist.ReduceOp.MAX)
            sms = float(sms.item())
            sustained = {"value": total_streams * n_s / (sms / 1e3), "unit": UNIT, "steps": n_s,
                         "seconds": sms / 1e3, "ms_per_step": sms / n_s, "clocks": clocks.summary(win_s)}
    finally:
        clocks.__exit__(None, None, None)
    frames_total = total_streams * a.steps
    value = frames_total / (ms / 1e3)

    # decision statistics over every timed step of every rank (the only other
    # collective: a few counters, NCCL all-reduce over NVLink)
    c = cnt_dev.cpu().tolist()
    cnt = gather_counters({"frames": c[0], "tokens": c[0] * N, "reused_tokens": c[1], "flushes": c[2],
                           "cold": c[3]}, device=dev)
    reuse_ratio = cnt["reused_tokens"] / max(cnt["tokens"], 1)
    flush_rate = cnt["flushes"] / max(cnt["frames"], 1)

    # complete the last pipelined step's splice, then the serial pass
    t_next = pl.t_next
    spl.step(outs[(t_next - 1) & 1].src_map, fresh)
    n_spliced[0] += 1
    torch.cuda.synchronize()

    # ---- per-kernel timing pass (same steps, events between launches)
    kp_steps = min(a.steps, 16)
    names = ["rows_fwd", "cols", "rows_inv", "select", "rank", "splice"]
    kms = [0.0] * 6
    t0 = t_next
    for t in range(t0, t0 + kp_steps):
        one_step(t, kms)
    kms = [v / kp_steps for v in kms]
    splice_moved = splice_bytes[0] / kp_steps
    # the same splice alone with the copier twice as wide (2 CTAs per SM, the
    # standalone-best sizing): the step's copier is sized to co-run with the
    # select kernels and leaves them HBM, so alone it is slower
    wide = [0.0] * 6
    sb0 = splice_bytes[0]
    old = os.environ.get("FC_SPLICE_BULK_CTAS")
    os.environ["FC_SPLICE_BULK_CTAS"] = "2"
    try:
        for t in range(t0 + kp_steps, t0 + 2 * kp_steps):
            one_step(t, wide)
    finally:
        if old is None:
            os.environ.pop("FC_SPLICE_BULK_CTAS", None)
        else:
            os.environ["FC_SPLICE_BULK_CTAS"] = old
    wide_ms = wide[5] / kp_steps
    wide_bytes = (splice_bytes[0] - sb0) / kp_steps
    t_next = t0 + 2 * kp_steps
    hw = H * H
    spec = 8 * H * ((H // 2 + 7) // 8) * 8   # one packed half-spectrum, fp32 complex
    kbytes = [
        S * (12 * hw + spec + 8 * N),          # rows_fwd K_A: RGB in, packed rows (T1) out, energies
        S * ((3 if kms[2] == 0 else 4) * spec),  # cols K_B: T1 in, state in/out, T2 out (K_BC fused: no T2)
        S * spec,                              # rows_inv K_C: T2 in
        S * (3 * N + 14 * N + 136),            # select K_D: order + refresh mask in, masks/indices out
        S * (8 * N + 3 * N + 32),              # rank K_D1: energies in, order + refresh mask + stats out
        splice_moved,                          # splice: rows it must move (recomputed / shifted), map, ages
    ]
    nk = len(names)
    dom = max(range(nk), key=lambda k: kms[k])
    hbm, peak_kind = peaks()
    ach = kbytes[dom] / (kms[dom] / 1e3) / 1e9
    b_sel = 20 * hw + 16 * N
    b_spl = 4 * N * D + 20 * N
    frames_per_s_gpu = (S * a.steps) / (ms / 1e3) if world == 1 else value / world
    step_ach = (b_sel + b_spl) * frames_per_s_gpu / 1e9
    moved_ach = (b_sel + splice_moved / S) * frames_per_s_gpu / 1e9
    roofline = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                "traffic": None, "kernel": names[dom], "peak_kind": peak_kind,
                "bytes_per_launch": kbytes[dom], "ms_per_launch": kms[dom],
                "note": "serialised pass, each kernel configured as in the timed step; the splice copier is "
                        "sized to co-run with the select kernels (1 CTA/SM), see splice_alone_wide; splice "
                        "bytes = the rows it must move (in-place streams skip their reused rows)"}
    if names[dom] == "splice":
        # SURVEY 8(d)'s literal per-stream splice figure (the out-of-place
        # gather's bytes), which the in-place splice undercuts
        alg = S * (4 * N * D + 20 * N)
        roofline["bytes_per_launch_8d"] = alg
        roofline["frac_8d"] = alg / (kms[dom] / 1e3) / 1e9 / hbm
    splice_wide = {"ms": wide_ms, "bytes": wide_bytes, "gbs": wide_bytes / (wide_ms / 1e3) / 1e9,
                   "frac": wide_bytes / (wide_ms / 1e3) / 1e9 / hbm,
                   "config": "FC_SPLICE_BULK_CTAS=2 (2 copier CTAs per SM), same splices, serialised"}
    roofline_step = {"bound": "hbm", "achieved": step_ach, "peak": hbm, "unit": "GB/s", "frac": step_ach / hbm,
                     "bytes_per_frame": b_sel + b_spl, "select_bytes": b_sel, "splice_bytes": b_spl,
                     "splice_moved_bytes_per_frame": splice_moved / S,
                     "achieved_moved": moved_ach, "frac_moved": moved_ach / hbm,
                     "note": "SURVEY 8(d) algorithmic bytes; the in-place splice moves only recomputed "
                             "rows of zero-displacement streams: frac_moved counts the select bytes plus "
                             "the splice bytes actually moved"}
    # (a kind with no launch, e.g. rows_inv when K_B + K_C run fused, is left out)
    kernels = {names[k]: {"ms": kms[k], "share": kms[k] / sum(kms), "bytes": kbytes[k],
                          "gbs": kbytes[k] / (kms[k] / 1e3) / 1e9} for k in range(nk) if kms[k] > 0}
    # ncu DRAM bytes per launch of the same kernel, from the capture named in
    # profiles/traffic.json (tagged with its capture id: it is not re-measured
    # by this run)
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tr = json.load(f)
        if isinstance(tr.get("kernels"), dict) and tr["kernels"].get(names[dom]) is not None:
            roofline["traffic"] = tr["kernels"][names[dom]]
            roofline["traffic_capture"] = tr.get("capture")
    except (OSError, ValueError):
        pass

    # ---- end to end: pinned host frames -> device -> select + splice -> results to host
    HR = min(2, R)  # pinned host ring: 2 steps (2.5 GB per rank at config 5)
    host = torch.empty((HR, S, H, H, 3), dtype=torch.float32, pin_memory=True)
    for i in range(HR):
        host[i].copy_(frames[(t0 + kp_steps + i) % R])
    res_host = torch.empty((S, 136), dtype=torch.uint8, pin_memory=True)
    map_host = torch.empty((S, N), dtype=torch.int32, pin_memory=True)
    ke = max(1, a.e2e_steps)

    def run_e2e(engine, host_ring):
        """Timed e2e steps through the public engine API; returns frames/s (whole job)."""
        engine.reset()
        torch.cuda.synchronize()
        # copies on their own stream into double-buffered staging, so the H2D of
        # step i+1 overlaps select + splice of step i; results come back per step
        copy_s = torch.cuda.Stream(dev)
        stages = [torch.empty(host_ring.shape[1:], dtype=host_ring.dtype, device=dev) for _ in range(2)]
        h2d_ev = [torch.cuda.Event(), torch.cuda.Event()]
        use_ev = [torch.cuda.Event(), torch.cuda.Event()]
        for e in use_ev:
            e.record(stream)

        def issue_copy(i):
            k = i & 1
            with torch.cuda.stream(copy_s):
                copy_s.wait_event(use_ev[k])
                stages[k].copy_(host_ring[i % HR], non_blocking=True)
                h2d_ev[k].record(copy_s)

        def step(i):
            k = i & 1
            stream.wait_event(h2d_ev[k])
            out = engine.select(stages[k], cfg, refresh_shift=a.refresh_shift)
            use_ev[k].record(stream)
            spl.step(out.src_map, fresh)
            res_host.copy_(out.results, non_blocking=True)
            map_host.copy_(out.src_map, non_blocking=True)

        issue_copy(0)
        step(0)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        issue_copy(1)
        for i in range(1, ke + 1):
            if i + 1 <= ke:
                issue_copy(i + 1)
            step(i)
        e1.record(stream)
        barrier()
        ems = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        return total_streams * ke / (float(ems.item()) / 1e3), stages

    e2e_val, stages = run_e2e(eng, host)
    h2d = total_streams * H * H * 3 * 4          # whole job, per step
    d2h = total_streams * 136 + total_streams * N * 4
    # the link the e2e number is bound by: plain pinned H2D copy of one step's frames
    for _ in range(2):
        stages[0].copy_(host[0], non_blocking=True)
    torch.cuda.synchronize()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for i in range(3):
        stages[i & 1].copy_(host[i % HR], non_blocking=True)
    p1.record(stream)
    torch.cuda.synchronize()
    pcie_gbs = 3 * S * H * H * 3 * 4 / (p0.elapsed_time(p1) / 1e3) / 1e9
    e2e_h2d_gbs = S * H * H * 3 * 4 * e2e_val / total_streams / 1e9   # per rank (its own PCIe link)
    del stages
    # the same e2e with frames in the reference's own ingest format (PPM P6
    # uint8 payloads, frameio.py; gray = luma / 255): a quarter of the H2D bytes.
    # Different input values (the fp32 frames quantised), so reported beside the
    # contract's e2e, not as it.
    host8 = (host * 255.0).round_().to(torch.uint8).pin_memory()
    eng8 = FreqCacheEngine(S, H, H, P, fmt="rgb_u8", device=dev)
    e2e8_val, stages8 = run_e2e(eng8, host8)
    del stages8, eng8, host8
    e2e8_h2d_gbs = S * H * H * 3 * e2e8_val / total_streams / 1e9

    # ---- single-stream step latency (select + splice), CUDA-graph replay:
    # config 1 (224x224, fixed 50 % budget) and one config-2 stream (448x448)
    latency = {}
    if rank == 0:
        for name, size, budget in (("config1_224", 224, (0.5, 0.5)), ("config2_448", 448, None)):
            from paper_2604_24391_b200 import BudgetConfig
            c1 = CacheConfig(patch_size=P) if budget is None else CacheConfig(patch_size=P, budget=BudgetConfig(*budget))
            e1 = FreqCacheEngine(1, size, size, P, fmt="rgb", device=dev)
            n1 = e1.n_tokens
            fr1 = frames[:2, :1, :size, :size].contiguous() if size <= H else None
            c1c = torch.randn((2, 1, n1, D), device=dev).to(torch.bfloat16)
            a1 = torch.zeros((2, 1, n1), dtype=torch.int64, device=dev)
            sp1 = SpliceState(c1c, a1)
            fz = torch.randn((1, n1, D), device=dev).to(torch.bfloat16)
            src_frame = torch.empty((1, size, size, 3), dtype=torch.float32, device=dev)
            src_frame.copy_(fr1[0])
            e1.select(src_frame, c1)
            src_frame.copy_(fr1[1])
            gs = torch.cuda.Stream(dev)
            gs.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(gs):
                for _ in range(3):
                    o1 = e1.select(src_frame, c1)
                    sp1.step(o1.src_map, fz)
            torch.cuda.current_stream(dev).wait_stream(gs)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                o1 = e1.select(src_frame, c1)
                sp1.step(o1.src_map, fz)
            sp1.k = 0  # the captured step always reads slot buffer 0 -> 1
            graph.replay()
            torch.cuda.synchronize()
            q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 200
            q0.record()
            for _ in range(reps):
                graph.replay()
            q1.record()
            torch.cuda.synchronize()
            latency[name] = {"ms_per_step": q0.elapsed_time(q1) / reps, "streams": 1, "size": size,
                             "tokens": n1, "path": "CUDA graph: fc_select + fc_splice_inplace"}
        latency["reference_paper_a100_ms"] = 2.54

    # ---- weak-scaling leg beside the strong headline (N > 1): --streams per
    # rank (rank r owns streams [r S', (r + 1) S')), its own pipeline, warm-up
    # and K timed steps, max over ranks.  At N = 1 (or under --weak) it is the
    # headline's own workload and is not re-run.
    if world > 1 and not a.weak:
        sw = a.streams
        plw = Pipeline(a, dev, sw, rank * sw, rank, R)
        plw.advance(max(0, a.warmup - 1))
        barrier()
        w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0.record(stream)
        plw.advance(a.steps)
        w1.record(stream)
        barrier()
        wms = torch.tensor([w0.elapsed_time(w1)], dtype=torch.float64, device=dev)
        dist.all_reduce(wms, op=dist.ReduceOp.MAX)
        wms = float(wms.item())
        weak_leg = {"value": sw * world * a.steps / (wms / 1e3), "unit": UNIT, "streams_per_gpu": sw,
                    "streams_total": sw * world, "steps": a.steps, "ms_per_step": wms / a.steps,
                    "scaling": "weak", "note": "same pipelined step, --streams per rank; the headline "
                                               "value is the strong (512 in total) run"}
        del plw
        torch.cuda.synchronize()
    else:
        weak_leg = {"value": value, "unit": UNIT, "streams_per_gpu": S, "streams_total": total_streams,
                    "steps": a.steps, "ms_per_step": ms / a.steps, "scaling": "weak",
                    "note": "N = 1" if world == 1 else "the headline run is itself the weak run (--weak)"}

    # ---- CPU baseline (rank 0, N == 1 only)
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        kind = cpu_kind(a)
        v, cores, nfr = cpu_run(kind, a.cpu_streams, a.cpu_steps, 1, H, P, D, a.refresh_shift)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
               "sample": cpu_sample_text(kind, a.cpu_streams, a.cpu_steps, 1, nfr)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True,
            "scaling": "weak" if a.weak else "strong",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (frozen generator, torch draw on GPU; cache/fresh bf16 N(0,1))",
            "config": {"workload": (f"config5 {'weak: ' + str(a.streams) + ' streams per GPU' if a.weak else 'as written: ' + str(total_streams) + ' streams in total, ' + str(S) + ' per GPU'}"
                                    ": select + splice, adaptive budget, refresh on shift>1"),
                       "graph": not a.no_graph, "pipeline": not a.no_pipeline,
                       "graph_steps": pl.G if not a.no_graph else 0,
                       "splice_boost_ctas": pl.boost,
                       "streams_per_gpu": S, "streams_total": total_streams, "size": H, "channels": 3, "patch": P, "tokens": N,
                       "hidden": D, "hidden_dtype": "bf16", "frame_ring_steps": R,
                       "l2": f"inputs > L2 ({S * H * H * 12 / 1e9:.2f} GB of frames per step, "
                             f"{R * S * H * H * 12 / 1e9:.1f} GB ring)"},
            "tokens_per_s": value * N,
            "roofline": roofline, "roofline_step": roofline_step, "kernels": kernels,
            "splice_alone_wide": splice_wide,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "h2d_gbs": e2e_h2d_gbs, "pcie_copy_gbs": pcie_gbs, "link_frac": e2e_h2d_gbs / pcie_gbs,
                    "steps": ke, "path": "pinned host frames -> (copy stream, double-buffered) fc_select -> "
                                         "fc_splice_inplace -> results + splice map to pinned host"},
            "e2e_u8": {"value": e2e8_val, "unit": UNIT, "h2d_bytes_per_step": total_streams * H * H * 3,
                       "d2h_bytes_per_step": d2h, "h2d_gbs": e2e8_h2d_gbs, "link_frac": e2e8_h2d_gbs / pcie_gbs,
                       "steps": ke, "frames": "PPM P6 uint8 payloads (reference ingest format), "
                                              "round(255 * the fp32 workload frames)"},
            "gpu_launches": gpu_launches,
            "latency": latency,
            "clocks": clocks.summary(win_main),
            "decisions": {"reuse_ratio": reuse_ratio, "flush_rate": flush_rate,
                          "frames": int(cnt["frames"]), "cold": int(cnt["cold"]),
                          "over": "every timed step of every rank (select-kernel counters)"},
            "sustained": sustained,
            "weak_scaling": weak_leg,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    a = parse()
    ws = os.environ.get("WORLD_SIZE")
    if ws is None and a.gpus > 1:
        # one process per GPU: re-run this script under torchrun with N ranks
        # (the reference arm is CPU-only and runs on rank 0 alone, so it needs
        # no ranks)
        if a.impl == "reference":
            run_reference(a)
            return
        sys.exit(subprocess.call(launch_command(sys.argv[1:], a.gpus, free_port())))
    if ws is not None and int(ws) != a.gpus:
        sys.stderr.write(f"bench.py: WORLD_SIZE={ws} but --gpus {a.gpus}; refusing the mismatch\n")
        sys.exit(2)
    if os.environ.get("FC_BENCH_PLUMBING") == "1":
        run_plumbing(a)
    elif a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
