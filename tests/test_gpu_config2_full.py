"""BASELINE config 2 at full size: 64 concurrent streams x 64 steps of
448x448x3 frames (P = 14, N = 1024, adaptive budget, refresh on shift > 1),
batched on one GPU.  Every one of the 64 x 63 decisions is checked against
the CPU oracle (oracle/parity.py: discrete outputs bit-exact outside the
1e-4 decision margins, floats within 1e-3), the oracle running in a process
pool over streams.
"""

import multiprocessing as mp
import os

import pytest

from oracle import freqcache_oracle as O
from oracle.parity import ParityReport, compare

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

S, T, H, P = 64, 64, 448, 14


def _oracle_stream(args):
    from threadpoolctl import threadpool_limits
    frames, = args  # (T, H, W, 3) float32
    oc = O.OracleConfig(patch_size=P)
    oc.refresh_shift = 1
    with threadpool_limits(1):  # one core per worker process
        return [O.decide(frames[t - 1], frames[t], oc, step=t) for t in range(1, len(frames))]


def test_config2_full_64x64(cuda):
    import torch
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200.api import decision_from_device
    from paper_2604_24391_b200.synth import torch_stream_frames
    frames = torch.empty((T, S, H, H, 3), dtype=torch.float32, device="cuda")
    for c0 in range(0, S, 16):
        frames[:, c0:c0 + 16] = torch_stream_frames(16, T, H, H, seed=2000 + c0, device="cuda")
    cfg = fc.CacheConfig(patch_size=P)
    eng = fc.FreqCacheEngine(S, H, H, P, fmt="rgb")
    dev = []  # per step: host copies of the decision outputs
    for t in range(T):
        out = eng.select(frames[t], cfg, refresh_shift=1)
        if t:
            dev.append((out.host_results(), out.reuse_idx.cpu().numpy(), out.recompute_idx.cpu().numpy(),
                        out.refresh_mask.cpu().numpy(), out.energy.cpu().numpy()))
    torch.cuda.synchronize()

    workers = max(1, min(16, len(os.sched_getaffinity(0))))
    oc = O.OracleConfig(patch_size=P)
    oc.refresh_shift = 1
    rep = ParityReport()
    n_exact = n_set = n_pairs = 0
    flushes = 0
    ctx = mp.get_context("fork")  # workers run numpy only (no CUDA)
    with ctx.Pool(workers) as pool:
        jobs = ((frames[:, s].cpu().numpy(),) for s in range(S))
        for s, ora in enumerate(pool.imap(_oracle_stream, jobs)):
            for t in range(1, T):
                res, ri, rc, rm, en = dev[t - 1]
                d = decision_from_device(res[s], ri[s], rc[s], rm[s], step=t)
                o = ora[t - 1]
                compare(d, o, oc, energies=en[s], rep=rep)
                same_refresh = tuple(d.refresh_set) == o.refresh_set
                n_exact += tuple(d.reuse_set) == o.reuse_set and same_refresh
                n_set += set(d.reuse_set) == set(o.reuse_set) and same_refresh
                flushes += int(o.flushed)
                n_pairs += max(0, len(o.reuse_set) - 1)
    assert rep.ok, rep.errors[:10]
    # every decision has the oracle's sets; the only exemptions are reuse-order
    # swaps between energies inside the tie margin, a bounded fraction of all
    # neighbouring reused pairs
    assert n_set == S * (T - 1), n_set
    assert set(rep.exemptions) <= {"order"}, rep.exemptions
    assert rep.exemptions.get("order", 0) <= 0.05 * n_pairs, (rep.exemptions, n_pairs)
    print(f"config 2 full: {n_set}/{S * (T - 1)} decisions with identical reuse and refresh sets, "
          f"{n_exact} also in identical reuse order (order differs only among energies inside the "
          f"parity margins); oracle flushes {flushes}; exemptions {rep.exemptions} of {n_pairs} neighbouring "
          f"reused pairs")
