"""Edge cases on the 448 x 448 fast path (batched engine; the generic-path
versions are in test_gpu_parity.py): constant, zero and non-finite frames in
one batch next to normal streams, the stream after a non-finite frame, and a
constant previous frame — each stream against the CPU oracle or the
reference's error behaviour."""

import numpy as np
import pytest

from oracle import freqcache_oracle as O
from oracle.parity import ParityReport, compare

pytestmark = pytest.mark.gpu

H, P = 448, 14


def test_fast_path_degenerate_and_nonfinite_streams(cuda):
    import torch
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200.api import decision_from_device
    from paper_2604_24391_b200.synth import stream_frames
    S, T = 7, 3
    fr = np.stack([stream_frames(4100, s, T, H, H) for s in range(S)], axis=1)  # T, S, H, W, 3
    fr[1, 1] = 0.5            # stream 1: constant frame at t = 1
    fr[1, 2] = 0.0            # stream 2: zero frame at t = 1
    fr[1, 3, 100, 200, 1] = np.nan   # stream 3: NaN pixel at t = 1
    fr[1, 5, 7, 9, 0] = np.inf       # stream 5: +Inf pixel at t = 1
    fr[0, 4] = 0.25           # stream 4: constant previous frame
    fr[2, 6] = fr[1, 6]       # stream 6: identical consecutive frames at t = 2
    eng = fc.FreqCacheEngine(S, H, H, P, fmt="rgb")
    cfg = fc.CacheConfig(patch_size=P)
    oc = O.OracleConfig(patch_size=P)
    rep = ParityReport()
    for t in range(T):
        out = eng.select(torch.from_numpy(np.ascontiguousarray(fr[t])).cuda(), cfg)
        res = out.host_results()
        if t == 0:
            assert (res["cold"] == 1).all()
            continue
        ri, rc, rm = out.reuse_idx.cpu().numpy(), out.recompute_idx.cpu().numpy(), out.refresh_mask.cpu().numpy()
        en = out.energy.cpu().numpy()
        for s in range(S):
            bad_now = t == 1 and s in (3, 5)
            if bad_now:
                # the reference raises ValueError("frame contains non-finite values")
                assert res["status"][s] == 4 and res["k_final"][s] == 0
                with pytest.raises(ValueError, match="non-finite"):
                    O.decide(fr[t - 1, s], fr[t, s], oc, step=t)
                continue
            if t == 2 and s in (3, 5):
                # after a non-finite frame the stream restarts cold
                assert res["cold"][s] == 1 and res["status"][s] == 0
                continue
            assert res["status"][s] == 0 and res["cold"][s] == 0
            d = decision_from_device(res[s], ri[s], rc[s], rm[s], step=t)
            o = O.decide(fr[t - 1, s], fr[t, s], oc, step=t)
            compare(d, o, oc, energies=en[s], rep=rep)
            if (t, s) == (1, 1) or (t, s) == (2, 1):
                assert d.flushed and d.diagnostic == "no texture; displacement undefined"
            if (t, s) == (1, 2) or (t, s) == (2, 2):
                assert d.flushed and d.diagnostic == "degenerate spectrum"
            if (t, s) == (1, 4):
                assert d.flushed and d.diagnostic == "no texture; displacement undefined"
            if (t, s) == (2, 6):
                assert d.displacement.di == 0 and d.displacement.dj == 0 and d.sim_freq == pytest.approx(1.0)
    assert rep.ok, rep.errors
