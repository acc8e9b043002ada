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


def test_fast_path_formats_agree(cuda):
    """448 x 448: the same frames as RGB fp32, as their fp64 luma and as
    fp32 gray give the decisions the oracle gives for the same gray values;
    RGB fp32 and its exact fp64 luma give bitwise-identical energies."""
    import torch
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200.api import decision_from_device
    from paper_2604_24391_b200.synth import stream_frames
    S, T = 2, 4
    rgb = np.stack([stream_frames(4200, s, T, H, H) for s in range(S)], axis=1)       # T, S, H, W, 3 fp32
    r, g, b = (rgb[..., i].astype(np.float64) for i in range(3))
    g64 = (0.299 * r + 0.587 * g) + 0.114 * b
    g32 = g64.astype(np.float32)
    cfg = fc.CacheConfig(patch_size=P)
    oc = O.OracleConfig(patch_size=P)
    outs = {}
    for name, fmt, fr in (("rgb", "rgb", rgb), ("gray64", "gray64", g64), ("gray32", "gray32", g32)):
        eng = fc.FreqCacheEngine(S, H, H, P, fmt=fmt)
        outs[name] = []
        for t in range(T):
            o = eng.select(torch.from_numpy(np.ascontiguousarray(fr[t])).cuda(), cfg)
            outs[name].append((o.host_results(), o.reuse_idx.cpu().numpy(), o.recompute_idx.cpu().numpy(),
                               o.refresh_mask.cpu().numpy(), o.energy.cpu().numpy()))
    rep = ParityReport()
    for t in range(1, T):
        assert np.array_equal(outs["rgb"][t][4], outs["gray64"][t][4])  # identical fp64 luma -> energies
        for name, ref in (("rgb", g64), ("gray64", g64), ("gray32", g32.astype(np.float64))):
            res, ri, rc, rm, en = outs[name][t]
            for s in range(S):
                d = decision_from_device(res[s], ri[s], rc[s], rm[s], step=t)
                o = O.decide(ref[t - 1, s], ref[t, s], oc, step=t)
                compare(d, o, oc, energies=en[s], rep=rep)
    assert rep.ok, rep.errors


@pytest.mark.parametrize("h,w,p", [(1008, 1008, 16), (1344, 448, 28), (448, 224, 14), (1536, 1536, 24)])
def test_generic_path_envelope(cuda, h, w, p):
    """Near the generic kernels' envelope (N <= 4096, P <= 32, the row pass's
    shared memory ~ 12 P W bytes <= 227 KB): 1008^2 / P 16 (N = 3969), a tall
    1344 x 448 / P 28 frame and a rectangular 448 x 224 frame, two streams
    against the oracle; 1536^2 / P 24 is outside (shared memory) and refused
    at plan creation."""
    import torch
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200._native import NativeError
    from paper_2604_24391_b200.api import decision_from_device
    if (h, w, p) == (1536, 1536, 24):
        with pytest.raises(NativeError, match="envelope"):
            fc.FreqCacheEngine(1, h, w, p, fmt="gray64")
        return
    rng = np.random.default_rng(h + w + p)
    base = rng.random((h, w))
    fr = np.stack([np.stack([np.roll(base, (3 * t + s, 2 * t), axis=(0, 1)) for s in range(2)]) for t in range(3)])
    eng = fc.FreqCacheEngine(2, h, w, p, fmt="gray64")
    cfg = fc.CacheConfig(patch_size=p)
    oc = O.OracleConfig(patch_size=p)
    rep = ParityReport()
    for t in range(3):
        out = eng.select(torch.from_numpy(np.ascontiguousarray(fr[t])).cuda(), cfg)
        if t == 0:
            continue
        res = out.host_results()
        ri, rc, rm = out.reuse_idx.cpu().numpy(), out.recompute_idx.cpu().numpy(), out.refresh_mask.cpu().numpy()
        en = out.energy.cpu().numpy()
        for s in range(2):
            d = decision_from_device(res[s], ri[s], rc[s], rm[s], step=t)
            o = O.decide(fr[t - 1, s], fr[t, s], oc, step=t)
            compare(d, o, oc, energies=en[s], rep=rep)
    assert rep.ok, rep.errors


def test_fast_path_refuses_misaligned_frames(cuda):
    # K_A stages frames with bulk copies: a frames pointer off 16 bytes is
    # refused up front (FC_EINVAL -> ValueError) instead of faulting
    import torch
    import paper_2604_24391_b200 as fc
    eng = fc.FreqCacheEngine(2, H, H, P, fmt="rgb")
    n = 2 * H * H * 3
    buf = torch.zeros(n + 1, dtype=torch.float32, device="cuda")
    frames = buf[1:].view(2, H, H, 3)
    assert frames.is_contiguous() and frames.data_ptr() % 16 == 4
    with pytest.raises(ValueError):
        eng.select(frames, fc.CacheConfig(patch_size=P))
    out = eng.select(buf[:n].view(2, H, H, 3), fc.CacheConfig(patch_size=P))   # aligned: fine
    torch.cuda.synchronize()
    assert (out.host_results()["cold"] == 1).all()


@pytest.mark.parametrize("kw,shift", [
    ({"budget": (0.0, 0.0)}, 1),            # K_reuse = 0: nothing reused
    ({"budget": (1.0, 1.0)}, 1),            # K_reuse = N: every candidate reused
    ({"tau_mig": 0.0}, -1),                 # gate never closes on similarity; shift rule off
    ({"tau_mig": 1.0}, 0),                  # gate closes unless the frames are identical
    ({"edge_lambda": -5.0}, 1),             # (almost) every token refreshed
    ({"edge_lambda": 1e12}, 1),             # no token refreshed
])
def test_fast_path_config_extremes(cuda, kw, shift):
    """The 448 x 448 fast path at the configuration extremes (budget 0 / 1,
    the migration threshold at 0 / 1, refresh thresholds below / above every
    energy, the config-2 shift rule off / at 0): each stream's decision
    against the CPU oracle."""
    import torch
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200.api import decision_from_device
    from paper_2604_24391_b200.synth import stream_frames
    S, T = 4, 3
    fr = np.stack([stream_frames(4200, s, T, H, H) for s in range(S)], axis=1)
    fr[2, 3] = fr[1, 3]                      # one identical consecutive pair
    b = kw.get("budget", (0.08, 0.5))
    cfg = fc.CacheConfig(patch_size=P, tau_mig=kw.get("tau_mig", 0.12), edge_lambda=kw.get("edge_lambda", 0.25),
                         budget=fc.BudgetConfig(*b))
    oc = O.OracleConfig(patch_size=P, tau_mig=cfg.tau_mig, edge_lambda=cfg.edge_lambda, alpha_min=b[0],
                        alpha_max=b[1], refresh_shift=None if shift < 0 else shift)
    eng = fc.FreqCacheEngine(S, H, H, P, fmt="rgb")
    rep = ParityReport()
    for t in range(T):
        out = eng.select(torch.from_numpy(np.ascontiguousarray(fr[t])).cuda(), cfg, refresh_shift=shift)
        if t == 0:
            continue
        res = out.host_results()
        ri, rc, rm = out.reuse_idx.cpu().numpy(), out.recompute_idx.cpu().numpy(), out.refresh_mask.cpu().numpy()
        en = out.energy.cpu().numpy()
        for s in range(S):
            d = decision_from_device(res[s], ri[s], rc[s], rm[s], step=t)
            compare(d, O.decide(fr[t - 1, s], fr[t, s], oc, step=t), oc, energies=en[s], rep=rep)
            if b == (0.0, 0.0):
                assert len(d.reuse_set) == 0
    assert rep.ok, rep.errors
