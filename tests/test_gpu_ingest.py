"""GPU tests: frame ingest in the compact on-disk layouts (§8f #4).

8-bit P5 / P6 payloads and rawf32 go to the device as they are stored and
the decision kernels form the gray value themselves (FC_FMT_GRAY_U8 /
FC_FMT_RGB_U8 / FC_FMT_GRAY_F32).  Parity target: the oracle on the frames the
reference's own reader produces (frameio.read_netpbm: v / 255, luma / 255 in
fp64), decisions bit-exact outside the 1e-4 margins (oracle/parity.py).
"""

import numpy as np
import pytest

from oracle import freqcache_oracle as O
from oracle.parity import ParityReport, compare

pytestmark = pytest.mark.gpu


def _cfg(p, **kw):
    import paper_2604_24391_b200 as fc
    c = fc.CacheConfig(patch_size=p, **kw)
    oc = O.OracleConfig(tau_mig=c.tau_mig, edge_lambda=c.edge_lambda, alpha_min=c.budget.alpha_min,
                        alpha_max=c.budget.alpha_max, patch_size=p)
    return c, oc


def _ref_gray(px):
    """frameio.py:81-88 on uint8 pixels."""
    p = px.astype(np.float64)
    if p.ndim == 2:
        return p / 255.0
    return (0.299 * p[..., 0] + 0.587 * p[..., 1] + 0.114 * p[..., 2]) / 255.0


def _u8_sequence(seed, steps, h, w, rgb):
    """Quantised synthetic stream (the config generator, then * 255)."""
    from paper_2604_24391_b200.synth import stream_frames
    fr = stream_frames(seed, 0, steps, h, w)
    u8 = np.round(np.clip(fr, 0.0, 1.0) * 255.0).astype(np.uint8)
    if not rgb:
        u8 = u8[..., 1].copy()
    return u8


@pytest.mark.parametrize("size,p,rgb,shift", [(448, 14, True, 1), (448, 14, False, None),
                                              (224, 14, True, None), (64, 8, False, None)])
def test_u8_select_matches_reader_then_oracle(cuda, size, p, rgb, shift):
    import torch
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200.api import decision_from_device
    S, T = 2, 6
    seqs = [_u8_sequence(300 + s, T, size, size, rgb) for s in range(S)]
    frames = np.stack(seqs, axis=1)  # T, S, ...
    c, oc = _cfg(p)
    oc.refresh_shift = shift
    eng = fc.FreqCacheEngine(S, size, size, p, fmt="rgb_u8" if rgb else "gray_u8")
    rep = ParityReport()
    for t in range(T):
        out = eng.select(torch.from_numpy(np.ascontiguousarray(frames[t])).cuda(), c, refresh_shift=shift)
        if t == 0:
            continue
        res = out.host_results()
        en = out.energy.cpu().numpy()
        ri, rc, rm = out.reuse_idx.cpu().numpy(), out.recompute_idx.cpu().numpy(), out.refresh_mask.cpu().numpy()
        for s in range(S):
            d = decision_from_device(res[s], ri[s], rc[s], rm[s], step=t)
            o = O.decide(_ref_gray(frames[t - 1, s]), _ref_gray(frames[t, s]), oc, step=t)
            compare(d, o, oc, energies=en[s], rep=rep)
    assert rep.ok, rep.errors


def test_u8_energy_bitwise_vs_gray64(cuda):
    """The in-kernel u8 -> gray conversion equals the reader's float64 frame
    exactly: energies from the u8 layout and from the float64 gray frame of
    the same pixels are identical."""
    import torch
    import paper_2604_24391_b200 as fc
    u8 = _u8_sequence(77, 1, 448, 448, True)
    g = np.ascontiguousarray(_ref_gray(u8[0])[None])
    e8 = fc.FreqCacheEngine(1, 448, 448, 14, fmt="rgb_u8").patch_energy(torch.from_numpy(u8[:1].copy()).cuda())
    e64 = fc.FreqCacheEngine(1, 448, 448, 14, fmt="gray64").patch_energy(torch.from_numpy(g).cuda())
    assert torch.equal(e8, e64)


def test_u8_compare_cosines(cuda):
    import torch
    from paper_2604_24391_b200.engine import compare_cosines
    u8 = _u8_sequence(5, 2, 112, 112, True)
    vis, nf = compare_cosines(torch.from_numpy(u8[:1].copy()).cuda(), torch.from_numpy(u8[1:].copy()).cuda(), 14)
    ov, on = O.compare_cosines(_ref_gray(u8[0]), _ref_gray(u8[1]), 14)
    np.testing.assert_allclose(vis[0].cpu().numpy(), ov, rtol=0, atol=1e-9)
    np.testing.assert_allclose(nf[0].cpu().numpy(), on, rtol=0, atol=1e-9)


def test_load_frames_device(cuda, tmp_path):
    import torch
    from paper_2604_24391_b200 import frameio
    from paper_2604_24391_b200.types import FrameParseError
    rng = np.random.default_rng(3)
    d = tmp_path / "ppm"
    d.mkdir()
    imgs = [rng.integers(0, 256, (28, 42, 3), dtype=np.uint8) for _ in range(3)]
    for i, im in enumerate(imgs):
        (d / f"{i}.ppm").write_bytes(b"P6\n42 28\n255\n" + im.tobytes())
    t, fmt = frameio.load_frames_device(d)
    assert fmt == "rgb_u8" and t.is_cuda and t.dtype == torch.uint8
    assert np.array_equal(t.cpu().numpy(), np.stack(imgs))
    (d / "9.pgm").write_bytes(b"P5\n42 28\n255\n" + bytes(42 * 28))
    with pytest.raises(ValueError, match="mixes"):
        frameio.load_frames_device(d)
    fr = [rng.random((14, 28)) for _ in range(2)]
    frameio.save_rawf32(tmp_path / "s.raw", fr)
    t, fmt = frameio.load_frames_device(tmp_path / "s.raw")
    assert fmt == "gray32" and np.array_equal(t.cpu().numpy(), np.stack(fr).astype(np.float32))
    bad = np.stack(fr).astype("<f4")
    bad[1, 0, 0] = np.nan
    (tmp_path / "b.raw").write_bytes(b"FQC1" + np.array([14, 28, 2], "<u4").tobytes() + bad.tobytes())
    with pytest.raises(FrameParseError, match="frame 1"):
        frameio.load_frames_device(tmp_path / "b.raw")
    # the device frames drive the engine directly
    import paper_2604_24391_b200 as fc
    t, fmt = frameio.load_frames_device(d.parent / "s.raw")
    eng = fc.FreqCacheEngine(1, 14, 28, 14, fmt=fmt)
    eng.select(t[0:1].contiguous(), fc.CacheConfig(patch_size=14))
