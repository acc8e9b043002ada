"""GPU tests: the comparison baselines (reference compare.py, §8f #3).

fc_compare_cosines / fc_row_cosines against the oracle restatement and
against the reference-recorded fixtures (tests/golden/golden_compare.json);
compare_domains reports against the reference's own reports.  Cosines are
computed in fp64 on the GPU: agreement within 1e-9 absolute; policy sets
(cosine > tau) bit-exact wherever a cosine is more than 1e-9 from tau.
"""

import json
import math
import sys
import zlib
from pathlib import Path

import numpy as np
import pytest

from oracle import freqcache_oracle as O

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(GOLD))
from cases import compare_cases, fhash  # noqa: E402

ATOL = 1e-9


def _cfg(c):
    import paper_2604_24391_b200 as fc
    return fc.CacheConfig(tau_mig=c.get("tau_mig", 0.12), edge_lambda=c.get("edge_lambda", 0.25),
                          budget=fc.BudgetConfig(c.get("alpha_min", 0.08), c.get("alpha_max", 0.5)),
                          patch_size=c["patch_size"])


def _dev(frames, dtype):
    import torch
    return torch.from_numpy(np.ascontiguousarray(np.stack(frames))).to("cuda", dtype)


@pytest.mark.parametrize("shape,p,fmt", [((64, 64), 8, "gray64"), ((112, 112), 14, "gray64"),
                                         ((96, 64), 16, "gray32"), ((64, 96), 32, "gray64"),
                                         ((448, 448), 14, "rgb"), ((224, 224), 14, "rgb"),
                                         ((30, 45), 3, "gray64")])
def test_compare_cosines_vs_oracle(cuda, shape, p, fmt):
    import torch
    from paper_2604_24391_b200.engine import compare_cosines
    rng = np.random.default_rng(zlib.crc32(repr((shape, p, fmt)).encode()))
    B = 3
    if fmt == "rgb":
        prev = [rng.random(shape + (3,)).astype(np.float32) for _ in range(B)]
        curr = [np.roll(f, (2, -3), axis=(0, 1)) for f in prev]
        dt = torch.float32
    else:
        prev = [rng.random(shape) for _ in range(B)]
        curr = [np.roll(f, (1, 5), axis=(0, 1)) + 0.05 * rng.standard_normal(shape) for f in prev]
        if fmt == "gray32":
            prev = [f.astype(np.float32) for f in prev]
            curr = [f.astype(np.float32) for f in curr]
        dt = torch.float32 if fmt == "gray32" else torch.float64
    vis, nf = compare_cosines(_dev(prev, dt), _dev(curr, dt), p)
    vis, nf = vis.cpu().numpy(), nf.cpu().numpy()
    for b in range(B):
        ov, on = O.compare_cosines(prev[b], curr[b], p)
        np.testing.assert_allclose(vis[b], ov, rtol=0, atol=ATOL)
        np.testing.assert_allclose(nf[b], on, rtol=0, atol=ATOL)


def test_compare_cosines_golden_pair(cuda):
    """BASELINE geometry (448^2 RGB, P = 14) against the reference's values."""
    import torch
    from paper_2604_24391_b200.engine import compare_cosines
    from paper_2604_24391_b200.synth import stream_frames
    pair = json.loads((GOLD / "golden_compare.json").read_text())["pair"]
    r = pair["recipe"]
    fr = stream_frames(r["seed"], 0, 2, r["size"], r["size"])
    assert [fhash(f) for f in fr] == pair["frames"]
    vis, nf = compare_cosines(_dev([fr[0]], torch.float32), _dev([fr[1]], torch.float32), r["patch"])
    np.testing.assert_allclose(vis[0].cpu().numpy(), pair["visual"], rtol=0, atol=ATOL)
    np.testing.assert_allclose(nf[0].cpu().numpy(), pair["naive_freq"], rtol=0, atol=ATOL)


def test_compare_cosines_zero_norm_and_identity(cuda):
    import torch
    from paper_2604_24391_b200.engine import compare_cosines
    f = np.random.default_rng(5).random((32, 32))
    z = np.zeros((32, 32))
    z[:8, :8] = f[:8, :8]  # patch 0 equal, the rest zero
    vis, nf = compare_cosines(_dev([f, z], torch.float64), _dev([f, z * 3.0], torch.float64), 8)
    vis, nf = vis.cpu().numpy(), nf.cpu().numpy()
    np.testing.assert_allclose(vis[0], 1.0, atol=1e-12)
    np.testing.assert_allclose(nf[0], 1.0, atol=1e-12)
    assert vis[1][0] == pytest.approx(1.0, abs=1e-12) and nf[1][0] == pytest.approx(1.0, abs=1e-12)
    assert (vis[1][1:] == 0.0).all() and (nf[1][1:] == 0.0).all()


def test_compare_cosines_errors(cuda):
    import torch
    from paper_2604_24391_b200 import _native as nat
    from paper_2604_24391_b200.engine import compare_cosines
    a = torch.zeros((1, 66, 66), dtype=torch.float64, device="cuda")
    with pytest.raises(nat.NativeError):
        compare_cosines(a, a, 33)  # P > 32
    with pytest.raises(ValueError):
        compare_cosines(a, a, 4)   # does not tile
    with pytest.raises(ValueError):
        compare_cosines(a, a[:, :64, :64].contiguous(), 2)


def test_row_cosines(cuda):
    import torch
    from paper_2604_24391_b200.engine import row_cosines
    rng = np.random.default_rng(6)
    a, b = rng.standard_normal((300, 37)), rng.standard_normal((300, 37))
    a[3] = 0.0
    out = row_cosines(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
    np.testing.assert_allclose(out, O.position_cosines(a, b), rtol=0, atol=1e-12)
    assert out[3] == 0.0


def test_compare_domains_matches_reference_reports(cuda):
    from paper_2604_24391_b200.compare import compare_domains
    gold = {c["name"]: c for c in json.loads((GOLD / "golden_compare.json").read_text())["cases"]}
    for name, frames, c, labels in compare_cases():
        g = gold[name]["report"]
        rep = compare_domains(frames, _cfg(c), edge_labels=labels)
        assert rep["n_steps"] == g["n_steps"] and rep["n_tokens"] == g["n_tokens"]
        assert rep["thresholds"] == g["thresholds"]
        assert math.isclose(rep["baseline_latency_ms"], g["baseline_latency_ms"], rel_tol=1e-12)
        for pol, gp in g["policies"].items():
            rp = rep["policies"][pol]
            assert rp["reuse_ratio"] == gp["reuse_ratio"], (name, pol)
            assert rp["edge_false_reuse"] == gp["edge_false_reuse"], (name, pol)
            assert math.isclose(rp["mean_latency_ms"], gp["mean_latency_ms"], rel_tol=1e-12), (name, pol)
            assert math.isclose(rp["speedup"], gp["speedup"], rel_tol=1e-12), (name, pol)


def test_compare_domains_reference_properties(cuda):
    """The reference's own compare tests (test_compare.py:9-66), on the
    fixture scenes: frequency policy never reuses a labelled edge patch, the
    position-wise ones do; static scene caps; labels absent -> None."""
    from paper_2604_24391_b200.compare import compare_domains
    cases = {n: (f, c, lab) for n, f, c, lab in compare_cases()}
    f, c, lab = cases["edge"]
    rep = compare_domains(f, _cfg(c), edge_labels=lab)["policies"]
    assert rep["freqcache"]["edge_false_reuse"] == 0
    assert rep["visual"]["edge_false_reuse"] > 0 and rep["naive_freq"]["edge_false_reuse"] > 0
    f, c, _ = cases["static"]
    r = compare_domains(f, _cfg(c))
    n = r["n_tokens"]
    assert r["policies"]["freqcache"]["reuse_ratio"] == pytest.approx(int(0.4 * n) / n)
    assert r["policies"]["visual"]["reuse_ratio"] == 1.0 and r["policies"]["naive_freq"]["reuse_ratio"] == 1.0
    f, c, _ = cases["random"]
    r = compare_domains(f, _cfg(c))
    for stats in r["policies"].values():
        assert stats["edge_false_reuse"] is None
        assert stats["mean_latency_ms"] <= r["baseline_latency_ms"] and stats["speedup"] >= 1.0
    with pytest.raises(ValueError):
        compare_domains(f[:1], _cfg(c))


def test_compare_domains_custom_token_fn(cuda):
    """A host token_fn (the user's model) goes through fc_row_cosines."""
    from paper_2604_24391_b200 import default_token_fn
    from paper_2604_24391_b200.compare import compare_domains
    f, c = [(x[1], x[2]) for x in compare_cases() if x[0] == "translate"][0]
    rep = compare_domains(f, _cfg(c), token_fn=default_token_fn, tau_visual=0.99)
    p = c["patch_size"]
    reused = 0
    for t in range(1, len(f)):
        ta = np.stack([default_token_fn(x) for x in O.patch_pixels(f[t - 1], p).reshape(-1, p, p)])
        tb = np.stack([default_token_fn(x) for x in O.patch_pixels(f[t], p).reshape(-1, p, p)])
        reused += int((O.position_cosines(ta, tb) > 0.99).sum())
    assert rep["policies"]["visual"]["reuse_ratio"] == reused / ((len(f) - 1) * rep["n_tokens"])
