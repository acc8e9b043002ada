"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Discrete outputs bit-exact outside the 1e-4 decision margins, floats within
1e-3 relative (oracle/parity.py); bf16 splice bit-exact.
"""

import numpy as np
import pytest

from oracle import freqcache_oracle as O
from oracle.parity import ParityReport, compare

pytestmark = pytest.mark.gpu


def _cfg(**kw):
    import paper_2604_24391_b200 as fc
    budget = kw.pop("budget", None)
    c = fc.CacheConfig(**kw) if budget is None else fc.CacheConfig(budget=fc.BudgetConfig(*budget), **kw)
    oc = O.OracleConfig(tau_mig=c.tau_mig, edge_lambda=c.edge_lambda, alpha_min=c.budget.alpha_min,
                        alpha_max=c.budget.alpha_max, patch_size=c.patch_size)
    return c, oc


def _check(dev, ora, oc, rep=None):
    rep = compare(dev, ora, oc, rep=rep)
    assert rep.ok, rep.errors
    return rep


def test_identical_frames(cuda):
    import paper_2604_24391_b200 as fc
    c, oc = _cfg(patch_size=8)
    f = np.random.default_rng(0).random((32, 32))
    d = fc.decide(f, f, c)
    assert not d.flushed and (d.displacement.di, d.displacement.dj) == (0, 0)
    _check(d, O.decide(f, f, oc), oc)


@pytest.mark.parametrize("shape,p", [((16, 16), 4), ((32, 32), 8), ((48, 48), 8), ((64, 64), 8),
                                     ((64, 64), 16), ((96, 96), 8), ((112, 112), 8), ((224, 224), 16),
                                     ((224, 224), 14), ((448, 448), 14), ((64, 96), 8), ((56, 84), 14)])
def test_random_shift_pairs(cuda, shape, p):
    import paper_2604_24391_b200 as fc
    c, oc = _cfg(patch_size=p)
    rng = np.random.default_rng(shape[0] * 31 + p)
    rep = ParityReport()
    for _ in range(6):
        prev = rng.random(shape)
        sh = (int(rng.integers(-shape[0] // 3, shape[0] // 3 + 1)), int(rng.integers(-shape[1] // 3, shape[1] // 3 + 1)))
        curr = np.roll(prev, sh, axis=(0, 1))
        d = fc.decide(prev, curr, c)
        o = O.decide(prev, curr, oc)
        _check(d, o, oc, rep)
        assert (d.displacement.di, d.displacement.dj) == sh


def test_reference_buckets(cuda):
    """The reference's decide/decide_reference buckets, 1,000 instances as in its
    acceptance criterion 6 (test_acceptance.py:156-204)."""
    import paper_2604_24391_b200 as fc
    rng = np.random.default_rng(600)
    cfgs = {
        "base": _cfg(patch_size=8), "flush": _cfg(patch_size=8, tau_mig=1.0),
        "empty": _cfg(patch_size=8, edge_lambda=-5.0),
        "capped": _cfg(patch_size=8, budget=(0.1, 0.2)),
    }
    rep = ParityReport()
    seen = {"flush": 0, "empty": 0, "capped": 0}
    for i in range(1000):
        bucket = i % 5
        prev = rng.random((32, 32))
        if bucket == 0:
            curr = np.roll(prev, (int(rng.integers(-16, 17)), int(rng.integers(-16, 17))), axis=(0, 1))
            c, oc = cfgs["base"]
        elif bucket == 1:
            curr = rng.random((32, 32))
            c, oc = cfgs["flush"]
        elif bucket == 2:
            curr = np.roll(prev, (int(rng.integers(-8, 9)), 0), axis=(0, 1))
            c, oc = cfgs["empty"]
        elif bucket == 3:
            curr = np.roll(prev, (0, int(rng.integers(-8, 9))), axis=(0, 1))
            c, oc = cfgs["capped"]
        else:
            curr = rng.random((32, 32))
            dup = np.full((8, 8), 0.5)
            dup[0, 0] = 0.52
            blocks = curr.reshape(4, 8, 4, 8).swapaxes(1, 2)
            for bi, bj in ((0, 1), (1, 2), (2, 0), (3, 3)):
                blocks[bi, bj] = dup
            sh = (int(rng.integers(-4, 5)), int(rng.integers(-4, 5)))
            prev = np.roll(curr, (-sh[0], -sh[1]), axis=(0, 1))
            c, oc = cfgs["capped"] if i % 2 else cfgs["base"]
        d = fc.decide(prev, curr, c, step=i)
        o = O.decide(prev, curr, oc, step=i)
        _check(d, o, oc, rep)
        assert d.step == i
        seen["flush"] += d.flushed
        seen["empty"] += d.k_candidate == 0 and not d.flushed
        seen["capped"] += 0 < d.k_final == d.k_reuse < d.k_candidate
    assert seen["flush"] >= 200 and seen["empty"] >= 200 and seen["capped"] >= 150


def test_tied_energies_order(cuda):
    import paper_2604_24391_b200 as fc
    c, oc = _cfg(patch_size=8)
    tile = np.random.default_rng(17).random((8, 8))
    frame = np.tile(tile, (2, 2))
    d = fc.decide(frame, frame, c)
    o = O.decide(frame, frame, oc)
    _check(d, o, oc)


def test_degenerate_frames(cuda):
    import paper_2604_24391_b200 as fc
    c, oc = _cfg(patch_size=8)
    f = np.random.default_rng(8).random((32, 32))
    d = fc.decide(np.zeros((32, 32)), f, c)
    assert d.flushed and d.diagnostic == "degenerate spectrum"
    _check(d, O.decide(np.zeros((32, 32)), f, oc), oc)
    d2 = fc.decide(np.full((32, 32), 0.5), f, c)
    assert d2.flushed and d2.diagnostic == "no texture; displacement undefined"
    _check(d2, O.decide(np.full((32, 32), 0.5), f, oc), oc)
    d3 = fc.decide(f, np.zeros((32, 32)), c)
    o3 = O.decide(f, np.zeros((32, 32)), oc)
    assert d3.diagnostic == o3.diagnostic == "degenerate spectrum"
    assert d3.entropy.bin_count == 32 * 32 and d3.k_reuse == 0 and d3.alpha_t == 0.0
    _check(d3, o3, oc)


def test_errors(cuda):
    import paper_2604_24391_b200 as fc
    c, _ = _cfg(patch_size=8)
    f = np.random.default_rng(1).random((32, 32))
    bad = f.copy()
    bad[3, 4] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        fc.decide(f, bad, c)
    with pytest.raises(ValueError, match="non-finite"):
        fc.decide(bad, f, c)
    with pytest.raises(ValueError):
        fc.decide(np.ones((32, 32)), np.ones((16, 16)), c)
    with pytest.raises(ValueError):
        fc.decide(np.ones((30, 30)), np.ones((30, 30)), c)


def test_determinism(cuda):
    import paper_2604_24391_b200 as fc
    c, _ = _cfg(patch_size=14)
    rng = np.random.default_rng(9)
    a, b = rng.random((224, 224)), rng.random((224, 224))
    assert fc.decide(a, b, c) == fc.decide(a, b, c)
    assert fc.decide(a, b, c, parallel=True) == fc.decide(a, b, c)


def test_config1_rgb_sequence(cuda):
    """BASELINE config 1: 224x224x3 fp32, P=14, fixed 50% budget, 32 frames."""
    import torch
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200.synth import stream_frames
    frames = stream_frames(1000, 0, 32, 224, 224)
    c, oc = _cfg(patch_size=14, budget=(0.5, 0.5))
    eng = fc.FreqCacheEngine(1, 224, 224, 14, fmt="rgb")
    rep = ParityReport()
    from paper_2604_24391_b200.api import decision_from_device, _fetch
    for t in range(32):
        out = eng.select(torch.from_numpy(frames[t:t + 1]).cuda(), c)
        res, ri, rc, rm = _fetch(out)
        if t == 0:
            assert res["cold"] == 1
            continue
        d = decision_from_device(res, ri, rc, rm, step=t)
        o = O.decide(frames[t - 1], frames[t], oc, step=t)
        compare(d, o, oc, energies=out.energy[0].cpu().numpy(), rep=rep)
        assert d.k_reuse == 128 or d.flushed
    assert rep.ok, rep.errors


def test_config2_batched_streams(cuda):
    """BASELINE config 2 shape: 448x448x3, P=14, adaptive budget, shift>1 flush."""
    import torch
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200.api import decision_from_device
    from paper_2604_24391_b200.synth import stream_frames
    S, T = 3, 14
    frames = np.stack([stream_frames(2000, s, T, 448, 448) for s in range(S)], axis=1)  # T,S,H,W,3
    c, oc = _cfg(patch_size=14)
    oc.refresh_shift = 1
    eng = fc.FreqCacheEngine(S, 448, 448, 14, fmt="rgb")
    rep = ParityReport()
    for t in range(T):
        out = eng.select(torch.from_numpy(np.ascontiguousarray(frames[t])).cuda(), c, refresh_shift=1)
        if t == 0:
            continue
        res = out.host_results()
        en = out.energy.cpu().numpy()
        ri, rc, rm = out.reuse_idx.cpu().numpy(), out.recompute_idx.cpu().numpy(), out.refresh_mask.cpu().numpy()
        for s in range(S):
            d = decision_from_device(res[s], ri[s], rc[s], rm[s], step=t)
            o = O.decide(frames[t - 1, s], frames[t, s], oc, step=t)
            compare(d, o, oc, energies=en[s], rep=rep)
    assert rep.ok, rep.errors


def test_splice_bf16_bit_exact(cuda):
    import torch
    import paper_2604_24391_b200 as fc
    B, N, D = 4, 64, 1152
    g = torch.Generator(device="cuda").manual_seed(3000)
    cache = torch.randn((B, N, D), generator=g, device="cuda").to(torch.bfloat16)
    fresh = torch.randn((B, N, D), generator=g, device="cuda").to(torch.bfloat16)
    ages = torch.randint(0, 5, (B, N), device="cuda", dtype=torch.int64)
    rng = np.random.default_rng(5)
    rows = cols = 8
    src_host = np.empty((B, N), dtype=np.int32)
    decs = []
    for b in range(B):
        dip, djp = int(rng.integers(-2, 3)), int(rng.integers(-2, 3))
        al = [q for q in range(N) if 0 <= q // cols - dip < rows and 0 <= q % cols - djp < cols]
        reuse = tuple(int(v) for v in rng.permutation(al)[: len(al) // 2])
        d = O.OracleDecision(step=1, flushed=False, sim_freq=1.0, displacement=(0, 0, dip, djp),
                             entropy=(0, 0, 0), alpha_t=0.5, k_reuse=len(reuse), k_candidate=len(reuse),
                             k_final=len(reuse), reuse_set=reuse,
                             recompute_set=tuple(q for q in range(N) if q not in reuse),
                             rows=rows, cols=cols, refresh_set=())
        decs.append(d)
        m = fc.splice_map(rows, cols, torch.tensor(reuse, dtype=torch.int32, device="cuda"), dip, djp)
        src_host[b] = m.cpu().numpy()
    src = torch.from_numpy(src_host).cuda()
    for compact in (False, True):
        out = torch.empty_like(cache)
        oages = torch.empty_like(ages)
        if compact:
            fr = torch.zeros_like(fresh)
            for b in range(B):
                rec = list(decs[b].recompute_set)
                fr[b, : len(rec)] = fresh[b, rec]
        else:
            fr = fresh
        fc.splice(src, cache, ages, fr, out, oages, compact=compact)
        for b in range(B):
            rec = list(decs[b].recompute_set)
            exp, exp_age = O.splice(cache[b].view(torch.int16).cpu().numpy(), ages[b].cpu().numpy(), decs[b],
                                    fresh[b, rec].view(torch.int16).cpu().numpy())
            assert np.array_equal(out[b].view(torch.int16).cpu().numpy(), exp)
            assert np.array_equal(oages[b].cpu().numpy(), exp_age)


def test_run_sequence_matches_oracle(cuda):
    import paper_2604_24391_b200 as fc
    rng = np.random.default_rng(24)
    frames = [rng.random((64, 64)) for _ in range(8)]
    c, oc = _cfg(patch_size=8)
    rep = fc.run_sequence(frames, c)
    assert rep.flush_count == 0
    # regression anchor of the reference (test_fusion.py:237-245)
    assert rep.mean_reuse_ratio == pytest.approx(0.3392857142857143, abs=1e-12)
    pr = ParityReport()
    for t, d in enumerate(rep.decisions, start=1):
        compare(d, O.decide(frames[t - 1], frames[t], oc, step=t), oc, rep=pr)
    assert pr.ok, pr.errors


def test_step_displacement_mapped_sourcing(cuda):
    import paper_2604_24391_b200 as fc
    rng = np.random.default_rng(20)
    prev = rng.random((32, 32))
    curr = np.roll(prev, (8, 0), axis=(0, 1))
    cache = fc.populate_cache(prev, 8, fc.default_token_fn)
    cache.tokens += rng.random(cache.tokens.shape)
    d = fc.decide(prev, curr, fc.CacheConfig(patch_size=8, budget=fc.BudgetConfig(1.0, 1.0), edge_lambda=1e12))
    assert d.displacement.di_patches == 1
    new, rep = fc.step(cache, d, curr, fc.default_token_fn)
    assert np.array_equal(new.tokens[2, 3], cache.tokens[1, 3])
    assert new.ages[2, 3] == cache.ages[1, 3] + 1
    assert rep.n_reused == d.k_final


def test_phase_correlation_and_energy(cuda):
    import paper_2604_24391_b200 as fc
    rng = np.random.default_rng(6)
    f = rng.random((64, 64))
    assert (lambda d: (d.di, d.dj))(fc.phase_correlation(f, np.roll(f, (3, 5), axis=(0, 1)))) == (3, 5)
    assert (lambda d: (d.di, d.dj))(fc.phase_correlation(f, np.roll(f, (61, 0), axis=(0, 1)))) == (-3, 0)
    d = fc.phase_correlation(f, np.roll(f, (12, -4), axis=(0, 1)), patch_size=8)
    assert (d.di_patches, d.dj_patches) == (1, 0)
    with pytest.raises(fc.ConstantFrameError):
        fc.phase_correlation(np.full((8, 8), 0.5), rng.random((8, 8)))
    frame = rng.random((64, 64))
    e = fc.patch_energy(fc.PatchGrid(frame, 8)).energies
    np.testing.assert_allclose(e, O.block_energy(frame, 8), rtol=1e-10, atol=1e-14)


def test_config2_sweep_16_streams(cuda):
    """Wider parity sweep on the fast path: 16 config-2 streams x 13 steps
    (one scene cut), batched, refresh rule on; every decision checked."""
    import torch
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200.api import decision_from_device
    from paper_2604_24391_b200.synth import stream_frames
    S, T = 16, 14
    frames = np.stack([stream_frames(2500, s, T, 448, 448) for s in range(S)], axis=1)
    c, oc = _cfg(patch_size=14)
    oc.refresh_shift = 1
    eng = fc.FreqCacheEngine(S, 448, 448, 14, fmt="rgb")
    rep = ParityReport()
    n_exact = n_pairs = 0
    for t in range(T):
        out = eng.select(torch.from_numpy(np.ascontiguousarray(frames[t])).cuda(), c, refresh_shift=1)
        if t == 0:
            continue
        res = out.host_results()
        en = out.energy.cpu().numpy()
        ri, rc, rm = out.reuse_idx.cpu().numpy(), out.recompute_idx.cpu().numpy(), out.refresh_mask.cpu().numpy()
        for s in range(S):
            d = decision_from_device(res[s], ri[s], rc[s], rm[s], step=t)
            o = O.decide(frames[t - 1, s], frames[t, s], oc, step=t)
            compare(d, o, oc, energies=en[s], rep=rep)
            n_exact += tuple(d.reuse_set) == o.reuse_set and tuple(d.refresh_set) == o.refresh_set
            n_pairs += max(0, len(o.reuse_set) - 1)
    assert rep.ok, rep.errors
    # bounded exemptions: only reuse-order swaps between tie-margin energies,
    # a small fraction of all neighbouring reused pairs
    assert set(rep.exemptions) <= {"order"}, rep.exemptions
    assert rep.exemptions.get("order", 0) <= 0.05 * n_pairs, (rep.exemptions, n_pairs)
    print(f"config-2 sweep: {n_exact}/{S * (T - 1)} decisions identical to the oracle; exemptions {rep.exemptions} "
          f"of {n_pairs} neighbouring reused pairs")


def test_acceptance_shift_recovery_and_latency(cuda):
    """The reference's acceptance criteria 3 and 9 through the façade: exact
    recovery of 100/100 random cyclic shifts, and decide() median under
    10 ms at 224x224 / P16."""
    import time
    import paper_2604_24391_b200 as fc
    c, _ = _cfg(patch_size=16)
    rng = np.random.default_rng(909)
    ok = 0
    for _ in range(100):
        prev = rng.random((64, 64))
        sh = (int(rng.integers(-31, 32)), int(rng.integers(-31, 32)))
        d = fc.decide(prev, np.roll(prev, sh, axis=(0, 1)), c)
        ok += (d.displacement.di, d.displacement.dj) == sh
    assert ok == 100
    a, b = rng.random((224, 224)), rng.random((224, 224))
    fc.decide(a, b, c)
    times = []
    for _ in range(21):
        t0 = time.perf_counter()
        fc.decide(a, b, c)
        times.append(time.perf_counter() - t0)
    med = sorted(times)[10]
    print(f"facade decide 224x224/P16 median {med * 1e3:.3f} ms")
    assert med < 10e-3
