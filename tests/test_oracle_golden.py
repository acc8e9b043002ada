"""Pin the CPU oracle (CPU-only).

(a) Against fixtures recorded by running the reference itself
    (tests/golden/make_golden.py): every discrete field bit-exact, floats
    within 1e-12 relative (the oracle uses the same scipy transforms).
(b) Against the known-answer values held by the reference's own tests.
"""

import json
import math
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import freqcache_oracle as O

GOLD = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(GOLD))
from cases import C1, C2, fhash, small_cases  # noqa: E402


def _ocfg(c):
    return O.OracleConfig(tau_mig=c.get("tau_mig", 0.12), edge_lambda=c.get("edge_lambda", 0.25),
                          alpha_min=c.get("alpha_min", 0.08), alpha_max=c.get("alpha_max", 0.5),
                          patch_size=c["patch_size"], refresh_shift=c.get("refresh_shift"))


def _same(d, g, ftol=1e-12):
    assert d.flushed == g["flushed"]
    assert list(d.displacement) == g["displacement"]
    assert d.k_reuse == g["k_reuse"] and d.k_candidate == g["k_candidate"] and d.k_final == g["k_final"]
    assert list(d.reuse_set) == g["reuse_set"]
    assert list(d.refresh_set) == g["refresh_set"]
    assert d.diagnostic == g["diagnostic"]
    assert (d.rows, d.cols) == (g["rows"], g["cols"])
    assert d.entropy[2] == g["entropy"][2]
    for a, b in ((d.sim_freq, g["sim_freq"]), (d.alpha_t, g["alpha_t"]),
                 (d.entropy[0], g["entropy"][0]), (d.entropy[1], g["entropy"][1])):
        assert abs(a - b) <= ftol * max(1.0, abs(b))


def test_small_cases_match_reference():
    gold = json.loads((GOLD / "golden_small.json").read_text())
    cases = small_cases()
    assert len(cases) == len(gold)
    for (name, prev, curr, c), g in zip(cases, gold):
        assert g["name"] == name and g["prev"] == fhash(prev) and g["curr"] == fhash(curr)
        _same(O.decide(prev, curr, _ocfg(c)), g["decision"])


def test_generator_is_frozen_and_c1_matches_reference():
    from paper_2604_24391_b200.synth import stream_frames
    gold = json.loads((GOLD / "golden_c1.json").read_text())
    fr = stream_frames(C1["seed"], C1["stream"], C1["steps"], C1["size"], C1["size"])
    assert [fhash(f) for f in fr] == gold["frames"]
    cfg = _ocfg({"patch_size": C1["patch"], "alpha_min": C1["alpha"][0], "alpha_max": C1["alpha"][1]})
    for t, g in enumerate(gold["decisions"], start=1):
        if t % 4:  # every 4th step keeps the CPU suite fast; GPU tests cover all
            continue
        _same(O.decide(fr[t - 1], fr[t], cfg, step=t), g)


def test_c2_shift_rule_matches_reference_adapter():
    """The oracle reproduces every one of golden_c2's 26 reference decisions
    (2 streams x 13 steps at 448x448, config-2 shift rule) exactly."""
    from paper_2604_24391_b200.synth import stream_frames
    gold = json.loads((GOLD / "golden_c2.json").read_text())
    cfg = _ocfg({"patch_size": C2["patch"], "refresh_shift": C2["refresh_shift"]})
    n = 0
    for s, rec in enumerate(gold["streams"]):
        fr = stream_frames(C2["seed"], s, C2["steps"], C2["size"], C2["size"])
        assert [fhash(f) for f in fr] == rec["frames"]
        for t in range(1, C2["steps"]):
            _same(O.decide(fr[t - 1], fr[t], cfg, step=t), rec["decisions"][t - 1])
            n += 1
    assert n == 26


def test_splice_matches_reference_step():
    gold = json.loads((GOLD / "golden_step.json").read_text())
    rng = np.random.default_rng(77)
    frames = [rng.random((64, 64))]
    for _ in range(5):
        frames.append(np.roll(frames[-1], (int(rng.integers(-9, 10)), int(rng.integers(-9, 10))), axis=(0, 1)))
    assert [fhash(f) for f in frames] == gold["frames"]
    cfg = O.OracleConfig(patch_size=8, alpha_min=0.6, alpha_max=0.6)

    def token_fn(p):
        counts, _ = np.histogram(np.clip(p, 0.0, 1.0), bins=16, range=(0.0, 1.0))
        return np.concatenate([counts.astype(np.float64), [p.mean(), p.var()]])

    n = 64
    tokens = np.stack([token_fn(frames[0][i * 8:(i + 1) * 8, j * 8:(j + 1) * 8])
                       for i in range(8) for j in range(8)])
    ages = np.zeros(n, dtype=np.int64)
    for t, g in enumerate(gold["steps"], start=1):
        d = O.decide(frames[t - 1], frames[t], cfg, step=t)
        _same(d, g["decision"])
        fresh = np.stack([token_fn(frames[t][(q // 8) * 8:(q // 8 + 1) * 8, (q % 8) * 8:(q % 8 + 1) * 8])
                          for q in d.recompute_set])
        tokens, ages = O.splice(tokens, ages, d, fresh)
        assert fhash(tokens.reshape(8, 8, -1)) == g["tokens"]
        assert ages.tolist() == g["ages"]


# ------------------------------------------------ reference known answers --

def test_refresh_known_answer():
    # test_edge_refresh.py:101-108
    mask, mu, sd, thr = O.refresh(np.array([[0.0, 0.0], [0.0, 100.0]]), 0.25)
    assert mu == 25.0
    assert thr == pytest.approx(35.825317547305483)
    assert mask.tolist() == [[False, False], [False, True]]
    m2, _, s2, _ = O.refresh(np.full((3, 3), 4.2), 0.25)
    assert s2 == 0.0 and not m2.any()


def test_budget_known_answers():
    # test_budget.py:86-94
    assert O.budget(0.0, 0.08, 0.5, 196) == (0.5, 98)
    assert O.budget(1.0, 0.08, 0.5, 196)[1] == 45
    with pytest.raises(ValueError):
        O.budget(1.0000000000000002, 0.08, 0.5, 196)


def test_entropy_known_answers():
    # test_budget.py:20-39
    amp = np.zeros((8, 8))
    amp[3, 5] = 7.0
    assert O.entropy(amp)[:2] == (0.0, 0.0)
    raw, psi, bins = O.entropy(np.full((8, 8), 2.0))
    assert raw == pytest.approx(math.log(64), abs=1e-12) and psi == pytest.approx(1.0, abs=1e-12)
    amp = np.zeros((8, 8))
    amp[0, 1] = amp[5, 2] = 3.0
    raw, psi, _ = O.entropy(amp)
    assert raw == pytest.approx(math.log(2), abs=1e-12) and psi == pytest.approx(1 / 6, abs=1e-12)


def test_topk_known_answers():
    # test_fusion.py:31-46
    assert O.topk_ascending([0, 1, 2], np.array([5.0, 1.0, 3.0]), 2) == (1, 2)
    assert O.topk_ascending([0, 1, 2, 3], np.array([4.0, 2.0, 9.0, 1.0]), 10) == (3, 1, 0, 2)
    assert O.topk_ascending([2, 0, 1, 3], np.array([2.0, 2.0, 2.0, 1.0]), 3) == (3, 0, 1)
    assert O.topk_ascending([], np.array([]), 5) == ()


@pytest.mark.parametrize("pixels,expected", [(0, 0), (3, 0), (4, 0), (5, 1), (8, 1), (12, 1), (13, 2),
                                             (-3, 0), (-4, 0), (-5, -1), (-12, -1), (-13, -2)])
def test_quantisation_table(pixels, expected):
    # test_migration.py:136-143
    assert O.to_patches(pixels, 8) == expected


def test_phase_correlation_known_shifts():
    # test_migration.py:102-112
    f = np.random.default_rng(6).random((64, 64))
    r = O.correlation_response(np.fft.fft2(f), np.fft.fft2(np.roll(f, (3, 5), axis=(0, 1))))
    assert O.peak_displacement(r) == (3, 5)
    f = np.random.default_rng(7).random((64, 64))
    r = O.correlation_response(np.fft.fft2(f), np.fft.fft2(np.roll(f, (61, 0), axis=(0, 1))))
    assert O.peak_displacement(r) == (-3, 0)


def test_degenerate_diagnostics():
    # test_fusion.py:102-109
    f = np.random.default_rng(8).random((32, 32))
    cfg = O.OracleConfig(patch_size=8)
    d = O.decide(np.zeros((32, 32)), f, cfg)
    assert d.flushed and d.diagnostic == "degenerate spectrum"
    d = O.decide(np.full((32, 32), 0.5), f, cfg)
    assert d.flushed and d.diagnostic == "no texture; displacement undefined"


def test_white_noise_regression_anchor():
    # test_fusion.py:237-245 (mean reuse of run_sequence on white noise)
    gold = json.loads((GOLD / "golden_step.json").read_text())
    rng = np.random.default_rng(24)
    frames = [rng.random((64, 64)) for _ in range(8)]
    cfg = O.OracleConfig(patch_size=8)
    ks = [O.decide(frames[t - 1], frames[t], cfg).k_final for t in range(1, 8)]
    assert sum(ks) / (7 * 64) == pytest.approx(0.3392857142857143, abs=1e-12)
    assert gold["sequence_mean_reuse"] > 0


# ------------------------------------------- comparison baselines (§8f #3) --

def _report_same(rep, gold, ftol=1e-12):
    assert rep["n_steps"] == gold["n_steps"] and rep["n_tokens"] == gold["n_tokens"]
    assert rep["thresholds"] == gold["thresholds"]
    assert math.isclose(rep["baseline_latency_ms"], gold["baseline_latency_ms"], rel_tol=ftol)
    for name, g in gold["policies"].items():
        r = rep["policies"][name]
        assert r["reuse_ratio"] == g["reuse_ratio"], name
        assert r["edge_false_reuse"] == g["edge_false_reuse"], name
        assert math.isclose(r["mean_latency_ms"], g["mean_latency_ms"], rel_tol=ftol), name
        assert math.isclose(r["speedup"], g["speedup"], rel_tol=ftol), name


def test_oracle_compare_domains_matches_reference():
    from cases import compare_cases
    gold = {c["name"]: c for c in json.loads((GOLD / "golden_compare.json").read_text())["cases"]}
    for name, frames, c, labels in compare_cases():
        g = gold[name]
        assert [fhash(f) for f in frames] == g["frames"], name
        _report_same(O.compare_domains(frames, _ocfg(c), edge_labels=labels), g["report"])


def test_oracle_compare_cosines_baseline_pair():
    from paper_2604_24391_b200.synth import stream_frames
    pair = json.loads((GOLD / "golden_compare.json").read_text())["pair"]
    r = pair["recipe"]
    fr = stream_frames(r["seed"], 0, 2, r["size"], r["size"])
    assert [fhash(f) for f in fr] == pair["frames"]
    vis, nf = O.compare_cosines(fr[0], fr[1], r["patch"])
    np.testing.assert_allclose(vis, pair["visual"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(nf, pair["naive_freq"], rtol=1e-12, atol=1e-14)


def test_oracle_position_cosines_zero_norm():
    a = np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 1.0]])
    b = np.array([[1.0, 1.0], [0.0, 1.0], [2.0, 2.0]])
    np.testing.assert_allclose(O.position_cosines(a, b), [0.0, 0.0, 1.0])
