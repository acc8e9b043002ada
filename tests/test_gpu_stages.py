"""GPU tests: stand-alone stage operators, reference-recorded goldens,
multi-chunk / multi-lane scheduling, and the known answers of the
reference's own stage tests (test_budget.py, test_edge_refresh.py,
test_migration.py, test_fusion.py)."""

import json
import math
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import freqcache_oracle as O
from oracle.parity import ParityReport, compare

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(GOLD))
from cases import C1, C2, fhash, small_cases  # noqa: E402


class _G:
    """Golden record -> object with CacheDecision-like fields for compare()."""

    def __init__(self, g):
        self.__dict__.update(g)


def _ocfg(c):
    return O.OracleConfig(tau_mig=c.get("tau_mig", 0.12), edge_lambda=c.get("edge_lambda", 0.25),
                          alpha_min=c.get("alpha_min", 0.08), alpha_max=c.get("alpha_max", 0.5),
                          patch_size=c["patch_size"], refresh_shift=c.get("refresh_shift"))


def _fcfg(c):
    import paper_2604_24391_b200 as fc
    return fc.CacheConfig(tau_mig=c.get("tau_mig", 0.12), edge_lambda=c.get("edge_lambda", 0.25),
                          budget=fc.BudgetConfig(c.get("alpha_min", 0.08), c.get("alpha_max", 0.5)),
                          patch_size=c["patch_size"])


# ------------------------------------------------------ stage operators ----

def test_sim_freq(cuda):
    import paper_2604_24391_b200 as fc
    amp = np.abs(np.fft.fft2(np.random.default_rng(3).random((16, 16))))
    assert fc.sim_freq(amp, amp) == pytest.approx(1.0, abs=1e-12)
    f = np.random.default_rng(4).random((24, 24))
    assert fc.sim_freq(np.abs(np.fft.fft2(f)), np.abs(np.fft.fft2(np.roll(f, (5, 11), axis=(0, 1))))) >= 1 - 1e-9
    a, b = np.zeros((4, 4)), np.zeros((4, 4))
    a[0, 1] = b[2, 3] = 1.0
    assert fc.sim_freq(a, b) == 0.0
    with pytest.raises(fc.DegenerateSpectrumError, match="degenerate spectrum"):
        fc.sim_freq(np.zeros((4, 4)), np.ones((4, 4)))
    with pytest.raises(ValueError):
        fc.sim_freq(np.full((4, 4), -1.0), np.ones((4, 4)))
    with pytest.raises(ValueError):
        fc.sim_freq(np.full((4, 4), np.nan), np.ones((4, 4)))
    rng = np.random.default_rng(9)
    for _ in range(5):
        x, y = rng.random((37, 53)), rng.random((37, 53))
        assert fc.sim_freq(x, y) == pytest.approx(O.similarity(x, y), rel=1e-13)


def test_spectral_entropy(cuda):
    import paper_2604_24391_b200 as fc
    amp = np.zeros((8, 8))
    amp[3, 5] = 7.0
    r = fc.spectral_entropy(amp)
    assert r.raw == 0.0 and r.normalized == 0.0 and r.bin_count == 64
    r = fc.spectral_entropy(np.full((8, 8), 2.0))
    assert r.raw == pytest.approx(math.log(64), abs=1e-12) and r.normalized == pytest.approx(1.0, abs=1e-12)
    amp = np.zeros((8, 8))
    amp[0, 1] = amp[5, 2] = 3.0
    r = fc.spectral_entropy(amp)
    assert r.raw == pytest.approx(math.log(2), abs=1e-12) and r.normalized == pytest.approx(1 / 6, abs=1e-12)
    with pytest.raises(fc.DegenerateSpectrumError):
        fc.spectral_entropy(np.zeros((4, 4)))
    amp = np.zeros((4, 4))
    amp[0, 0], amp[1, 1], amp[2, 2] = 10.0, 1.0, 1.0
    r = fc.spectral_entropy(amp, include_dc=False)
    assert r.raw == pytest.approx(math.log(2), abs=1e-12)
    rng = np.random.default_rng(0)
    a = rng.random((64, 64))
    assert fc.spectral_entropy(a).raw == pytest.approx(O.entropy(a)[0], abs=1e-12)


def test_refresh_mask(cuda):
    import paper_2604_24391_b200 as fc
    r = fc.refresh_mask(fc.EnergyMap(np.array([[0.0, 0.0], [0.0, 100.0]]), 8, 2), 0.25)
    assert r.mean_energy == pytest.approx(25.0)
    assert r.mean_energy + 0.25 * r.std_energy == pytest.approx(35.825317547305483)
    assert r.mask.tolist() == [[False, False], [False, True]]
    r = fc.refresh_mask(fc.EnergyMap(np.full((3, 3), 4.2), 8, 2), 0.25)
    assert r.std_energy == 0.0 and not r.mask.any()
    e = np.random.default_rng(3).random((4, 4))
    assert not fc.refresh_mask(fc.EnergyMap(e, 8, 2), math.inf).mask.any()
    big = np.random.default_rng(5).random((300, 300))
    m, mu, sd, _ = O.refresh(big, 0.25)
    r = fc.refresh_mask(fc.EnergyMap(big, 8, 2), 0.25)
    assert r.mean_energy == pytest.approx(mu, rel=1e-13) and r.std_energy == pytest.approx(sd, rel=1e-12)
    assert np.array_equal(r.mask, m)


def test_topk_ascending(cuda):
    import paper_2604_24391_b200 as fc
    assert fc.topk_ascending([0, 1, 2], np.array([5.0, 1.0, 3.0]), 2) == (1, 2)
    assert fc.topk_ascending([0, 1, 2, 3], np.array([4.0, 2.0, 9.0, 1.0]), 10) == (3, 1, 0, 2)
    assert fc.topk_ascending([2, 0, 1, 3], np.array([2.0, 2.0, 2.0, 1.0]), 3) == (3, 0, 1)
    assert fc.topk_ascending([], np.array([]), 5) == ()
    assert fc.topk_ascending([1], np.array([0.0, 1.0]), 0) == ()
    rng = np.random.default_rng(11)
    e = np.round(rng.random(5000), 2)  # many exact ties
    cand = rng.permutation(5000)[:3000]
    assert fc.topk_ascending(cand, e, 1700) == O.topk_ascending(cand, e, 1700)


# ---------------------------------------------- reference-recorded goldens --

def test_small_goldens_through_gpu(cuda):
    """GPU decisions against the reference's own recorded decisions (margins
    from the pinned oracle)."""
    import paper_2604_24391_b200 as fc
    gold = json.loads((GOLD / "golden_small.json").read_text())
    rep = ParityReport()
    for (name, prev, curr, c), g in zip(small_cases(), gold):
        assert g["prev"] == fhash(prev) and g["curr"] == fhash(curr)
        d = fc.decide(prev, curr, _fcfg(c))
        o = O.decide(prev, curr, _ocfg(c))
        gd = _G(g["decision"])
        assert list(o.reuse_set) == gd.reuse_set  # oracle pinned on this case
        compare(d, o, _ocfg(c), rep=rep)
    assert rep.ok, rep.errors


def test_c1_golden_sequence(cuda):
    import torch
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200.api import _fetch, decision_from_device
    from paper_2604_24391_b200.synth import stream_frames
    gold = json.loads((GOLD / "golden_c1.json").read_text())
    fr = stream_frames(C1["seed"], C1["stream"], C1["steps"], C1["size"], C1["size"])
    assert [fhash(f) for f in fr] == gold["frames"]
    cfg = fc.CacheConfig(patch_size=14, budget=fc.BudgetConfig(0.5, 0.5))
    oc = _ocfg({"patch_size": 14, "alpha_min": 0.5, "alpha_max": 0.5})
    eng = fc.FreqCacheEngine(1, 224, 224, 14, fmt="rgb")
    rep = ParityReport()
    exact = 0
    for t in range(len(fr)):
        out = eng.select(torch.from_numpy(fr[t:t + 1]).cuda(), cfg)
        if t == 0:
            continue
        d = decision_from_device(*_fetch(out), step=t)
        g = gold["decisions"][t - 1]
        o = O.decide(fr[t - 1], fr[t], oc, step=t)
        assert list(o.reuse_set) == g["reuse_set"]
        compare(d, o, oc, rep=rep)
        exact += list(d.reuse_set) == g["reuse_set"] and list(d.refresh_set) == g["refresh_set"]
    assert rep.ok, rep.errors
    print("config-1 steps bit-identical to the reference:", exact, "of", len(fr) - 1, rep.exemptions)


def test_c2_golden_two_streams_batched(cuda):
    """Config-2 reference decisions (golden_c2.json: 2 streams x 13 steps,
    recorded by running the reference itself plus the config-2 rule): the
    batched device decision is compared field by field with the REFERENCE's
    record — flush, displacement, k_reuse / k_candidate / k_final, refresh
    set and reuse set exactly, reuse order except between tokens whose
    energies lie inside the 1e-4 / rounding-floor tie margin — and through
    the margin-aware checker against the oracle (pinned to the same 26
    records on the CPU).  Only order exemptions are allowed."""
    import torch
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200.api import decision_from_device
    from paper_2604_24391_b200.synth import stream_frames
    from oracle.parity import REL
    gold = json.loads((GOLD / "golden_c2.json").read_text())
    S, T = C2["streams"], C2["steps"]
    frames = np.stack([stream_frames(C2["seed"], s, T, 448, 448) for s in range(S)], axis=1)
    for s in range(S):
        assert [fhash(f) for f in frames[:, s]] == gold["streams"][s]["frames"]
    cfg = fc.CacheConfig(patch_size=14)
    oc = _ocfg({"patch_size": 14, "refresh_shift": 1})
    eng = fc.FreqCacheEngine(S, 448, 448, 14, fmt="rgb")
    rep = ParityReport()
    n_dec = n_order = 0
    for t in range(T):
        out = eng.select(torch.from_numpy(np.ascontiguousarray(frames[t])).cuda(), cfg, refresh_shift=1)
        if t == 0:
            continue
        res = out.host_results()
        ri, rc, rm = out.reuse_idx.cpu().numpy(), out.recompute_idx.cpu().numpy(), out.refresh_mask.cpu().numpy()
        en = out.energy.cpu().numpy()
        for s in range(S):
            d = decision_from_device(res[s], ri[s], rc[s], rm[s], step=t)
            g = gold["streams"][s]["decisions"][t - 1]
            o = O.decide(frames[t - 1, s], frames[t, s], oc, step=t)
            compare(d, o, oc, energies=en[s], rep=rep)
            # device vs the reference's own record, every discrete field
            assert d.flushed == g["flushed"], (s, t)
            assert d.diagnostic == g["diagnostic"], (s, t)
            assert [d.displacement.di, d.displacement.dj, d.displacement.di_patches,
                    d.displacement.dj_patches] == g["displacement"], (s, t)
            assert (d.k_reuse, d.k_candidate, d.k_final) == (g["k_reuse"], g["k_candidate"], g["k_final"]), (s, t)
            assert list(d.refresh_set) == g["refresh_set"], (s, t)
            assert set(d.reuse_set) == set(g["reuse_set"]), (s, t)
            assert list(d.recompute_set) == sorted(set(range(d.rows * d.cols)) - set(g["reuse_set"]))
            assert abs(d.sim_freq - g["sim_freq"]) <= 1e-3 * g["sim_freq"]
            assert abs(d.entropy.normalized - g["entropy"][1]) <= 1e-3 * g["entropy"][1]
            # order: wherever two neighbours of the reference's order differ in
            # energy by more than the tie margin, the device keeps their order
            pos = {q: i for i, q in enumerate(d.reuse_set)}
            e, floor = o.energies, 1e-6 * float(o.energies.mean())
            for a, b in zip(g["reuse_set"], g["reuse_set"][1:]):
                if abs(e[a] - e[b]) > REL * max(e[a], e[b]) + floor:
                    assert pos[a] < pos[b], (s, t, a, b)
            n_order += list(d.reuse_set) == g["reuse_set"]
            n_dec += 1
    assert rep.ok, rep.errors
    assert set(rep.exemptions) <= {"order"}, rep.exemptions
    print(f"config-2 golden: {n_dec}/{n_dec} decisions with the reference's sets, {n_order} in its exact "
          f"order; exemptions {rep.exemptions}")


def test_multichunk_multilane_batch(cuda, monkeypatch):
    """70 streams in 16-stream chunks on 3 lanes: every stream's decision
    equals the single-stream result (chunking never mixes streams)."""
    import torch
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200.synth import torch_stream_frames
    monkeypatch.setenv("FC_CHUNK", "16")
    monkeypatch.setenv("FC_LANES", "3")
    S = 70
    frames = torch_stream_frames(S, 3, 448, 448, seed=99, device="cuda")
    cfg = fc.CacheConfig(patch_size=14)
    big = fc.FreqCacheEngine(S, 448, 448, 14, fmt="rgb")
    monkeypatch.setenv("FC_CHUNK", "512")
    monkeypatch.setenv("FC_LANES", "1")
    one = fc.FreqCacheEngine(S, 448, 448, 14, fmt="rgb")
    for t in range(3):
        a = big.select(frames[t], cfg, refresh_shift=1)
        b = one.select(frames[t], cfg, refresh_shift=1)
        assert torch.equal(a.results, b.results)
        assert torch.equal(a.reuse_idx, b.reuse_idx)
        assert torch.equal(a.src_map, b.src_map)
        assert torch.equal(a.energy, b.energy)
    res = a.host_results()
    assert (res["cold"] == 0).all() and (res["status"] == 0).all()
    # spot-check two streams against the oracle
    oc = O.OracleConfig(patch_size=14, refresh_shift=1)
    from paper_2604_24391_b200.api import decision_from_device
    rep = ParityReport()
    f1, f2 = frames[1].cpu().numpy(), frames[2].cpu().numpy()
    for s in (0, 69):
        d = decision_from_device(res[s], a.reuse_idx[s].cpu().numpy(), a.recompute_idx[s].cpu().numpy(),
                                 a.refresh_mask[s].cpu().numpy(), step=2)
        compare(d, O.decide(f1[s], f2[s], oc), oc, energies=a.energy[s].cpu().numpy(), rep=rep)
    assert rep.ok, rep.errors


def test_engine_reset_and_partial_reset(cuda):
    import torch
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200.synth import stream_frames
    f = np.stack([stream_frames(5, s, 3, 224, 224) for s in range(3)], axis=1)
    eng = fc.FreqCacheEngine(3, 224, 224, 14, fmt="rgb")
    cfg = fc.CacheConfig(patch_size=14)
    eng.select(torch.from_numpy(np.ascontiguousarray(f[0])).cuda(), cfg)
    eng.reset(first=1, count=1)
    r = eng.select(torch.from_numpy(np.ascontiguousarray(f[1])).cuda(), cfg).host_results()
    assert list(r["cold"]) == [0, 1, 0]
    assert r["k_final"][1] == 0 and r["flushed"][1] == 1


def test_records_rerun_byte_identical(cuda, tmp_path):
    """Acceptance criterion 7 of the reference (test_acceptance.py:207-234):
    identical inputs give byte-identical JSONL / CSV / PGM outputs; masks
    rendered on the GPU equal the index-set rendering."""
    import torch
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200 import records
    rng = np.random.default_rng(21)
    base = rng.random((64, 64))
    frames = [np.roll(base, (3 * t, 5 * t), axis=(0, 1)) for t in range(8)]
    cfg = fc.CacheConfig(patch_size=8)
    outs = []
    for run in ("a", "b"):
        rep = fc.run_sequence(frames, cfg)
        d = tmp_path / run
        d.mkdir()
        records.write_decisions_jsonl(d / "decisions.jsonl", rep.decisions)
        records.write_metrics_csv(d / "metrics.csv", rep)
        records.export_masks(records.read_decisions_jsonl(d / "decisions.jsonl"), d / "masks")
        outs.append(d)
    for name in ("decisions.jsonl", "metrics.csv"):
        assert (outs[0] / name).read_bytes() == (outs[1] / name).read_bytes()
    pa, pb = sorted((outs[0] / "masks").glob("*.pgm")), sorted((outs[1] / "masks").glob("*.pgm"))
    assert len(pa) == 7 and all(x.read_bytes() == y.read_bytes() for x, y in zip(pa, pb))
    # device-rendered masks == host rendering of the same decisions
    eng = fc.FreqCacheEngine(1, 64, 64, 8, fmt="gray64")
    dev_imgs, decs = [], []
    from paper_2604_24391_b200.api import _fetch, decision_from_device
    for t, f in enumerate(frames):
        out = eng.select(torch.from_numpy(f).cuda().unsqueeze(0), cfg)
        if t == 0:
            continue
        dev_imgs.append(records.render_masks(out, eng)[0].cpu().numpy())
        decs.append(decision_from_device(*_fetch(out), step=t))
    paths = records.export_masks(decs, tmp_path / "host")
    for img, p in zip(dev_imgs, paths):
        data = p.read_bytes()
        assert data.endswith(img.tobytes())


def test_vit_cached_encoder_small(cuda):
    """Config-4 plumbing on a small ViT: cold steps equal a full recompute;
    reused rows are bit copies of the shifted cache."""
    import torch
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200.synth import torch_stream_frames
    from paper_2604_24391_b200.vit import CachedEncoder, ViT, ViTConfig, cosine
    c = ViTConfig(image=112, patch=14, width=64, mlp=128, heads=2, layers=3)
    model = ViT(c).cuda().float().eval()
    frames = torch_stream_frames(2, 4, 112, 112, seed=3, device="cuda")
    cfg = fc.CacheConfig(patch_size=14)
    with torch.no_grad():
        for mode in ("layer1", "subset"):
            enc = CachedEncoder(model, 2, mode=mode)
            y0, out0 = enc.step(frames[0], cfg)
            assert (out0.host_results()["cold"] == 1).all()
            ref = model(frames[0])
            assert torch.allclose(y0, ref, atol=2e-5, rtol=1e-4)
            prev_h = enc.h1[enc.cur].clone()
            y1, out1 = enc.step(frames[1], cfg)
            cache_now = enc.h1[enc.cur]
            sm = out1.src_map
            for b in range(2):
                for p in range(c.tokens):
                    s = int(sm[b, p])
                    if s >= 0:
                        assert torch.equal(cache_now[b, p], prev_h[b, s])
            assert float(cosine(y1, model(frames[1])).min()) > 0.5
            enc.check()


@pytest.mark.parametrize("dtype", ["float32", "bfloat16"])
def test_vit_layer1_step_matches_reference_semantics(cuda, dtype):
    """layer1 mode against a plain-torch restatement of its semantics on a
    small fp32 ViT, with the next step's select issued ahead: for every
    stream, block-0 queries = recomputed tokens, keys / values = the
    displacement-mapped cached K/V rows for reused tokens and fresh ones for
    recomputed tokens; block-0 outputs spliced; blocks 1.. on all tokens."""
    import torch
    import torch.nn.functional as F
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200.synth import torch_stream_frames
    from paper_2604_24391_b200.vit import CachedEncoder, ViT, ViTConfig
    c = ViTConfig(image=112, patch=14, width=64, mlp=128, heads=2, layers=3)
    dt = getattr(torch, dtype)   # bf16: the flash-attention varlen path; fp32: per-stream SDPA
    model = ViT(c).cuda().to(dt).eval()
    T = 5
    frames = torch_stream_frames(3, T, 112, 112, seed=9, device="cuda")
    cfg = fc.CacheConfig(patch_size=14)
    enc = CachedEncoder(model, 3, mode="layer1")
    blk = model.blocks[0]
    d = c.width
    with torch.no_grad():
        kc = vc = hc = None
        for t in range(T):
            y, out = enc.step(frames[t], cfg, next_frames=frames[t + 1] if t + 1 < T else None)
            x0 = model.embed_tokens(model.patches(frames[t].to(dt)))            # all tokens, layer 0
            q, k, v = F.linear(blk.ln1(x0), blk.qkv.weight, blk.qkv.bias).split(d, dim=-1)
            sm = out.src_map.long()
            if kc is not None:
                idx = sm.clamp_min(0)[..., None].expand(-1, -1, d)
                reuse = (sm >= 0)[..., None]
                k = torch.where(reuse, torch.gather(kc, 1, idx), k)
                v = torch.where(reuse, torch.gather(vc, 1, idx), v)
            att = F.scaled_dot_product_attention(blk._heads(q), blk._heads(k), blk._heads(v))
            x = x0 + blk.proj(att.transpose(1, 2).flatten(-2))
            h = x + blk.fc2(F.gelu(blk.fc1(blk.ln2(x)), approximate="tanh"))
            if hc is not None:
                h = torch.where((sm >= 0)[..., None], torch.gather(hc, 1, sm.clamp_min(0)[..., None].expand(-1, -1, d)), h)
            kc, vc, hc = k, v, h
            xr = h
            for b2 in model.blocks[1:]:
                xr = b2(xr)
            ref = model.ln(xr)
            if dt == torch.float32:
                assert torch.allclose(y, ref, atol=1e-4, rtol=1e-3), (t, float((y - ref).abs().max()))
                assert torch.allclose(enc.h1[enc.cur], h, atol=1e-5)
            else:
                from paper_2604_24391_b200.vit import cosine
                assert float(cosine(y, ref).min()) > 0.999, t
                assert float(cosine(enc.h1[enc.cur], h).min()) > 0.999, t
        enc.check()


def test_vit_subset_step_matches_reference_semantics(cuda):
    """subset mode (bf16: the packed encoder replayed from a CUDA graph per
    row bucket, flash-attention varlen with zero-length and padding
    segments) against a plain-torch restatement, stream by stream: the
    recomputed tokens (row-major) run the whole encoder attending among
    themselves; reused tokens take their displacement-mapped cached final
    state.  Also equal to the eager (ungraphed) packed path."""
    import torch
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200.synth import torch_stream_frames
    from paper_2604_24391_b200.vit import CachedEncoder, ViT, ViTConfig, cosine
    c = ViTConfig(image=112, patch=14, width=64, mlp=128, heads=2, layers=3)
    model = ViT(c).cuda().to(torch.bfloat16).eval()
    T, B = 5, 3
    frames = torch_stream_frames(B, T, 112, 112, seed=13, device="cuda")
    cfg = fc.CacheConfig(patch_size=14)
    enc = CachedEncoder(model, B, mode="subset")
    assert enc.sub_graphs, "the bf16 subset path must be graphed"
    eager = CachedEncoder(model, B, mode="subset", graphs=False)
    with torch.no_grad():
        hc = None
        for t in range(T):
            nxt = frames[t + 1] if t + 1 < T else None
            y, out = enc.step(frames[t], cfg, next_frames=nxt)
            ye, oute = eager.step(frames[t], cfg, next_frames=nxt)
            assert torch.equal(out.src_map, oute.src_map)
            assert float(cosine(y, ye).min()) > 0.9999, t
            x0 = model.embed_tokens(model.patches(frames[t].to(torch.bfloat16)))
            sm = out.src_map.long()
            h = torch.empty_like(x0)
            for b in range(B):
                rec = (sm[b] < 0).nonzero().flatten()
                if rec.numel():
                    xr = x0[b, rec][None]
                    for blk in model.blocks:
                        xr = blk(xr)
                    h[b, rec] = model.ln(xr)[0]
                keep = (sm[b] >= 0).nonzero().flatten()
                if keep.numel():
                    h[b, keep] = hc[b, sm[b, keep]]
            hc = h
            assert float(cosine(y, h).min()) > 0.999, t
        enc.check()
        eager.check()


def test_inplace_splice_matches_oracle(cuda):
    """fc_splice_inplace: zero-displacement streams update in place (reused
    rows untouched), shifted streams ping-pong; results equal the oracle
    splice bit for bit (bf16)."""
    import torch
    import paper_2604_24391_b200 as fc
    B, rows, cols, D = 5, 8, 8, 96
    N = rows * cols
    g = torch.Generator(device="cuda").manual_seed(1)
    cache = torch.empty((2, B, N, D), dtype=torch.bfloat16, device="cuda")
    cache[0] = torch.randn((B, N, D), generator=g, device="cuda").to(torch.bfloat16)
    ages = torch.zeros((2, B, N), dtype=torch.int64, device="cuda")
    ages[0] = torch.randint(0, 4, (B, N), generator=g, device="cuda")
    st = fc.SpliceState(cache, ages)
    rng = np.random.default_rng(7)
    ref_tok = [cache[0, b].view(torch.int16).cpu().numpy().copy() for b in range(B)]
    ref_age = [ages[0, b].cpu().numpy().copy() for b in range(B)]
    for stepi in range(4):
        src = np.empty((B, N), dtype=np.int32)
        decs = []
        for b in range(B):
            dip, djp = [(0, 0), (1, 0), (0, -1), (0, 0), (2, 1)][(b + stepi) % 5]
            al = [q for q in range(N) if 0 <= q // cols - dip < rows and 0 <= q % cols - djp < cols]
            reuse = tuple(int(v) for v in rng.permutation(al)[: len(al) // 2])
            flushed = (b + stepi) % 7 == 6
            d = O.OracleDecision(step=1, flushed=flushed, sim_freq=1.0, displacement=(0, 0, dip, djp),
                                 entropy=(0, 0, 0), alpha_t=0.5, k_reuse=0, k_candidate=0,
                                 k_final=0 if flushed else len(reuse), reuse_set=() if flushed else reuse,
                                 recompute_set=(), rows=rows, cols=cols, refresh_set=())
            decs.append(d)
            m = fc.splice_map(rows, cols, torch.tensor(d.reuse_set, dtype=torch.int32, device="cuda")
                              if d.reuse_set else None, dip, djp)
            src[b] = m.cpu().numpy()
        fresh = torch.randn((B, N, D), generator=g, device="cuda").to(torch.bfloat16)
        st.step(torch.from_numpy(src).cuda(), fresh, compact=False)
        tok, age = st.current()
        fr = fresh.view(torch.int16).cpu().numpy()
        for b in range(B):
            rec = [q for q in range(N) if q not in set(decs[b].reuse_set)]
            exp, exp_age = O.splice(ref_tok[b], ref_age[b], decs[b], fr[b][rec])
            assert np.array_equal(tok[b].view(torch.int16).cpu().numpy(), exp), (stepi, b)
            assert np.array_equal(age[b].cpu().numpy(), exp_age), (stepi, b)
            ref_tok[b], ref_age[b] = exp, exp_age


def test_tensor_store_variants_bit_identical(cuda, monkeypatch):
    """K_A / K_B write T1 / T2 with TMA tensor stores by default; the
    per-thread store variants (FC_T1_TMA=0, FC_T2_TMA=0) compute the same
    values, so every output must be bit-identical (checks the tensor maps'
    layout and swizzle, including the multi-lane path)."""
    import torch
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200.synth import torch_stream_frames
    S = 40
    frames = torch_stream_frames(S, 3, 448, 448, seed=123, device="cuda")
    cfg = fc.CacheConfig(patch_size=14)
    engines = []
    for t1, t2, chunk, lanes in (("1", "1", "512", "1"), ("0", "0", "512", "1"), ("1", "0", "16", "2"),
                                 ("0", "1", "16", "3")):
        monkeypatch.setenv("FC_T1_TMA", t1)
        monkeypatch.setenv("FC_T2_TMA", t2)
        monkeypatch.setenv("FC_CHUNK", chunk)
        monkeypatch.setenv("FC_LANES", lanes)
        engines.append(fc.FreqCacheEngine(S, 448, 448, 14, fmt="rgb"))
    for t in range(3):
        outs = [e.select(frames[t], cfg, refresh_shift=1) for e in engines]
        for o in outs[1:]:
            assert torch.equal(o.results, outs[0].results)
            assert torch.equal(o.reuse_idx, outs[0].reuse_idx)
            assert torch.equal(o.src_map, outs[0].src_map)
            assert torch.equal(o.energy, outs[0].energy)
    for e in engines:
        assert torch.equal(e.state, engines[0].state)   # previous-frame spectra, bit for bit


@pytest.mark.parametrize("size,streams", [(448, 9), (224, 5), (448, 100)])
def test_split_phase_pipeline_bit_identical(cuda, size, streams):
    """fc_select_front / fc_select_back software-pipelined across steps (the
    front of step t + 1 enqueued on its own stream BEFORE the back of step t,
    alternating workspace slots, double-buffered outputs) gives exactly the
    decisions, splice maps and spectrum state of plain fc_select per step —
    including the small-batch two-lane chunking (100 streams)."""
    import torch
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200.synth import torch_stream_frames
    T = 5
    frames = torch_stream_frames(streams, T, size, size, seed=77, device="cuda")
    cfg = fc.CacheConfig(patch_size=14)
    ref = fc.FreqCacheEngine(streams, size, size, 14, fmt="rgb")
    pip = fc.FreqCacheEngine(streams, size, size, 14, fmt="rgb")
    outs = [pip.new_output(), pip.new_output()]
    fs = torch.cuda.Stream()
    cur = torch.cuda.current_stream()
    pip.select_front(frames[0], cfg, outs[0], 0, refresh_shift=1)
    for t in range(T):
        r = ref.select(frames[t], cfg, refresh_shift=1)
        fs.wait_stream(cur)
        if t + 1 < T:
            with torch.cuda.stream(fs):
                pip.select_front(frames[t + 1], cfg, outs[(t + 1) & 1], (t + 1) & 1, refresh_shift=1)
        o = pip.select_back(cfg, outs[t & 1], t & 1, refresh_shift=1)
        torch.cuda.synchronize()
        assert torch.equal(o.results, r.results), t
        for name in ("reuse_idx", "recompute_idx", "src_map", "reuse_mask", "refresh_mask", "energy"):
            assert torch.equal(getattr(o, name), getattr(r, name)), (t, name)
        cur.wait_stream(fs)
    assert torch.equal(pip.state, ref.state)


@pytest.mark.parametrize("streams", [40, 3])
def test_fused_cluster_colsinv_matches_split_kernels(cuda, monkeypatch, streams):
    """K_BC (FC_FUSED_BC=1: K_B + K_C in one 8-CTA cluster per stream, the
    cross-power handed over through distributed shared memory) computes the
    same transforms as K_B -> T2 -> K_C: identical decisions, splice maps,
    energies and spectrum state; sim / entropy within fp64 rounding of a
    different partial-sum grouping; and the oracle agrees."""
    import torch
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200.api import decision_from_device
    from paper_2604_24391_b200.synth import torch_stream_frames
    T = 4
    frames = torch_stream_frames(streams, T, 448, 448, seed=31, device="cuda")
    cfg = fc.CacheConfig(patch_size=14)
    monkeypatch.setenv("FC_FUSED_BC", "0")
    split = fc.FreqCacheEngine(streams, 448, 448, 14, fmt="rgb")
    monkeypatch.setenv("FC_FUSED_BC", "1")
    fused = fc.FreqCacheEngine(streams, 448, 448, 14, fmt="rgb")
    oc = O.OracleConfig(patch_size=14, refresh_shift=1)
    rep = ParityReport()
    for t in range(T):
        a = split.select(frames[t], cfg, refresh_shift=1)
        b = fused.select(frames[t], cfg, refresh_shift=1)
        for name in ("reuse_idx", "recompute_idx", "src_map", "reuse_mask", "refresh_mask", "energy"):
            assert torch.equal(getattr(a, name), getattr(b, name)), (t, name)
        ra, rb = a.host_results(), b.host_results()
        for f in ("status", "cold", "flushed", "diagnostic", "k_reuse", "k_candidate", "k_final", "di", "dj",
                  "di_patches", "dj_patches", "n_refresh"):
            assert np.array_equal(ra[f], rb[f]), (t, f)
        for f in ("peak", "peak_runner_up"):
            assert np.array_equal(ra[f], rb[f]), (t, f)   # same transforms, same argmax
        for f in ("sim_freq", "entropy_raw", "entropy_norm", "alpha"):
            assert np.allclose(ra[f], rb[f], rtol=1e-12, atol=0), (t, f)
        if t:
            fr = frames.cpu().numpy()
            for s in (0, streams - 1):
                d = decision_from_device(rb[s], b.reuse_idx[s].cpu().numpy(), b.recompute_idx[s].cpu().numpy(),
                                         b.refresh_mask[s].cpu().numpy(), step=t)
                compare(d, O.decide(fr[t - 1, s], fr[t, s], oc, step=t), oc, energies=b.energy[s].cpu().numpy(),
                        rep=rep)
    assert torch.equal(split.state, fused.state)
    assert rep.ok, rep.errors


@pytest.mark.parametrize("streams,lag,discard", [(40, 8, "1"), (3, 1, "1"), (20, 64, "0"), (200, 4, "1")])
def test_flow_colsinv_matches_split_kernels(cuda, monkeypatch, streams, lag, discard):
    """The K_B + K_C flow kernel (FC_BC_FLOW=1: one launch of ticket-ordered
    work items, K_C items of a stream waiting for its K_B items, T2 read from
    L2 and discarded) runs the same items as K_B -> T2 -> K_C: every output and
    the spectrum state bit-identical, through fc_select (small batches: two
    concurrent half-batch launches with their own tickets) and the split-phase
    front / back, over cold starts, a reset stream and repeated launches (the
    counters re-arm)."""
    import torch
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200.synth import torch_stream_frames
    T = 5
    frames = torch_stream_frames(streams, T, 448, 448, seed=37, device="cuda")
    cfg = fc.CacheConfig(patch_size=14)
    monkeypatch.setenv("FC_BC_FLOW", "0")
    ref = fc.FreqCacheEngine(streams, 448, 448, 14, fmt="rgb")
    monkeypatch.setenv("FC_BC_FLOW", "1")
    monkeypatch.setenv("FC_BC_LAG", str(lag))
    monkeypatch.setenv("FC_BC_DISCARD", discard)
    flow = fc.FreqCacheEngine(streams, 448, 448, 14, fmt="rgb")
    chunks = (ref.launches_per_select - 1) // 4
    assert flow.launches_per_select == ref.launches_per_select - chunks
    outs = [flow.new_output(), flow.new_output()]

    def same(a, b, t):
        for name in ("reuse_idx", "recompute_idx", "src_map", "reuse_mask", "refresh_mask", "energy", "results"):
            assert torch.equal(getattr(a, name), getattr(b, name)), (t, name)

    for t in range(T):
        if t == 3:
            ref.reset(streams // 2, 1)
            flow.reset(streams // 2, 1)
        a = ref.select(frames[t], cfg, refresh_shift=1)
        if t % 2 == 0:
            b = flow.select(frames[t], cfg, refresh_shift=1)
        else:
            b = outs[t & 1]
            flow.select_front(frames[t], cfg, b, t & 1, refresh_shift=1)
            flow.select_back(cfg, b, t & 1, refresh_shift=1)
        same(a, b, t)
        assert torch.equal(ref.state, flow.state), t


@pytest.mark.parametrize("streams", [64, 5])
def test_pdl_back_matches_plain_launches(cuda, monkeypatch, streams):
    """FC_PDL=1: K_C and K_D of the split-phase back launched as programmatic
    dependents (scheduled while their predecessor drains, griddepcontrol.wait
    before reading its outputs) give bit-identical outputs and state, also
    when captured in a CUDA graph."""
    import torch
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200.synth import torch_stream_frames
    T = 4
    frames = torch_stream_frames(streams, T, 448, 448, seed=41, device="cuda")
    cfg = fc.CacheConfig(patch_size=14)
    monkeypatch.setenv("FC_PDL", "0")
    ref = fc.FreqCacheEngine(streams, 448, 448, 14, fmt="rgb")
    monkeypatch.setenv("FC_PDL", "1")
    pdl = fc.FreqCacheEngine(streams, 448, 448, 14, fmt="rgb")
    oa = [ref.new_output(), ref.new_output()]
    ob = [pdl.new_output(), pdl.new_output()]
    for t in range(T):
        for eng, o in ((ref, oa), (pdl, ob)):
            eng.select_front(frames[t], cfg, o[t & 1], t & 1, refresh_shift=1)
            if t == T - 1 and eng is pdl:
                g = fc.StepGraph(lambda: eng.select_back(cfg, o[t & 1], t & 1, refresh_shift=1))
                g.replay()
            else:
                eng.select_back(cfg, o[t & 1], t & 1, refresh_shift=1)
        torch.cuda.synchronize()
        for name in ("reuse_idx", "recompute_idx", "src_map", "reuse_mask", "refresh_mask", "energy", "results"):
            assert torch.equal(getattr(oa[t & 1], name), getattr(ob[t & 1], name)), (t, name)
        assert torch.equal(ref.state, pdl.state), t


def test_gather_patches_matches_torch_patchify(cuda):
    """fc_gather_patches (config 4's recomputed-token pixels, straight from
    fp32 RGB frames to bf16) equals torch's patchify + cast + row gather bit
    for bit, including ragged, repeated and boundary token indices."""
    import torch
    from paper_2604_24391_b200.engine import gather_patches
    from paper_2604_24391_b200.vit import ViT, ViTConfig
    c = ViTConfig(image=112, patch=14, width=64, mlp=128, heads=2, layers=1)
    model = ViT(c).cuda().eval()
    g = torch.Generator(device="cuda").manual_seed(4)
    frames = torch.rand((5, 112, 112, 3), generator=g, device="cuda")
    n = c.tokens
    idx = torch.tensor([0, n - 1, n, 3 * n + 17, 5 * n - 1, 17, 17, 2 * n + 33], dtype=torch.int64, device="cuda")
    got = gather_patches(frames, 14, idx)
    ref = model.patches(frames.to(torch.bfloat16)).reshape(-1, 3 * 14 * 14).index_select(0, idx)
    assert torch.equal(got.view(torch.int16), ref.view(torch.int16))


def test_c_abi_from_plain_c(cuda):
    """examples/select_c.c: the C ABI driven from C99 through cudart (no
    Python, no torch) — two shifted 448 x 448 RGB streams; the displacement
    and every reused token's source must come out as the shift dictates."""
    import subprocess
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    r = subprocess.run(["make", "-s", "-C", str(root / "examples"), "select_c"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(root / "examples" / "select_c")], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().endswith("OK")
    assert "di_patches 1 " in r.stdout and "di_patches 2 " in r.stdout
