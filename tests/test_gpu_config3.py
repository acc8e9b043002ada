"""BASELINE config 3: selection plus token splice at 256 streams.

Config-2 frames (448x448x3, P = 14, N = 1024 tokens), a seeded cache of bf16
hidden states 1024 x 1152 per stream ~ N(0, 1) and fresh states ~ N(0, 1),
reuse ratio swept through BudgetConfig(r, r) for r in 0.2 .. 0.8.  For every
stream the spliced tensor must equal, bit for bit, the gather the decision
defines (reused token <- cache[source], recomputed token <- fresh row), for
both the out-of-place and the in-place (ping-pong) splice; decisions of a few
streams are checked against the CPU oracle.
"""

import numpy as np
import pytest

from oracle import freqcache_oracle as O
from oracle.parity import ParityReport, compare

pytestmark = pytest.mark.gpu

S, H, P, D = 256, 448, 14, 1152


@pytest.fixture(scope="module")
def c3():
    import torch
    from paper_2604_24391_b200.synth import torch_stream_frames
    frames = torch.empty((2, S, H, H, 3), dtype=torch.float32, device="cuda")
    for c0 in range(0, S, 64):
        frames[:, c0:c0 + 64] = torch_stream_frames(64, 2, H, H, seed=3000 + c0, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(3000)
    cache = torch.randn((S, 1024, D), generator=g, device="cuda").to(torch.bfloat16)
    fresh = torch.randn((S, 1024, D), generator=g, device="cuda").to(torch.bfloat16)
    ages = torch.randint(0, 7, (S, 1024), generator=g, device="cuda", dtype=torch.int64)
    return frames, cache, fresh, ages


def _expected(src, cache, ages, fresh):
    """Gather the decision defines (fusion.py:481-504), on the device."""
    import torch
    reused = src >= 0
    idx = src.clamp(min=0).long()
    exp = torch.where(reused[..., None], torch.gather(cache, 1, idx[..., None].expand(-1, -1, D)), fresh)
    exp_ages = torch.where(reused, torch.gather(ages, 1, idx) + 1, torch.zeros_like(ages))
    return exp, exp_ages


@pytest.mark.parametrize("r", [0.2, 0.35, 0.5, 0.65, 0.8])
def test_config3_select_splice(cuda, c3, r):
    import torch
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200.api import decision_from_device
    frames, cache, fresh, ages = c3
    cfg = fc.CacheConfig(patch_size=P, budget=fc.BudgetConfig(r, r))
    eng = fc.FreqCacheEngine(S, H, H, P, fmt="rgb")
    eng.select(frames[0], cfg)
    out = eng.select(frames[1], cfg)
    res = out.host_results()
    assert (res["status"] == 0).all() and (res["cold"] == 0).all()
    N = eng.n_tokens
    kf = res["k_final"]
    assert (kf <= np.floor(r * N)).all()                      # K_final = min(K_reuse, K_cand)
    src = out.src_map
    assert torch.equal((src >= 0).sum(1).cpu(), torch.from_numpy(kf.astype(np.int64)))

    # out-of-place splice, every stream against the gather it must equal
    exp, exp_ages = _expected(src, cache, ages, fresh)
    o = torch.empty_like(cache)
    oa = torch.empty_like(ages)
    fc.splice(src, cache, ages, fresh, o, oa)
    assert torch.equal(o.view(torch.int16), exp.view(torch.int16))
    assert torch.equal(oa, exp_ages)

    # in-place ping-pong splice gives the same tensors
    pp = torch.empty((2, S, N, D), dtype=torch.bfloat16, device="cuda")
    pa = torch.empty((2, S, N), dtype=torch.int64, device="cuda")
    pp[0].copy_(cache)
    pa[0].copy_(ages)
    st = fc.SpliceState(pp, pa)
    st.step(src, fresh)
    cur, cur_ages = st.current()
    assert torch.equal(cur.view(torch.int16), exp.view(torch.int16))
    assert torch.equal(cur_ages, exp_ages)

    # decisions of three streams against the CPU oracle
    oc = O.OracleConfig(patch_size=P, alpha_min=r, alpha_max=r)
    rep = ParityReport()
    ri, rc_, rm = out.reuse_idx.cpu().numpy(), out.recompute_idx.cpu().numpy(), out.refresh_mask.cpu().numpy()
    en = out.energy.cpu().numpy()
    for s in (0, 101, 255):
        d = decision_from_device(res[s], ri[s], rc_[s], rm[s], step=1)
        o_ = O.decide(frames[0, s].cpu().numpy(), frames[1, s].cpu().numpy(), oc, step=1)
        compare(d, o_, oc, energies=en[s], rep=rep)
    assert rep.ok, rep.errors
    print(f"config 3, target reuse {r}: achieved {kf.mean() / N:.3f} "
          f"(min {kf.min() / N:.3f}, max {kf.max() / N:.3f}); flushed {res['flushed'].mean():.3f}")
