"""BASELINE config 5 at its full per-GPU size (the bench workload: 512 streams
of 448x448x3 fp32, P = 14, 1024 tokens, 1152-wide bf16 hidden states), checked
through size-independent properties:

* batch invariance — each stream's decision in the 512-stream batch is
  bit-identical to the same stream decided in a 5-stream batch;
* decision invariants for every stream (``_assert_decision``,
  fusion.py:245-262: |reuse| = K_final = min(K_reuse, K_cand), flush => 0,
  recompute = row-major complement) and agreement of the splice map with
  the reuse list, the displacement and the recompute order;
* the in-place ping-pong splice equals the out-of-place gather the decision
  defines, bit for bit, for all 512 streams (tokens and ages);
* oracle parity on a sample of streams at two steps.
"""

import numpy as np
import pytest

from oracle import freqcache_oracle as O
from oracle.parity import ParityReport, compare

pytestmark = pytest.mark.gpu

S, H, P, D, T = 512, 448, 14, 1152, 3
N = (H // P) ** 2


def test_config5_full_size_properties(cuda):
    import torch
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200.api import decision_from_device
    from paper_2604_24391_b200.synth import torch_stream_frames

    dev = torch.device("cuda")
    frames = torch.empty((T, S, H, H, 3), dtype=torch.float32, device=dev)
    for c0 in range(0, S, 64):
        frames[:, c0:c0 + 64] = torch_stream_frames(64, T, H, H, seed=5000 + c0, device=dev)
    cfg = fc.CacheConfig(patch_size=P)
    eng = fc.FreqCacheEngine(S, H, H, P, fmt="rgb", device=dev)
    pick = [0, 1, 255, 300, 511]
    small = fc.FreqCacheEngine(len(pick), H, H, P, fmt="rgb", device=dev)
    idx = torch.tensor(pick, device=dev)

    g = torch.Generator(device=dev).manual_seed(3000)
    cache = torch.empty((2, S, N, D), dtype=torch.bfloat16, device=dev)
    cache[0].normal_(generator=g)
    ages = torch.zeros((2, S, N), dtype=torch.int64, device=dev)
    fresh = torch.empty((S, N, D), dtype=torch.bfloat16, device=dev).normal_(generator=g)
    state = fc.SpliceState(cache, ages)
    oc = O.OracleConfig(patch_size=P, refresh_shift=1)
    rep = ParityReport()
    rows = cols = H // P
    grid_i = np.arange(N) // cols
    grid_j = np.arange(N) % cols

    for t in range(T):
        out = eng.select(frames[t], cfg, refresh_shift=1)
        ref = small.select(frames[t][idx].contiguous(), cfg, refresh_shift=1)
        # batch invariance (bit-exact)
        assert torch.equal(out.results[idx], ref.results)
        assert torch.equal(out.reuse_idx[idx], ref.reuse_idx)
        assert torch.equal(out.recompute_idx[idx], ref.recompute_idx)
        assert torch.equal(out.src_map[idx], ref.src_map)
        assert torch.equal(out.energy[idx], ref.energy)

        # splice: in place (ping-pong) vs the out-of-place gather of the same map
        before_tok, before_age = state.current()
        before_tok, before_age = before_tok.clone(), before_age.clone()
        state.step(out.src_map, fresh)
        after_tok, after_age = state.current()
        src = out.src_map.long()
        reused = src >= 0
        gathered = torch.gather(before_tok, 1, src.clamp(min=0)[..., None].expand(-1, -1, D))
        exp_tok = torch.where(reused[..., None], gathered, fresh)
        exp_age = torch.where(reused, torch.gather(before_age, 1, src.clamp(min=0)) + 1,
                              torch.zeros_like(before_age))
        assert torch.equal(after_tok.view(torch.int16), exp_tok.view(torch.int16))
        assert torch.equal(after_age, exp_age)
        del gathered, exp_tok, before_tok

        res = out.host_results()
        if t == 0:
            assert (res["cold"] == 1).all()
            continue
        assert (res["cold"] == 0).all() and (res["status"] == 0).all()
        ri, rc = out.reuse_idx.cpu().numpy(), out.recompute_idx.cpu().numpy()
        sm = out.src_map.cpu().numpy()
        for s in range(S):
            r = res[s]
            kf = int(r["k_final"])
            reuse = ri[s][ri[s] >= 0]
            rec = rc[s][rc[s] >= 0]
            assert len(reuse) == kf == min(int(r["k_reuse"]), int(r["k_candidate"]))
            if r["flushed"]:
                assert kf == 0 and int(r["k_candidate"]) == 0
            assert np.array_equal(np.sort(np.concatenate([reuse, rec])), np.arange(N))
            assert np.all(np.diff(rec) > 0)
            dip, djp = int(r["di_patches"]), int(r["dj_patches"])
            m = np.empty(N, dtype=np.int64)
            m[reuse] = (grid_i[reuse] - dip) * cols + (grid_j[reuse] - djp)
            m[rec] = -(np.arange(len(rec)) + 1)   # recomputed: -(rank in the recompute order + 1)
            assert np.array_equal(sm[s].astype(np.int64), m)
        # oracle parity on a sample of streams
        f0, f1 = frames[t - 1][idx].cpu().numpy(), frames[t][idx].cpu().numpy()
        for k, s in enumerate(pick):
            d = decision_from_device(res[s], ri[s], rc[s], out.refresh_mask[s].cpu().numpy(), step=t)
            compare(d, O.decide(f0[k], f1[k], oc, step=t), oc, energies=out.energy[s].cpu().numpy(), rep=rep)
    assert rep.ok, rep.errors


def test_config5_full_size_shifted_inplace_splice(cuda):
    """The in-place splice copier at the bench size (512 streams x 1024 x
    1152 bf16) with every kind of stream in one batch — zero displacement
    (updated in place), shifted by up to one patch (ping-pong to the other
    buffer), flushed — over several steps, against the gather each step's
    map defines (tokens bit for bit, ages)."""
    import torch
    import paper_2604_24391_b200 as fc

    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(11)
    cache = torch.empty((2, S, N, D), dtype=torch.bfloat16, device=dev)
    cache[0].normal_(generator=g)
    ages = torch.zeros((2, S, N), dtype=torch.int64, device=dev)
    ages[0] = torch.randint(0, 9, (S, N), generator=g, device=dev)
    state = fc.SpliceState(cache, ages)
    cols = H // P
    ii = (torch.arange(N, device=dev) // cols)[None]
    jj = (torch.arange(N, device=dev) % cols)[None]
    for stepi in range(4):
        kind = torch.randint(0, 4, (S,), generator=g, device=dev)            # 0, 1: zero shift; 2: shifted; 3: flush
        dip = torch.where(kind == 2, torch.randint(-1, 2, (S,), generator=g, device=dev), 0)
        djp = torch.where(kind == 2, torch.randint(-1, 2, (S,), generator=g, device=dev), 0)
        si, sj = ii - dip[:, None], jj - djp[:, None]
        aligned = (si >= 0) & (si < cols) & (sj >= 0) & (sj < cols)
        reuse = aligned & (torch.rand((S, N), generator=g, device=dev) < 0.45) & (kind != 3)[:, None]
        rank = torch.cumsum((~reuse).to(torch.int32), dim=1) - 1
        src = torch.where(reuse, si * cols + sj, -(rank + 1)).to(torch.int32).contiguous()
        fresh = torch.empty((S, N, D), dtype=torch.bfloat16, device=dev).normal_(generator=g)
        before_tok, before_age = state.current()
        state.step(src, fresh)
        after_tok, after_age = state.current()
        s64 = src.long().clamp(min=0)
        exp_tok = torch.where(reuse[..., None], torch.gather(before_tok, 1, s64[..., None].expand(-1, -1, D)), fresh)
        exp_age = torch.where(reuse, torch.gather(before_age, 1, s64) + 1, torch.zeros_like(before_age))
        assert torch.equal(after_tok.view(torch.int16), exp_tok.view(torch.int16)), stepi
        assert torch.equal(after_age, exp_age), stepi
        del before_tok, exp_tok, after_tok
