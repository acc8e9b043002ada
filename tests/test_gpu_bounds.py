"""GPU tests: the splice kernels bounds-check every row's source on the
device, as the reference asserts inside ``step`` (fusion.py:488-490):
a malformed src_map row is skipped, FC_EBOUNDS lands in the status word, and
the facade raises ``AssertionError``.  Well-formed rows of the same call are
still spliced bit for bit."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _setup(B=3, N=64, D=96, seed=5):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    cache = torch.randn((B, N, D), generator=g, device="cuda").to(torch.bfloat16)
    ages = torch.randint(0, 5, (B, N), generator=g, device="cuda")
    fresh = torch.randn((B, N, D), generator=g, device="cuda").to(torch.bfloat16)
    src = torch.empty((B, N), dtype=torch.int32)
    for b in range(B):
        for p in range(N):
            src[b, p] = p if p % 3 else -(p // 3 + 1)   # reuse 2/3 in place, compact fresh for the rest
    return cache, ages, fresh, src.cuda()


def _expected(cache, ages, fresh, src, compact):
    import torch
    B, N = src.shape
    out = torch.empty_like(cache)
    oa = torch.empty_like(ages)
    for b in range(B):
        for p in range(N):
            s = int(src[b, p])
            if s >= 0:
                out[b, p], oa[b, p] = cache[b, s], ages[b, s] + 1
            else:
                out[b, p], oa[b, p] = fresh[b, -s - 1 if compact else p], 0
    return out, oa


@pytest.mark.parametrize("bad", ["cache_hi", "compact_hi"])
@pytest.mark.parametrize("fn", ["splice", "splice_bytes", "packed"])
def test_out_of_place_splice_flags_bad_source(cuda, bad, fn):
    import torch
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200.engine import splice_packed
    cache, ages, fresh, src = _setup()
    B, N, D = cache.shape
    good_src = src.clone()
    if bad == "cache_hi":
        src[1, 4] = N + 7                      # cache source past the grid
    else:
        src[2, 0] = -(N + 3)                   # compact index past the fresh rows
    if fn == "splice_bytes":                   # 2-byte rows: the byte-granular kernel
        cache, fresh = cache[..., :1].contiguous(), fresh[..., :1].contiguous()
    out = torch.zeros_like(cache)
    oa = torch.full_like(ages, -9)
    with pytest.raises(AssertionError, match="out of bounds|bounds"):
        if fn == "packed":
            vals = fresh.reshape(B * N, -1)
            offs = torch.arange(B, device="cuda", dtype=torch.int64) * N
            splice_packed(src, cache, ages, vals, offs, out, oa)
        else:
            fc.splice(src, cache, ages, fresh, out, oa, compact=True)
    exp, ea = _expected(cache, ages, fresh, good_src, compact=True)
    bad_mask = src != good_src
    ok = ~bad_mask
    assert torch.equal(out.view(torch.int16)[ok], exp.view(torch.int16)[ok])
    assert torch.equal(oa[ok], ea[ok])
    assert bool((oa[bad_mask] == -9).all())   # the malformed row is skipped


def test_cache_source_without_cache_is_flagged(cuda):
    import torch
    import paper_2604_24391_b200 as fc
    cache, ages, fresh, src = _setup(B=1, N=16)
    out, oa = torch.empty_like(cache), torch.empty_like(ages)
    with pytest.raises(AssertionError):
        fc.splice(src, None, None, fresh, out, oa, compact=True)
    # an all-fresh map (cold start) needs no cache
    cold = -(torch.arange(16, dtype=torch.int32, device="cuda") + 1).reshape(1, 16)
    fc.splice(cold, None, None, fresh, out, oa, compact=True)
    assert torch.equal(out.view(torch.int16), fresh.view(torch.int16))


def test_status_word_stays_asynchronous(cuda):
    import torch
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200.engine import check_status
    cache, ages, fresh, src = _setup()
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    out, oa = torch.empty_like(cache), torch.empty_like(ages)
    fc.splice(src, cache, ages, fresh, out, oa, compact=True, status=st)
    check_status(st)                           # well-formed: no error
    src[0, 5] = 10 ** 6
    fc.splice(src, cache, ages, fresh, out, oa, compact=True, status=st)
    assert int(st.item()) == 6                 # FC_EBOUNDS
    with pytest.raises(AssertionError):
        check_status(st)


@pytest.mark.parametrize("bulk", ["1", "0"])
def test_inplace_splice_flags_bad_source(cuda, monkeypatch, bulk):
    """Both in-place copiers (TMA bulk and the per-warp fallback) skip a
    malformed row, keep every other row exact and report FC_EBOUNDS through
    SpliceState.check()."""
    import torch
    import paper_2604_24391_b200 as fc
    monkeypatch.setenv("FC_SPLICE_BULK", bulk)
    B, N, D = 4, 64, 96
    g = torch.Generator(device="cuda").manual_seed(11)
    cache = torch.zeros((2, B, N, D), dtype=torch.bfloat16, device="cuda")
    cache[0] = torch.randn((B, N, D), generator=g, device="cuda").to(torch.bfloat16)
    ages = torch.zeros((2, B, N), dtype=torch.int64, device="cuda")
    st = fc.SpliceState(cache, ages)
    before = cache[0].clone()
    src = torch.empty((B, N), dtype=torch.int32)
    for b in range(B):
        for p in range(N):
            # stream 1 is shifted (ping-pong: every row copied), others in place
            s = (p - 1 if p % 8 else -(p // 8 + 1)) if b == 1 else (p if p % 4 else -(p // 4 + 1))
            src[b, p] = s
    good = src.clone()
    src[1, 9] = N + 1          # shifted stream: bad cache source
    src[3, 4] = -(N + 50)      # in-place stream: bad compact index
    fresh = torch.randn((B, N, D), generator=g, device="cuda").to(torch.bfloat16)
    st.step(src.cuda(), fresh, compact=True)
    with pytest.raises(AssertionError):
        st.check()
    st.check()                 # the status word was cleared
    tok, age = st.current()
    for b in range(B):
        for p in range(N):
            s = int(good[b, p])
            if (b, p) in ((1, 9), (3, 4)):
                continue
            exp = before[b, s] if s >= 0 else fresh[b, -s - 1]
            assert torch.equal(tok[b, p].view(torch.int16), exp.view(torch.int16)), (b, p)
            assert int(age[b, p]) == (1 if s >= 0 else 0), (b, p)


def test_bulk_copier_lane_slot_variants(cuda, monkeypatch):
    """Every (lanes, slots) instance of the TMA copier gives the same cache
    (the kernel chosen must be the one its shared memory was sized for)."""
    import torch
    import paper_2604_24391_b200 as fc
    B, N, D = 6, 256, 1152
    g = torch.Generator(device="cuda").manual_seed(2)
    base = torch.randn((B, N, D), generator=g, device="cuda").to(torch.bfloat16)
    fresh = torch.randn((B, N, D), generator=g, device="cuda").to(torch.bfloat16)
    rng = np.random.default_rng(4)
    src = np.empty((B, N), dtype=np.int32)
    for b in range(B):
        shift = b % 2
        k = 0
        for p in range(N):
            if rng.random() < 0.5 and p - shift >= 0:
                src[b, p] = p - shift
            else:
                k += 1
                src[b, p] = -k
    src_t = torch.from_numpy(src).cuda()
    results = []
    for nl in ("2", "4", "8", "16"):
        for sl in ("2", "3", "4"):
            monkeypatch.setenv("FC_SPLICE_BULK_NL", nl)
            monkeypatch.setenv("FC_SPLICE_BULK_SLOTS", sl)
            cache = torch.zeros((2, B, N, D), dtype=torch.bfloat16, device="cuda")
            cache[0] = base
            ages = torch.zeros((2, B, N), dtype=torch.int64, device="cuda")
            st = fc.SpliceState(cache, ages)
            st.step(src_t, fresh, compact=True)
            st.check()
            tok, age = st.current()
            results.append((tok.clone(), age.clone()))
    for tok, age in results[1:]:
        assert torch.equal(tok.view(torch.int16), results[0][0].view(torch.int16))
        assert torch.equal(age, results[0][1])
