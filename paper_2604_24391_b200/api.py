"""Drop-in entry points with the reference's names and signatures.

``decide`` / ``step`` / ``populate_cache`` / ``run_sequence`` behave like
the reference's (fusion.py:121-242, 450-572) but execute on the GPU through
the C ABI: frames are uploaded, the sm_100a kernels compute the spectra,
masks, budget and top-K, and the token splice runs as a device gather.
``token_fn`` stays a host callable, exactly as in the reference (it is the
model that produces fresh token states).  Raises if the CUDA library or a
device is missing — there is no CPU fallback.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native as nat
from .engine import FreqCacheEngine, splice, splice_map
from .geometry import PatchGrid, coerce_frame, grid_shape
from .types import (
    DEFAULT_COST_MODEL,
    CacheDecision,
    ConstantFrameError,
    Displacement,
    EnergyMap,
    EntropyReading,
    SequenceReport,
    StepReport,
    TokenCache,
)

_ENGINES = {}


def _engine(h, w, p, fmt="gray64", batch=1):
    nat.lib()  # raises when the library or a CUDA device is missing
    key = (h, w, p, fmt, batch, torch.cuda.current_device())
    eng = _ENGINES.get(key)
    if eng is None:
        eng = FreqCacheEngine(batch, h, w, p, fmt=fmt)
        _ENGINES[key] = eng
    return eng


def _device_frame(a):
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    return t.to("cuda", non_blocking=False).unsqueeze(0)


def _raise_status(res):
    st = int(res["status"])
    if st == nat.FC_ENONFINITE:
        raise ValueError("frame contains non-finite values")
    if st == nat.FC_EPSI:
        raise ValueError(f"normalized entropy must lie in [0, 1], got {float(res['entropy_norm'])}")
    if st != nat.FC_OK:
        nat.check(st, "fc_select")


def decision_from_device(res, reuse_idx, recompute_idx, refresh_mask, step=0, timings=None):
    """fc_stream_result + index rows (host numpy) -> CacheDecision."""
    n = int(res["rows"]) * int(res["cols"])
    kf = int(res["k_final"])
    return CacheDecision(
        step=int(step),
        flushed=bool(res["flushed"]),
        sim_freq=float(res["sim_freq"]),
        displacement=Displacement(int(res["di"]), int(res["dj"]), int(res["di_patches"]),
                                  int(res["dj_patches"])),
        entropy=EntropyReading(float(res["entropy_raw"]), float(res["entropy_norm"]),
                               int(res["bin_count"])),
        alpha_t=float(res["alpha"]),
        k_reuse=int(res["k_reuse"]),
        k_candidate=int(res["k_candidate"]),
        k_final=kf,
        reuse_set=tuple(int(v) for v in reuse_idx[:kf]),
        recompute_set=tuple(int(v) for v in recompute_idx[: n - kf]),
        rows=int(res["rows"]),
        cols=int(res["cols"]),
        refresh_set=tuple(int(v) for v in np.flatnonzero(refresh_mask[:n])),
        diagnostic=nat.DIAG_TEXT[int(res["diagnostic"])],
        timings_us=dict(timings or {}),
    )


def stage_timings(prof):
    """Per-stage device microseconds of one profiled select in the
    reference's ``timings_us`` keys (fusion.py:137-221).  The kernels fuse
    stages, so each key holds the kernel that carries the stage's main work:
    transform = luma + block-DCT energies + row FFTs (K_A) and column FFTs
    (K_B, which also accumulates the similarity / entropy sums); migration =
    inverse row FFTs + impulse argmax (K_C); edge = energy statistics,
    refresh mask and token order (K_D1); budget = entropy / alpha / K (a few
    scalar instructions inside K_D; its sums are counted under transform);
    select = candidates, top-K and outputs (K_D)."""
    us = [1e3 * v for v in prof]
    return {"transform": int(us[0] + us[1]), "migration": int(us[2]), "edge": int(us[4]), "budget": 0,
            "select": int(us[3]), "device": int(sum(us))}


def _fetch(out, row=0):
    res = out.host_results()[row]
    ri = out.reuse_idx[row].cpu().numpy()
    rc = out.recompute_idx[row].cpu().numpy()
    rm = out.refresh_mask[row].cpu().numpy()
    return res, ri, rc, rm


def assert_decision(d, n):
    """In-run invariants of a decision (fusion.py:245-262)."""
    reuse, rec = set(d.reuse_set), set(d.recompute_set)
    assert not reuse & rec, "reuse and recompute sets overlap"
    assert len(reuse) + len(rec) == n, "sets do not partition the patches"
    assert d.k_final == len(d.reuse_set) == min(d.k_reuse, d.k_candidate), \
        "reuse count does not match the budget rule"
    if d.flushed:
        assert d.k_final == 0, "flushed step must reuse nothing"
    fresh = set(d.refresh_set)
    rows, cols = d.rows, d.cols
    dip, djp = d.displacement.di_patches, d.displacement.dj_patches
    for p in d.reuse_set:
        i, j = divmod(p, cols)
        assert 0 <= i - dip < rows and 0 <= j - djp < cols and p not in fresh, \
            f"reused patch {p} violates alignment/refresh safety"


# ------------------------------------------------------------------ decide --

def decide(prev, curr, cfg, *, step=0, parallel=False):
    """GPU decide (fusion.py:121-242).  ``parallel`` is accepted for API
    compatibility; the three analyses always run concurrently on the GPU."""
    prev = coerce_frame(prev)
    curr = coerce_frame(curr)
    if prev.shape != curr.shape:
        raise ValueError(f"frame shapes differ: {prev.shape} vs {curr.shape}")
    h, w = curr.shape
    rows, cols = grid_shape(h, w, cfg.patch_size)
    eng = _engine(h, w, cfg.patch_size)
    first = getattr(eng, "_aux_out", None)
    if first is None:
        first = eng._aux_out = eng.new_output()
    tp, tc = _device_frame(prev), _device_frame(curr)
    eng.reset()
    eng.select(tp, cfg, out=first)
    prof = []
    out = eng.select(tc, cfg, profile=prof)
    res0 = first.host_results()[0]
    _raise_status(res0)
    res, ri, rc, rm = _fetch(out)
    _raise_status(res)
    d = decision_from_device(res, ri, rc, rm, step=step, timings=stage_timings(prof))
    assert_decision(d, rows * cols)
    return d


# -------------------------------------------------------------------- step --

def default_token_fn(patch):
    """Reference stand-in model (fusion.py:97-101): 16-bin histogram over
    [0, 1] plus mean and variance.  Host callable, like any token_fn."""
    p = np.asarray(patch, dtype=np.float64)
    counts, _ = np.histogram(np.clip(p, 0.0, 1.0), bins=16, range=(0.0, 1.0))
    return np.concatenate([counts.astype(np.float64), [p.mean(), p.var()]])


def populate_cache(frame, patch_size, token_fn):
    """Cold start: token_fn on every patch, row-major, ages 0 (fusion.py:450-459)."""
    grid = PatchGrid(frame, patch_size)
    vecs = [np.asarray(token_fn(grid.patch(*grid.position(q))), dtype=np.float64).ravel()
            for q in range(grid.n_patches)]
    tokens = np.stack(vecs).reshape(grid.rows, grid.cols, -1)
    return TokenCache(tokens, np.zeros((grid.rows, grid.cols), dtype=np.int64))


def _fresh_rows(grid, order, token_fn):
    vecs = [np.asarray(token_fn(grid.patch(*grid.position(q))), dtype=np.float64).ravel()
            for q in order]
    return np.stack(vecs) if vecs else None


def step(cache, decision, curr, token_fn, cost_model=None):
    """Apply a decision: device gather of reused slots from their
    displacement-mapped source, fresh token_fn rows elsewhere
    (fusion.py:462-512)."""
    curr = coerce_frame(curr)
    cost_model = cost_model or DEFAULT_COST_MODEL
    rows, cols = decision.rows, decision.cols
    h, w = curr.shape
    if h % rows or w % cols or h // rows != w // cols:
        raise ValueError(f"decision grid {rows}x{cols} does not tile frame {h}x{w}")
    grid = PatchGrid(curr, h // rows)
    n = grid.n_patches
    reuse = () if cache is None or decision.flushed else tuple(decision.reuse_set)
    reused = set(reuse)
    order = [q for q in range(n) if q not in reused]
    fresh = _fresh_rows(grid, order, token_fn)
    dim = fresh.shape[1] if fresh is not None else cache.tokens.shape[2]
    dev = torch.device("cuda")
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    ridx = torch.tensor(reuse, dtype=torch.int32, device=dev) if reuse else None
    smap = splice_map(rows, cols, ridx, decision.displacement.di_patches,
                      decision.displacement.dj_patches, flag=flag).view(1, n)
    if int(flag.item()) != 0:
        raise AssertionError("reuse source out of bounds")
    if reuse:
        ctok = torch.from_numpy(np.ascontiguousarray(cache.tokens, dtype=np.float64)
                                .reshape(1, n, -1)).to(dev)
        cage = torch.from_numpy(np.ascontiguousarray(cache.ages, dtype=np.int64).reshape(1, n)).to(dev)
    else:
        ctok = cage = None
    fr = torch.from_numpy(fresh).to(dev).view(1, -1, dim) if fresh is not None else \
        torch.zeros((1, 1, dim), dtype=torch.float64, device=dev)
    out = torch.empty((1, n, dim), dtype=torch.float64, device=dev)
    ages = torch.empty((1, n), dtype=torch.int64, device=dev)
    splice(smap, ctok, cage, fr, out, ages, compact=True)
    tokens = out.cpu().numpy().reshape(rows, cols, dim)
    new_ages = ages.cpu().numpy().reshape(rows, cols)
    n_rec = n - len(reused)
    report = StepReport(step=decision.step, n_reused=len(reused), n_recomputed=n_rec,
                        latency_model_ms=cost_model.latency_ms(n_rec))
    return TokenCache(tokens, new_ages), report


# ------------------------------------------------------------ run_sequence --

def run_sequence(frames, cfg, token_fn=default_token_fn, cost_model=None, parallel=False):
    """Sequence driver (fusion.py:534-572).  The previous frame's spectrum and
    the token cache stay on the device between steps, so each frame is
    transformed once and tokens never round-trip through the host."""
    if len(frames) < 2:
        raise ValueError("need at least 2 frames")
    frames = [coerce_frame(f) for f in frames]
    shape = frames[0].shape
    for t, f in enumerate(frames):
        if f.shape != shape:
            raise ValueError(f"frame at step {t}: dimension mismatch {f.shape} vs {shape}")
    cost_model = cost_model or DEFAULT_COST_MODEL
    h, w = shape
    p = cfg.patch_size
    rows, cols = grid_shape(h, w, p)
    n = rows * cols
    eng = FreqCacheEngine(1, h, w, p, fmt="gray64")
    aux = eng.new_output()
    cache = populate_cache(frames[0], p, token_fn)
    dim = cache.tokens.shape[2]
    dev = eng.device
    tokens = torch.from_numpy(cache.tokens.reshape(1, n, dim).copy()).to(dev)
    ages = torch.zeros((1, n), dtype=torch.int64, device=dev)
    eng.select(_device_frame(frames[0]), cfg, out=aux)
    _raise_status(aux.host_results()[0])
    decisions, reports = [], []
    for t in range(1, len(frames)):
        prof = []
        out = eng.select(_device_frame(frames[t]), cfg, profile=prof)
        res, ri, rc, rm = _fetch(out)
        _raise_status(res)
        d = decision_from_device(res, ri, rc, rm, step=t, timings=stage_timings(prof))
        assert_decision(d, n)
        grid = PatchGrid(frames[t], p)
        fresh = _fresh_rows(grid, d.recompute_set, token_fn)
        fr = torch.from_numpy(fresh).to(dev).view(1, -1, dim) if fresh is not None else \
            torch.zeros((1, 1, dim), dtype=torch.float64, device=dev)
        new_tokens = torch.empty_like(tokens)
        new_ages = torch.empty_like(ages)
        splice(out.src_map, tokens, ages, fr, new_tokens, new_ages, compact=True)
        tokens, ages = new_tokens, new_ages
        n_rec = n - d.k_final
        decisions.append(d)
        reports.append(StepReport(step=t, n_reused=d.k_final, n_recomputed=n_rec,
                                  latency_model_ms=cost_model.latency_ms(n_rec)))
    total_reused = sum(d.k_final for d in decisions)
    mean_latency = sum(r.latency_model_ms for r in reports) / len(reports)
    baseline = cost_model.latency_ms(n)
    return SequenceReport(
        n_frames=len(frames), n_tokens=n, decisions=decisions, step_reports=reports,
        mean_reuse_ratio=total_reused / (len(decisions) * n), mean_latency_ms=mean_latency,
        baseline_latency_ms=baseline, speedup=baseline / mean_latency,
        flush_count=sum(1 for d in decisions if d.flushed),
    )


# --------------------------------------------------------- stage functions --

def _stage_patch(h, w):
    """A plan patch size for stage calls that do not fix one: the largest
    divisor of gcd(H, W) in [2, 32] (only the pixel results are used)."""
    g = math.gcd(h, w)
    for p in range(min(32, g), 1, -1):
        if g % p == 0 and (h // p) * (w // p) <= 4096:
            return p
    raise nat.NativeError(f"no supported plan geometry for a {h}x{w} frame")


def patch_energy(grid):
    """High-pass block-DCT energy per patch on the GPU (edge_refresh.py:48-59)."""
    h, w = grid.frame.shape
    eng = _engine(h, w, grid.patch_size)
    e = eng.patch_energy(_device_frame(grid.frame))
    c = max(1, grid.patch_size // 4)
    return EnergyMap(e.cpu().numpy().reshape(grid.rows, grid.cols), grid.patch_size, c)


def phase_correlation(prev, curr, patch_size=1):
    """Cyclic displacement of curr w.r.t. prev on the GPU (migration.py:108-125)."""
    prev = coerce_frame(prev)
    curr = coerce_frame(curr)
    if prev.shape != curr.shape:
        raise ValueError(f"frame shapes differ: {prev.shape} vs {curr.shape}")
    from .types import CacheConfig, BudgetConfig
    h, w = curr.shape
    p = _stage_patch(h, w)
    eng = _engine(h, w, p)
    first = getattr(eng, "_aux_out", None)
    if first is None:
        first = eng._aux_out = eng.new_output()
    cfg = CacheConfig(patch_size=p, budget=BudgetConfig(0.5, 0.5))
    eng.reset()
    eng.select(_device_frame(prev), cfg, out=first)
    out = eng.select(_device_frame(curr), cfg)
    res0 = first.host_results()[0]
    if int(res0["status"]) == nat.FC_ENONFINITE:
        raise ValueError("frame contains non-finite values")
    res = out.host_results()[0]
    if int(res["status"]) == nat.FC_ENONFINITE:
        raise ValueError("frame contains non-finite values")
    if int(res["diagnostic"]) in (nat.FC_DIAG_DEGENERATE, nat.FC_DIAG_NO_TEXTURE):
        raise ConstantFrameError("no texture; displacement undefined")
    return Displacement.from_pixels(int(res["di"]), int(res["dj"]), patch_size)


# ------------------------------------------ array stage operators (GPU) ----

def _stage_ws(dev):
    ws = _STAGE_WS.get(dev)
    if ws is None:
        ws = torch.empty(nat.lib().fc_stage_workspace_bytes(), dtype=torch.uint8, device=dev)
        _STAGE_WS[dev] = ws
    return ws


_STAGE_WS = {}


def _dev_f64(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64)).ravel()).to("cuda")


def sim_freq(amp_prev, amp_curr):
    """Cosine of two amplitude grids, clamped to 1 (migration.py:87-105)."""
    from .engine import _ptr, _stream
    from .types import DegenerateSpectrumError
    a = np.asarray(amp_prev, dtype=np.float64)
    b = np.asarray(amp_curr, dtype=np.float64)
    if a.ravel().shape != b.ravel().shape:
        raise ValueError("amplitude grids must have equal dimensions")
    lib = nat.lib()
    ta, tb = _dev_f64(a), _dev_f64(b)
    out = torch.empty(3, dtype=torch.float64, device="cuda")
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    nat.check(lib.fc_amp_cosine(_ptr(ta), _ptr(tb), int(ta.numel()), _ptr(_stage_ws(ta.device)), _ptr(out),
                                _ptr(flags), _stream(ta.device)), "fc_amp_cosine")
    f = int(flags.item())
    if f & 1:
        raise ValueError("amplitude grids contain non-finite values")
    if f & 2:
        raise ValueError("amplitude grids must be nonnegative")
    dot, n2a, n2b = out.tolist()
    na, nb = math.sqrt(n2a), math.sqrt(n2b)
    if na == 0.0 or nb == 0.0:
        raise DegenerateSpectrumError("degenerate spectrum")
    return min(1.0, dot / (na * nb))


def spectral_entropy(amplitude, include_dc=True):
    """Normalised Shannon entropy of the power spectrum (budget.py:34-58)."""
    from .engine import _ptr, _stream
    from .types import DegenerateSpectrumError
    a = np.asarray(amplitude, dtype=np.float64)
    if a.size < 2:
        raise ValueError("amplitude grid must have at least 2 bins")
    lib = nat.lib()
    ta = _dev_f64(a)
    out = torch.empty(2, dtype=torch.float64, device="cuda")
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    nat.check(lib.fc_spectral_sums(_ptr(ta), int(ta.numel()), 1 if include_dc else 0, _ptr(_stage_ws(ta.device)),
                                   _ptr(out), _ptr(flags), _stream(ta.device)), "fc_spectral_sums")
    f = int(flags.item())
    if f & 1:
        raise ValueError("amplitude grid contains non-finite values")
    if f & 2:
        raise ValueError("amplitude grid must be nonnegative")
    total, plogp = out.tolist()
    if total <= 0.0:
        raise DegenerateSpectrumError("degenerate spectrum")
    raw = -plogp + 0.0
    return EntropyReading(raw, raw / math.log(a.size), a.size)


def refresh_mask(energy, sensitivity):
    """Population mean/std threshold, strict '>' (edge_refresh.py:62-73)."""
    from .engine import _ptr, _stream
    from .types import RefreshMask
    e = np.asarray(energy.energies, dtype=np.float64)
    lib = nat.lib()
    te = _dev_f64(e)
    mask = torch.empty(te.numel(), dtype=torch.uint8, device="cuda")
    stats = torch.empty(3, dtype=torch.float64, device="cuda")
    nat.check(lib.fc_refresh_mask(_ptr(te), int(te.numel()), float(sensitivity), _ptr(_stage_ws(te.device)),
                                  _ptr(mask), _ptr(stats), _stream(te.device)), "fc_refresh_mask")
    mu, sd, _ = stats.tolist()
    return RefreshMask(mask.cpu().numpy().astype(bool).reshape(e.shape), mu, sd, float(sensitivity))


def topk_ascending(candidates, energies, k):
    """First k candidates by ascending energy, ties row-major (fusion.py:104-115)."""
    from .engine import _ptr, _stream
    cand = np.asarray(candidates, dtype=np.int64).ravel()
    if cand.size == 0 or k <= 0:
        return ()
    lib = nat.lib()
    e = _dev_f64(energies)
    tc = torch.from_numpy(cand).to("cuda")
    kout = min(int(k), cand.size)
    out = torch.empty(kout, dtype=torch.int64, device="cuda")
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    nat.check(lib.fc_topk_ascending(_ptr(tc), int(cand.size), _ptr(e), int(e.numel()), int(k), _ptr(out),
                                    _ptr(flags), _stream(tc.device)), "fc_topk_ascending")
    if int(flags.item()) & 4:
        raise IndexError("candidate index out of range")
    return tuple(int(v) for v in out.cpu().tolist())


def sim_spatial(prev, curr, grid, token_fn):
    """Mean position-wise cosine of patch embeddings — the visual-domain
    baseline score (migration.py:53-84).  ``token_fn`` is host model code as
    in the reference; the cosines run on the GPU (``fc_row_cosines``, fp64).
    Zero-norm pairs contribute 0 and trigger a RuntimeWarning."""
    import warnings

    from .engine import row_cosines
    from .geometry import validate_frame

    prev = validate_frame(prev)
    curr = validate_frame(curr)
    if prev.shape != curr.shape:
        raise ValueError(f"frame shapes differ: {prev.shape} vs {curr.shape}")
    pos = [(i, j) for i in range(grid.rows) for j in range(grid.cols)]
    a = np.stack([np.asarray(token_fn(grid.patch(i, j, prev)), dtype=np.float64).ravel() for i, j in pos])
    b = np.stack([np.asarray(token_fn(grid.patch(i, j, curr)), dtype=np.float64).ravel() for i, j in pos])
    cos = row_cosines(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
    degenerate = int(((np.linalg.norm(a, axis=1) == 0.0) | (np.linalg.norm(b, axis=1) == 0.0)).sum())
    if degenerate:
        warnings.warn(f"{degenerate} patch position(s) had zero-norm embeddings and contributed 0 similarity",
                      RuntimeWarning, stacklevel=2)
    total = 0.0
    for c in cos:
        total += float(c)
    return total / grid.n_patches
