"""CPU oracle for the FreqCache decision path — TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy/scipy, the per-step token-cache
decision of the reference (``/root/reference/pkg/src/freqcache``) so the
CUDA path can be checked against it.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import
it, and only as the checker / the timed CPU baseline.  The product path
(``paper_2604_24391_b200``) never imports it.

Pinning: the restatement is checked against (a) golden decisions produced by
running the reference itself in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/golden_*.json``) and (b) the
known-answer values the reference's own tests hold (see
``tests/test_oracle_golden.py``).

Each function names the reference lines it follows.  Additions that are not
in the reference are marked as such:
  * ``luma_f64``            — fp32 RGB -> gray adapter (BASELINE configs are RGB)
  * ``refresh_shift``       — config-2's opt-in "flush on shift > k patches"
  * ``decision_margins``    — per-token / per-step distances to the decision
                              thresholds, used by the parity checker.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.fft
from scipy.special import xlogy

# fusion.py / migration.py constants
CROSS_POWER_EPS = 1e-12          # migration.py:14
LUMA = (0.299, 0.587, 0.114)     # frameio.py:26

DIAG_DEGENERATE = "degenerate spectrum"                  # errors.py:4, migration.py:103
DIAG_NO_TEXTURE = "no texture; displacement undefined"   # fusion.py:148


class _Degenerate(ValueError):
    pass


class _NoTexture(ValueError):
    pass


@dataclass
class OracleConfig:
    """CacheConfig + BudgetConfig (fusion.py:52-67, budget.py:12-24)."""

    tau_mig: float = 0.12
    edge_lambda: float = 0.25
    alpha_min: float = 0.08
    alpha_max: float = 0.5
    patch_size: int = 16
    refresh_shift: int | None = None   # NOT in the reference (config 2 rule)


@dataclass
class OracleDecision:
    """Field-for-field CacheDecision (fusion.py:70-94) plus diagnostics."""

    step: int
    flushed: bool
    sim_freq: float
    displacement: tuple          # (di, dj, di_patches, dj_patches)
    entropy: tuple               # (raw, normalized, bin_count)
    alpha_t: float
    k_reuse: int
    k_candidate: int
    k_final: int
    reuse_set: tuple
    recompute_set: tuple
    rows: int
    cols: int
    refresh_set: tuple
    diagnostic: str | None = None
    # extras for parity (not part of the reference decision)
    energies: np.ndarray = field(default=None, repr=False)
    energy_mean: float = 0.0
    energy_std: float = 0.0
    threshold: float = 0.0
    align: np.ndarray = field(default=None, repr=False)
    peak: float = 0.0
    runner_up: float = 0.0


# ----------------------------------------------------------------- frames --

def luma_f64(rgb):
    """fp32 RGB (H,W,3) -> float64 gray, BT.601 weights, evaluated as
    ``(0.299*R + 0.587*G) + 0.114*B`` left to right (frameio.py:85-88; the
    reference divides by 255 there because its input is uint8 — ours is
    already in [0,1])."""
    a = np.asarray(rgb)
    r = a[..., 0].astype(np.float64)
    g = a[..., 1].astype(np.float64)
    b = a[..., 2].astype(np.float64)
    return LUMA[0] * r + LUMA[1] * g + LUMA[2] * b


def as_gray(frame):
    """Accept (H,W) gray or (H,W,3) RGB; validate like frame.py:6-15."""
    a = np.asarray(frame)
    if a.ndim == 3 and a.shape[-1] == 3:
        a = luma_f64(a)
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError(f"frame must be 2D, got shape {a.shape}")
    if a.shape[0] < 1 or a.shape[1] < 1:
        raise ValueError(f"frame dimensions must be >= 1, got {a.shape}")
    if not np.all(np.isfinite(a)):
        raise ValueError("frame contains non-finite values")
    return a


def grid_dims(shape, p):
    """PatchGrid geometry checks (frame.py:27-41)."""
    p = int(p)
    if p < 2:
        raise ValueError(f"patch size must be >= 2, got {p}")
    h, w = shape
    if h % p or w % p:
        raise ValueError(f"patch size {p} does not divide frame dimensions {h}x{w}")
    return h // p, w // p


# ------------------------------------------------------------- module II --

def cutoff(p):
    """edge_refresh.py:9-11."""
    return max(1, int(p) // 4)


def block_energy(gray, p):
    """High-pass orthonormal block-DCT energy per patch (edge_refresh.py:48-59)."""
    h, w = gray.shape
    rows, cols = h // p, w // p
    blocks = gray.reshape(rows, p, cols, p).transpose(0, 2, 1, 3)
    coef = scipy.fft.dctn(blocks, axes=(-2, -1), norm="ortho")
    c = cutoff(p)
    coef[..., :c, :c] = 0.0
    return np.sum(coef * coef, axis=(-2, -1))


def refresh(energies, lam):
    """Population mean/std threshold, strict '>' (edge_refresh.py:62-73)."""
    mu = float(energies.mean())
    sd = float(energies.std())
    thr = mu + float(lam) * sd
    return energies > thr, mu, sd, thr


# ------------------------------------------------------------ module III --

def entropy(amp):
    """Normalised Shannon entropy of |F|^2 with DC included (budget.py:34-58)."""
    pw = (amp * amp).ravel()
    tot = float(pw.sum())
    if tot <= 0.0:
        raise _Degenerate(DIAG_DEGENERATE)
    prob = pw / tot
    raw = float(-np.sum(xlogy(prob, prob))) + 0.0
    return raw, raw / math.log(prob.size), prob.size


def budget(psi, amin, amax, n):
    """alpha = amin + (amax-amin) e^-psi ; K = floor(alpha N) (budget.py:61-75)."""
    psi = float(psi)
    if not 0.0 <= psi <= 1.0:
        raise ValueError(f"normalized entropy must lie in [0, 1], got {psi}")
    if int(n) < 1:
        raise ValueError(f"token count must be >= 1, got {n}")
    alpha = amin + (amax - amin) * math.exp(-psi)
    return alpha, int(math.floor(alpha * int(n)))


# ------------------------------------------------------------- module I ---

def similarity(amp_p, amp_c):
    """Amplitude cosine clamped to 1 (migration.py:87-105)."""
    a = amp_p.ravel()
    b = amp_c.ravel()
    na = float(np.linalg.norm(a))
    nb = float(np.linalg.norm(b))
    if na == 0.0 or nb == 0.0:
        raise _Degenerate(DIAG_DEGENERATE)
    return min(1.0, float(np.dot(a, b)) / (na * nb))


def canon(d, n):
    """migration.py:137-138."""
    return d - n if 2 * d >= n else d


def to_patches(d, p):
    """Half-patch rounds toward zero (migration.py:41-45)."""
    d = int(d)
    s = 1 if d >= 0 else -1
    return s * ((2 * abs(d) + int(p) - 1) // (2 * int(p)))


def correlation_response(spec_p, spec_c):
    """Normalised cross-power -> real inverse DFT (migration.py:128-134)."""
    x = spec_p * np.conj(spec_c)
    x /= np.abs(x) + CROSS_POWER_EPS
    return scipy.fft.ifft2(x).real


def peak_displacement(resp):
    """argmax with the reference tie rule (migration.py:141-159)."""
    h, w = resp.shape
    top = resp.max()
    best = None
    for pi, pj in np.argwhere(resp == top):
        di = canon(int(-pi) % h, h)
        dj = canon(int(-pj) % w, w)
        key = (abs(di) + abs(dj), int(pi), int(pj))
        if best is None or key < best[0]:
            best = (key, di, dj)
    return best[1], best[2]


def align_mask(dip, djp, rows, cols):
    """Rectangle of slots whose shifted source exists (migration.py:162-176)."""
    m = np.zeros((rows, cols), dtype=bool)
    r0, r1 = max(0, dip), min(rows, rows + dip)
    c0, c1 = max(0, djp), min(cols, cols + djp)
    if r0 < r1 and c0 < c1:
        m[r0:r1, c0:c1] = True
    return m


def topk_ascending(cand, energies, k):
    """Ascending (E, index) order, first k (fusion.py:104-115)."""
    cand = np.asarray(cand, dtype=np.int64)
    if cand.size == 0 or k <= 0:
        return ()
    e = np.asarray(energies, dtype=np.float64).ravel()
    order = np.lexsort((cand, e[cand]))
    return tuple(int(cand[o]) for o in order[: min(int(k), cand.size)])


# ------------------------------------------------------------- decision ---

def decide(prev, curr, cfg: OracleConfig, step=0):
    """Algorithm 1 with the reference's failure semantics (fusion.py:121-242).

    ``prev``/``curr`` may be gray (H,W) or fp32 RGB (H,W,3).  With
    ``cfg.refresh_shift`` set (NOT in the reference), a step whose quantised
    displacement exceeds it in either axis is flushed with no diagnostic.
    """
    prev = as_gray(prev)
    curr = as_gray(curr)
    if prev.shape != curr.shape:
        raise ValueError(f"frame shapes differ: {prev.shape} vs {curr.shape}")
    p = int(cfg.patch_size)
    rows, cols = grid_dims(curr.shape, p)
    n = rows * cols
    h, w = curr.shape

    spec_p = scipy.fft.fft2(prev)
    spec_c = scipy.fft.fft2(curr)
    amp_p = np.abs(spec_p)
    amp_c = np.abs(spec_c)

    # Module I (fusion.py:144-151); an exception discards every stage value
    mig_err = None
    sim, disp, align, peak, runner = 0.0, (0, 0, 0, 0), None, 0.0, 0.0
    try:
        s = similarity(amp_p, amp_c)
        if np.ptp(prev) == 0.0 or np.ptp(curr) == 0.0:
            raise _NoTexture(DIAG_NO_TEXTURE)
        resp = correlation_response(spec_p, spec_c)
        di, dj = peak_displacement(resp)
        flat = np.sort(resp.ravel())
        d = (di, dj, to_patches(di, p), to_patches(dj, p))
        sim, disp = s, d
        align = align_mask(d[2], d[3], rows, cols)
        peak, runner = float(flat[-1]), float(flat[-2]) if flat.size > 1 else 0.0
    except (_Degenerate, _NoTexture) as exc:
        mig_err = exc

    # Module II (fusion.py:153-157) — never fails
    energies = block_energy(curr, p)
    fresh, mu, sd, thr = refresh(energies, cfg.edge_lambda)
    refresh_set = tuple(int(q) for q in np.flatnonzero(fresh.ravel()))

    # Module III (fusion.py:159-163)
    bud_err = None
    ent, alpha, k_reuse = (0.0, 0.0, h * w), 0.0, 0
    try:
        e = entropy(amp_c)
        a, k = budget(e[1], cfg.alpha_min, cfg.alpha_max, n)
        ent, alpha, k_reuse = e, a, k
    except _Degenerate as exc:
        bud_err = exc

    failure = mig_err if mig_err is not None else bud_err
    shift_flush = (
        cfg.refresh_shift is not None and failure is None
        and max(abs(disp[2]), abs(disp[3])) > cfg.refresh_shift
    )
    if failure is not None:
        flushed, diag, k_cand, k_final, reuse = True, str(failure), 0, 0, ()
    elif sim < cfg.tau_mig or shift_flush:           # migration.py:179-185
        flushed, diag, k_cand, k_final, reuse = True, None, 0, 0, ()
    else:
        flushed, diag = False, None
        cand = np.flatnonzero((align & ~fresh).ravel())
        k_cand = int(cand.size)
        k_final = min(k_reuse, k_cand)
        reuse = topk_ascending(cand, energies, k_final)
    keep = np.ones(n, dtype=bool)
    keep[list(reuse)] = False
    recompute = tuple(int(q) for q in np.flatnonzero(keep))

    return OracleDecision(
        step=int(step), flushed=flushed, sim_freq=float(sim),
        displacement=tuple(int(v) for v in disp),
        entropy=(float(ent[0]), float(ent[1]), int(ent[2])),
        alpha_t=float(alpha), k_reuse=int(k_reuse), k_candidate=int(k_cand),
        k_final=int(k_final), reuse_set=reuse, recompute_set=recompute,
        rows=rows, cols=cols, refresh_set=refresh_set, diagnostic=diag,
        energies=energies.ravel(), energy_mean=mu, energy_std=sd, threshold=thr,
        align=None if align is None else align.ravel(), peak=peak,
        runner_up=runner,
    )


# ---------------------------------------------------------------- splice --

def splice(cache_tokens, cache_ages, decision, fresh_rows):
    """Token splice (fusion.py:462-512) on flat [N, D] arrays.

    Reused slot p=(i,j) takes cache row (i-dip, j-djp) and age+1; every other
    slot takes the next row of ``fresh_rows`` in row-major recompute order
    (the order ``step`` calls ``token_fn``) with age 0.  ``cache_tokens=None``
    or a flushed decision recomputes everything.
    """
    rows, cols = decision.rows, decision.cols
    n = rows * cols
    disp = decision.displacement
    dip, djp = (disp.di_patches, disp.dj_patches) if hasattr(disp, "di_patches") else (disp[2], disp[3])
    reuse = () if cache_tokens is None or decision.flushed else decision.reuse_set
    out = np.empty((n,) + np.asarray(fresh_rows).shape[1:], dtype=np.asarray(fresh_rows).dtype)
    ages = np.zeros(n, dtype=np.int64)
    reused = set()
    for q in reuse:
        i, j = divmod(int(q), cols)
        si, sj = i - dip, j - djp
        assert 0 <= si < rows and 0 <= sj < cols
        out[q] = cache_tokens[si * cols + sj]
        ages[q] = cache_ages[si * cols + sj] + 1
        reused.add(int(q))
    nxt = 0
    for q in range(n):
        if q in reused:
            continue
        out[q] = fresh_rows[nxt]
        nxt += 1
    return out, ages


# --------------------------------------------------------------- margins --

def decision_margins(d: OracleDecision, cfg: OracleConfig):
    """Distances of every discrete choice from its threshold.

    Returns a dict of per-step relative margins and per-token arrays; the
    parity checker exempts a choice whose margin is <= 1e-4.
    """
    e = d.energies
    thr = d.threshold
    scale = max(abs(thr), 1e-300)
    refresh_margin = np.abs(e - thr) / scale
    mean_e = float(e.mean()) if e.size else 0.0
    floor = 1e-6 * mean_e
    topk_margin = np.full(e.shape, np.inf)
    boundary = None
    if not d.flushed and 0 < d.k_final < d.k_candidate:
        # candidates ranked: boundary between the K-th and (K+1)-th energies
        cand = [q for q in range(e.size) if d.align[q] and q not in set(d.refresh_set)]
        ranked = sorted(cand, key=lambda q: (e[q], q))
        ek = e[ranked[d.k_final - 1]]
        ek1 = e[ranked[d.k_final]]
        boundary = (ek, ek1)
        b = 0.5 * (ek + ek1)
        topk_margin = (np.abs(e - b) - floor) / max(b, 1e-300)
        # both boundary tokens are within half the gap
        gap_rel = (ek1 - ek - 2 * floor) / max(ek1, 1e-300)
        topk_margin = np.minimum(topk_margin, np.where(
            (e == ek) | (e == ek1), gap_rel, np.inf))
    n = d.rows * d.cols
    an = d.alpha_t * n
    # K = floor(alpha N) flips when alpha N crosses an integer
    k_margin = min(an - math.floor(an), math.floor(an) + 1 - an) / an if an > 0 else math.inf
    disp_margin = (d.peak - d.runner_up) / abs(d.peak) if d.peak != 0 else 0.0
    gate_margin = abs(d.sim_freq - cfg.tau_mig) / max(cfg.tau_mig, 1e-300)
    return {
        "refresh": refresh_margin,
        "topk": topk_margin,
        "topk_boundary": boundary,
        "k": k_margin,
        "disp": disp_margin,
        "gate": gate_margin,
        "energy_floor": floor,
        "psi_one": abs(d.entropy[1] - 1.0),
    }


# ---------------------------------------------------- comparison baselines --
# compare.py: the two position-wise policies the paper compares against.

def position_cosines(prev_vecs, curr_vecs):
    """Row-wise cosine, zero-norm rows score 0 (compare.py:28-38)."""
    a = np.asarray(prev_vecs, dtype=np.float64)
    b = np.asarray(curr_vecs, dtype=np.float64)
    num = np.einsum("nd,nd->n", a, b)
    den = np.linalg.norm(a, axis=1) * np.linalg.norm(b, axis=1)
    out = np.zeros(a.shape[0])
    ok = den > 0.0
    out[ok] = num[ok] / den[ok]
    return out


def patch_pixels(gray, p):
    """Raw-pixel token stack in row-major patch order (compare.py:24-25,41-47)."""
    rows, cols = grid_dims(gray.shape, p)
    return gray.reshape(rows, p, cols, p).swapaxes(1, 2).reshape(rows * cols, p * p)


def patch_amplitudes(gray, p):
    """|fft2| of every patch, flattened (compare.py:50-52)."""
    rows, cols = grid_dims(gray.shape, p)
    blocks = gray.reshape(rows, p, cols, p).swapaxes(1, 2)
    return np.abs(scipy.fft.fft2(blocks, axes=(-2, -1))).reshape(rows * cols, -1)


def compare_cosines(prev, curr, p):
    """(visual, naive_freq) per-patch cosines for one frame pair
    (compare.py:90-95 with the default raw-pixel token_fn)."""
    a, b = as_gray(prev), as_gray(curr)
    return (position_cosines(patch_pixels(a, p), patch_pixels(b, p)),
            position_cosines(patch_amplitudes(a, p), patch_amplitudes(b, p)))


def latency_ms(full_ms, cached_ms, reuse_ratio, n_tokens, n_recompute):
    """CostModel.calibrated + latency_ms (fusion.py:34-44, 47-50): affine in
    the recomputed-token count, constants fitted in the reference's order."""
    n_full = float(n_tokens)
    n_cached = n_tokens * (1.0 - reuse_ratio)
    per = (full_ms - cached_ms) / (n_full - n_cached)
    return (full_ms - per * n_full) + per * n_recompute


def compare_domains(frames, cfg: OracleConfig, edge_labels=None, tau_visual=0.85, tau_naive_freq=0.85,
                    cost=(637.0, 401.0, 0.535, 196)):
    """Three-policy comparison over consecutive pairs (compare.py:55-114)."""
    if len(frames) < 2:
        raise ValueError("need at least 2 frames")
    gray = [as_gray(f) for f in frames]
    p = int(cfg.patch_size)
    rows, cols = grid_dims(gray[0].shape, p)
    n = rows * cols
    names = ("freqcache", "visual", "naive_freq")
    reused = dict.fromkeys(names, 0)
    false_reuse = dict.fromkeys(names, 0)
    lat = dict.fromkeys(names, 0.0)
    lm = lambda k: latency_ms(*cost, k)  # noqa: E731
    for t in range(1, len(gray)):
        d = decide(gray[t - 1], gray[t], cfg, step=t)
        vis, nf = compare_cosines(gray[t - 1], gray[t], p)
        sets = {"freqcache": set(d.reuse_set),
                "visual": set(np.flatnonzero(vis > tau_visual).tolist()),
                "naive_freq": set(np.flatnonzero(nf > tau_naive_freq).tolist())}
        labels = frozenset(edge_labels[t]) if edge_labels is not None else frozenset()
        for k, s in sets.items():
            reused[k] += len(s)
            false_reuse[k] += len(s & labels)
            lat[k] += lm(n - len(s))
    steps = len(gray) - 1
    base = lm(n)
    pol = {}
    for k in names:
        m = lat[k] / steps
        pol[k] = {"reuse_ratio": reused[k] / (steps * n),
                  "edge_false_reuse": false_reuse[k] if edge_labels is not None else None,
                  "mean_latency_ms": m, "speedup": base / m}
    return {"n_steps": steps, "n_tokens": n, "baseline_latency_ms": base,
            "thresholds": {"tau_visual": tau_visual, "tau_naive_freq": tau_naive_freq},
            "policies": pol}
