"""Three-policy comparison (reference compare.py:1-114) on the GPU.

``compare_domains`` has the reference's signature and report layout.  The
freqcache policy is the GPU decision path (one engine carries the previous
frame's spectrum, so each frame is transformed once); the two position-wise
baselines — raw-pixel cosine ("visual") and per-patch |DFT| cosine
("naive_freq") — come from ``fc_compare_cosines`` for every frame pair of the
sequence in one launch.  A custom ``token_fn`` stays a host callable (it is
the user's model, as in the reference); its vectors are compared on the GPU
with ``fc_row_cosines``.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as nat
from .api import _fetch, _raise_status, decision_from_device
from .engine import FreqCacheEngine, compare_cosines as _cosines_dev, row_cosines
from .geometry import PatchGrid, coerce_frame, grid_shape
from .types import DEFAULT_COST_MODEL


def _token_stack(grid, frame, token_fn):
    """token_fn over every patch, row-major (compare.py:41-47)."""
    vecs = [np.asarray(token_fn(grid.patch(*grid.position(q), frame)), dtype=np.float64).ravel()
            for q in range(grid.n_patches)]
    return np.stack(vecs)


def compare_cosines(prev, curr, patch_size):
    """(visual, naive_freq) per-patch cosines of one gray frame pair (host
    numpy in, host numpy out; the work runs on the GPU)."""
    nat.lib()
    a, b = coerce_frame(prev), coerce_frame(curr)
    if a.shape != b.shape:
        raise ValueError(f"frame shapes differ: {a.shape} vs {b.shape}")
    grid_shape(*a.shape, patch_size)
    tp = torch.from_numpy(a).to("cuda").unsqueeze(0)
    tc = torch.from_numpy(b).to("cuda").unsqueeze(0)
    vis, nf = _cosines_dev(tp, tc, patch_size)
    return vis[0].cpu().numpy(), nf[0].cpu().numpy()


def compare_domains(frames, cfg, *, token_fn=None, edge_labels=None, tau_visual=0.85, tau_naive_freq=0.85,
                    cost_model=None):
    """Run all three policies over consecutive frame pairs (compare.py:55-114)."""
    if len(frames) < 2:
        raise ValueError("need at least 2 frames")
    frames = [coerce_frame(f) for f in frames]
    cost_model = cost_model or DEFAULT_COST_MODEL
    grid = PatchGrid(frames[0], cfg.patch_size)
    n = grid.n_patches
    h, w = frames[0].shape
    for t, f in enumerate(frames):
        if f.shape != (h, w):
            raise ValueError(f"frame shape {f.shape} does not match grid shape {(h, w)}")
    have_labels = edge_labels is not None
    T = len(frames)

    # freqcache policy: the decision path over the sequence
    eng = FreqCacheEngine(1, h, w, cfg.patch_size, fmt="gray64")
    dev = eng.device
    stack = torch.from_numpy(np.ascontiguousarray(np.stack(frames))).to(dev)
    aux = eng.new_output()
    eng.select(stack[0:1], cfg, out=aux)
    _raise_status(aux.host_results()[0])
    reuse_sets = []
    for t in range(1, T):
        out = eng.select(stack[t:t + 1], cfg)
        res, ri, rc, rm = _fetch(out)
        _raise_status(res)
        d = decision_from_device(res, ri, rc, rm, step=t)
        reuse_sets.append(set(d.reuse_set))

    # position-wise baselines: every pair in one launch
    vis, nf = _cosines_dev(stack[:-1].contiguous(), stack[1:].contiguous(), cfg.patch_size)
    if token_fn is not None:
        vis = torch.stack([
            row_cosines(torch.from_numpy(_token_stack(grid, frames[t - 1], token_fn)).to(dev),
                        torch.from_numpy(_token_stack(grid, frames[t], token_fn)).to(dev))
            for t in range(1, T)])
    vis = vis.cpu().numpy()
    nf = nf.cpu().numpy()

    names = ("freqcache", "visual", "naive_freq")
    reused_total = dict.fromkeys(names, 0)
    false_reuse = dict.fromkeys(names, 0)
    latency_total = dict.fromkeys(names, 0.0)
    for t in range(1, T):
        sets = {
            "freqcache": reuse_sets[t - 1],
            "visual": set(np.flatnonzero(vis[t - 1] > tau_visual).tolist()),
            "naive_freq": set(np.flatnonzero(nf[t - 1] > tau_naive_freq).tolist()),
        }
        labels = frozenset(edge_labels[t]) if have_labels else frozenset()
        for name, reuse in sets.items():
            reused_total[name] += len(reuse)
            false_reuse[name] += len(reuse & labels)
            latency_total[name] += cost_model.latency_ms(n - len(reuse))

    n_steps = T - 1
    baseline = cost_model.latency_ms(n)
    policies = {}
    for name in names:
        mean_latency = latency_total[name] / n_steps
        policies[name] = {
            "reuse_ratio": reused_total[name] / (n_steps * n),
            "edge_false_reuse": false_reuse[name] if have_labels else None,
            "mean_latency_ms": mean_latency,
            "speedup": baseline / mean_latency,
        }
    return {
        "n_steps": n_steps,
        "n_tokens": n,
        "baseline_latency_ms": baseline,
        "thresholds": {"tau_visual": tau_visual, "tau_naive_freq": tau_naive_freq},
        "policies": policies,
    }
