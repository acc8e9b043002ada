"""Scalar / geometric stage helpers of the reference API.

These are host-side argument logic with no frame data (a scalar gate, the
budget formula, the high-pass corner shape, an alignment rectangle); the
same formulas run inside the select kernel on the device.
  cutoff_index / highpass_filter   edge_refresh.py:9-26
  alignment_mask                   migration.py:162-176
  migration_gate                   migration.py:179-185
  reuse_budget                     budget.py:61-75
"""

from __future__ import annotations

import math

import numpy as np

from .types import GateAction

CROSS_POWER_EPS = 1e-12  # migration.py:14, used by the K_B cross-power


def cutoff_index(patch_size):
    return max(1, int(patch_size) // 4)


def highpass_filter(patch_size):
    p = int(patch_size)
    if p < 2:
        raise ValueError(f"patch size must be >= 2, got {p}")
    c = cutoff_index(p)
    m = np.ones((p, p))
    m[:c, :c] = 0.0
    return m


def alignment_mask(disp, grid):
    """Slots whose displacement-mapped source lies inside the grid."""
    i = np.arange(grid.rows)[:, None] - disp.di_patches
    j = np.arange(grid.cols)[None, :] - disp.dj_patches
    return (i >= 0) & (i < grid.rows) & (j >= 0) & (j < grid.cols)


def migration_gate(sim, tau_mig):
    if not 0.0 <= sim <= 1.0:
        raise ValueError(f"similarity must lie in [0, 1], got {sim}")
    if not 0.0 <= tau_mig <= 1.0:
        raise ValueError(f"threshold must lie in [0, 1], got {tau_mig}")
    return GateAction.PROCEED if sim >= tau_mig else GateAction.FLUSH


def reuse_budget(normalized_entropy, cfg, n_tokens):
    psi = float(normalized_entropy)
    if not 0.0 <= psi <= 1.0:
        raise ValueError(f"normalized entropy must lie in [0, 1], got {psi}")
    n = int(n_tokens)
    if n < 1:
        raise ValueError(f"token count must be >= 1, got {n}")
    alpha = cfg.alpha_min + (cfg.alpha_max - cfg.alpha_min) * math.exp(-psi)
    return alpha, int(math.floor(alpha * n))
