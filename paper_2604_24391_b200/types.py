"""Data contracts of the drop-in API (reference names, fields and checks).

Mirrors the reference's frozen dataclasses and errors so callers of
``freqcache`` can switch imports:
  errors      errors.py:4-23
  BudgetConfig / EntropyReading        budget.py:12-31
  EnergyMap / RefreshMask              edge_refresh.py:29-45
  Displacement / GateAction            migration.py:17-50
  CostModel / CacheConfig / CacheDecision / TokenCache / StepReport /
  SequenceReport                       fusion.py:27-94, 426-447, 515-531
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import Enum

import numpy as np


# ------------------------------------------------------------------ errors --

class DegenerateSpectrumError(ValueError):
    """Amplitude grid with zero energy: spectral statistics are undefined."""


class ConstantFrameError(ValueError):
    """Frame without texture: displacement estimation is undefined."""


class FrameParseError(ValueError):
    """Unreadable frame file; ``offset`` is the failing byte position."""

    def __init__(self, message, offset=None):
        super().__init__(message if offset is None else f"{message} (byte offset {offset})")
        self.offset = offset


# ------------------------------------------------------------------ budget --

@dataclass(frozen=True)
class BudgetConfig:
    alpha_min: float = 0.08
    alpha_max: float = 0.5

    def __post_init__(self):
        lo, hi = self.alpha_min, self.alpha_max
        if not (0.0 <= lo <= hi <= 1.0):
            raise ValueError(f"need 0 <= alpha_min <= alpha_max <= 1, got ({lo}, {hi})")


@dataclass(frozen=True)
class EntropyReading:
    raw: float
    normalized: float
    bin_count: int


# -------------------------------------------------------------- edge stage --

@dataclass(frozen=True)
class EnergyMap:
    energies: np.ndarray
    patch_size: int
    cutoff: int


@dataclass(frozen=True)
class RefreshMask:
    mask: np.ndarray
    mean_energy: float
    std_energy: float
    sensitivity: float


# --------------------------------------------------------- migration stage --

def to_patch_units(d, patch_size):
    """Nearest whole patch, half-patch toward zero (migration.py:41-45)."""
    d, p = int(d), int(patch_size)
    q = (2 * abs(d) + p - 1) // (2 * p)
    return q if d >= 0 else -q


@dataclass(frozen=True)
class Displacement:
    di: int
    dj: int
    di_patches: int
    dj_patches: int

    @classmethod
    def from_pixels(cls, di, dj, patch_size=1):
        return cls(int(di), int(dj), to_patch_units(di, patch_size), to_patch_units(dj, patch_size))


class GateAction(Enum):
    FLUSH = "flush"
    PROCEED = "proceed"


# ------------------------------------------------------------------ fusion --

@dataclass(frozen=True)
class CostModel:
    """Modelled step latency, affine in the recomputed-token count."""

    base_ms: float
    per_token_ms: float

    def latency_ms(self, n_recompute):
        return self.base_ms + self.per_token_ms * n_recompute

    @classmethod
    def calibrated(cls, full_ms, cached_ms, reuse_ratio, n_tokens):
        # same operation order as fusion.py:37-44 (bit-identical constants)
        n_full = float(n_tokens)
        n_cached = n_tokens * (1.0 - reuse_ratio)
        per = (full_ms - cached_ms) / (n_full - n_cached)
        return cls(full_ms - per * n_full, per)


DEFAULT_COST_MODEL = CostModel.calibrated(637.0, 401.0, 0.535, 196)


@dataclass(frozen=True)
class CacheConfig:
    tau_mig: float = 0.12
    edge_lambda: float = 0.25
    budget: BudgetConfig = field(default_factory=BudgetConfig)
    patch_size: int = 16

    def __post_init__(self):
        if not (0.0 <= self.tau_mig <= 1.0):
            raise ValueError(f"tau_mig must lie in [0, 1], got {self.tau_mig}")
        if not math.isfinite(self.edge_lambda):
            raise ValueError("edge_lambda must be finite")
        if self.patch_size < 2:
            raise ValueError(f"patch_size must be >= 2, got {self.patch_size}")


@dataclass
class CacheDecision:
    step: int
    flushed: bool
    sim_freq: float
    displacement: Displacement
    entropy: EntropyReading
    alpha_t: float
    k_reuse: int
    k_candidate: int
    k_final: int
    reuse_set: tuple
    recompute_set: tuple
    rows: int
    cols: int
    refresh_set: tuple
    diagnostic: str = None
    timings_us: dict = field(default_factory=dict, compare=False)


@dataclass
class TokenCache:
    tokens: np.ndarray  # (rows, cols, dim)
    ages: np.ndarray    # (rows, cols) int64

    @property
    def rows(self):
        return self.tokens.shape[0]

    @property
    def cols(self):
        return self.tokens.shape[1]


@dataclass(frozen=True)
class StepReport:
    step: int
    n_reused: int
    n_recomputed: int
    latency_model_ms: float


@dataclass
class SequenceReport:
    n_frames: int
    n_tokens: int
    decisions: list
    step_reports: list
    mean_reuse_ratio: float
    mean_latency_ms: float
    baseline_latency_ms: float
    speedup: float
    flush_count: int
