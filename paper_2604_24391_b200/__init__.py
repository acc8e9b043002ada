"""B200-native FreqCache token-cache decision path (arXiv 2604.24391).

Drop-in for the reference package's decision path (``freqcache``,
``pkg/src/freqcache/__init__.py:11-98``): same names, signatures and error
behaviour for the path's entry points, executed by hand-written sm_100a
kernels behind the C ABI in ``include/freqcache_b200.h``.  The batched,
device-resident API for many streams per GPU is :class:`FreqCacheEngine`.

Importing the package does not need a GPU; calling into the path does (no
CPU fallback).
"""

__version__ = "0.1.0"

from .types import (  # noqa: F401
    DEFAULT_COST_MODEL,
    BudgetConfig,
    CacheConfig,
    CacheDecision,
    ConstantFrameError,
    CostModel,
    DegenerateSpectrumError,
    Displacement,
    EnergyMap,
    EntropyReading,
    FrameParseError,
    GateAction,
    RefreshMask,
    SequenceReport,
    StepReport,
    TokenCache,
)
from .geometry import PatchGrid, validate_frame  # noqa: F401
from .stages import (  # noqa: F401
    CROSS_POWER_EPS,
    alignment_mask,
    cutoff_index,
    highpass_filter,
    migration_gate,
    reuse_budget,
)
from .api import (  # noqa: F401
    decide,
    default_token_fn,
    patch_energy,
    phase_correlation,
    populate_cache,
    refresh_mask,
    run_sequence,
    sim_freq,
    sim_spatial,
    spectral_entropy,
    step,
    topk_ascending,
)
from .spectral import amplitude_phase, block_dct, dft2, idft2, phase_correlation_spectra  # noqa: F401
from .engine import FreqCacheEngine, SelectResult, SpliceState, StepGraph, splice, splice_map  # noqa: F401
from . import records  # noqa: F401
