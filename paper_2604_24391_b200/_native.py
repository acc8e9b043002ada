"""ctypes binding of the C ABI (``include/freqcache_b200.h``).

The product path has no CPU fallback: if the sm_100a library is missing or
no CUDA device is present, :func:`lib` raises.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

_LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libfreqcache_b200.so"

FC_OK = 0
FC_EINVAL = 1
FC_EUNSUPPORTED = 2
FC_ECUDA = 3
FC_ENONFINITE = 4
FC_EPSI = 5
FC_EBOUNDS = 6

FC_DIAG_NONE = 0
FC_DIAG_DEGENERATE = 1
FC_DIAG_NO_TEXTURE = 2
DIAG_TEXT = {
    FC_DIAG_NONE: None,
    FC_DIAG_DEGENERATE: "degenerate spectrum",
    FC_DIAG_NO_TEXTURE: "no texture; displacement undefined",
}

FC_FMT_RGB_F32 = 0
FC_FMT_GRAY_F32 = 1
FC_FMT_GRAY_F64 = 2
FC_FMT_GRAY_U8 = 3
FC_FMT_RGB_U8 = 4

FC_FRESH_DENSE = 0
FC_FRESH_COMPACT = 1

EXPORTS = (
    "fc_abi_version", "fc_strerror", "fc_plan_create", "fc_plan_destroy",
    "fc_plan_state_bytes", "fc_plan_workspace_bytes", "fc_plan_tokens", "fc_plan_launches",
    "fc_state_reset", "fc_select", "fc_select_front", "fc_select_back", "fc_select_profile", "fc_patch_energy", "fc_splice",
    "fc_splice_map", "fc_stage_workspace_bytes", "fc_amp_cosine", "fc_spectral_sums",
    "fc_refresh_mask", "fc_topk_ascending", "fc_render_masks", "fc_splice_packed",
    "fc_splice_inplace", "fc_splice_inplace_plan", "fc_splice_inplace_copy", "fc_splice_inplace_scratch_bytes", "fc_compare_cosines", "fc_row_cosines",
    "fc_graph_capture_begin", "fc_graph_capture_end", "fc_graph_launch", "fc_graph_destroy",
    "fc_dft2_workspace_bytes", "fc_dft2", "fc_phase_correlation_workspace_bytes", "fc_phase_correlation_spectra",
    "fc_block_dct", "fc_amplitude_phase", "fc_gather_patches",
)


class Geometry(C.Structure):
    _fields_ = [("batch", C.c_int32), ("height", C.c_int32), ("width", C.c_int32),
                ("patch_size", C.c_int32), ("format", C.c_int32)]


class Config(C.Structure):
    _fields_ = [("tau_mig", C.c_double), ("edge_lambda", C.c_double),
                ("alpha_min", C.c_double), ("alpha_max", C.c_double),
                ("refresh_shift", C.c_int32), ("reserved", C.c_int32)]


class SelectOut(C.Structure):
    _fields_ = [("results", C.c_void_p), ("reuse_idx", C.c_void_p),
                ("recompute_idx", C.c_void_p), ("src_map", C.c_void_p),
                ("reuse_mask", C.c_void_p), ("refresh_mask", C.c_void_p),
                ("energy", C.c_void_p), ("counters", C.c_void_p)]


# fc_stream_result as a numpy structured dtype (identical layout)
RESULT_DTYPE = np.dtype([
    ("status", "<i4"), ("cold", "<i4"), ("flushed", "<i4"), ("diagnostic", "<i4"),
    ("k_reuse", "<i4"), ("k_candidate", "<i4"), ("k_final", "<i4"), ("n_refresh", "<i4"),
    ("di", "<i4"), ("dj", "<i4"), ("di_patches", "<i4"), ("dj_patches", "<i4"),
    ("rows", "<i4"), ("cols", "<i4"), ("bin_count", "<i8"),
    ("sim_freq", "<f8"), ("entropy_raw", "<f8"), ("entropy_norm", "<f8"), ("alpha", "<f8"),
    ("energy_mean", "<f8"), ("energy_std", "<f8"), ("energy_threshold", "<f8"),
    ("peak", "<f8"), ("peak_runner_up", "<f8"),
])
assert RESULT_DTYPE.itemsize == 136


class NativeError(RuntimeError):
    pass


_lib = None


def load(path=None):
    """Load the shared library (no device needed); raises if it is absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else _LIB_PATH
    if not p.exists():
        raise NativeError(
            f"CUDA library {p} is missing — run `python -m paper_2604_24391_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(p))
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    sig = {
        "fc_abi_version": (C.c_int, []),
        "fc_strerror": (C.c_char_p, [C.c_int]),
        "fc_plan_create": (C.c_int, [C.POINTER(Geometry), C.POINTER(vp)]),
        "fc_plan_destroy": (None, [vp]),
        "fc_plan_state_bytes": (i64, [vp]),
        "fc_plan_workspace_bytes": (i64, [vp]),
        "fc_plan_tokens": (C.c_int, [vp]),
        "fc_plan_launches": (C.c_int, [vp]),
        "fc_state_reset": (C.c_int, [vp, vp, i32, i32, vp]),
        "fc_select": (C.c_int, [vp, C.POINTER(Config), vp, vp, vp, C.POINTER(SelectOut), vp]),
        "fc_select_front": (C.c_int, [vp, C.POINTER(Config), vp, vp, C.POINTER(SelectOut), i32, vp]),
        "fc_select_back": (C.c_int, [vp, C.POINTER(Config), vp, vp, C.POINTER(SelectOut), i32, vp]),
        "fc_select_profile": (C.c_int, [vp, C.POINTER(Config), vp, vp, vp, C.POINTER(SelectOut),
                                        C.POINTER(C.c_float), vp]),
        "fc_patch_energy": (C.c_int, [vp, vp, vp, vp, vp]),
        "fc_splice": (C.c_int, [i32, i32, i64, vp, vp, vp, vp, i32, i32, vp, vp, vp, vp]),
        "fc_splice_map": (C.c_int, [i32, i32, vp, i32, i32, i32, vp, vp, vp]),
        "fc_stage_workspace_bytes": (i64, []),
        "fc_render_masks": (C.c_int, [i32, i32, vp, vp, vp, vp, vp]),
        "fc_splice_packed": (C.c_int, [i32, i32, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
        "fc_splice_inplace": (C.c_int, [i32, i32, i64, vp, vp, vp, vp, vp, vp, vp, vp, i32, i32, vp, vp, vp]),
        "fc_splice_inplace_plan": (C.c_int, [i32, i32, i64, vp, vp, vp, vp, vp, vp, vp, vp, i32, i32, vp, vp]),
        "fc_splice_inplace_copy": (C.c_int, [i32, i32, i64, vp, vp, vp, vp, vp, vp, vp, vp, i32, i32, vp, vp, i32,
                                             vp]),
        "fc_splice_inplace_scratch_bytes": (i64, [i32, i32]),
        "fc_amp_cosine": (C.c_int, [vp, vp, i64, vp, vp, vp, vp]),
        "fc_spectral_sums": (C.c_int, [vp, i64, i32, vp, vp, vp, vp]),
        "fc_refresh_mask": (C.c_int, [vp, i64, C.c_double, vp, vp, vp, vp]),
        "fc_topk_ascending": (C.c_int, [vp, i64, vp, i64, i64, vp, vp, vp]),
        "fc_compare_cosines": (C.c_int, [C.POINTER(Geometry), vp, vp, vp, vp, vp]),
        "fc_row_cosines": (C.c_int, [i64, i64, vp, vp, vp, vp]),
        "fc_graph_capture_begin": (C.c_int, [vp]),
        "fc_graph_capture_end": (C.c_int, [vp, C.POINTER(vp)]),
        "fc_graph_launch": (C.c_int, [vp, vp]),
        "fc_graph_destroy": (None, [vp]),
        "fc_dft2_workspace_bytes": (i64, [i32, i32]),
        "fc_dft2": (C.c_int, [i32, i32, vp, i32, i32, vp, vp, vp]),
        "fc_phase_correlation_workspace_bytes": (i64, [i32, i32]),
        "fc_phase_correlation_spectra": (C.c_int, [i32, i32, vp, vp, vp, vp, vp]),
        "fc_block_dct": (C.c_int, [i32, i32, vp, vp, vp]),
        "fc_amplitude_phase": (C.c_int, [i64, vp, vp, vp, vp]),
        "fc_gather_patches": (C.c_int, [i32, i32, i32, i32, i32, vp, vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def lib():
    """The library, for device work: also requires a CUDA device."""
    import torch

    if not torch.cuda.is_available():
        raise NativeError("no CUDA device: the FreqCache B200 path has no CPU fallback")
    return load()


def check(rc, what=""):
    if rc != FC_OK:
        msg = load().fc_strerror(rc).decode()
        if rc in (FC_EINVAL, FC_ENONFINITE, FC_EPSI):
            raise ValueError(f"{what}: {msg}" if what else msg)
        if rc == FC_EBOUNDS:
            raise AssertionError(f"{what}: {msg}" if what else msg)
        raise NativeError(f"{what}: {msg} (code {rc})")
