"""The reference's public transform wrappers on the GPU, in fp64.

Drop-ins for ``spectral.py:24-72`` (``dft2``, ``idft2``, ``amplitude_phase``,
``block_dct``) and ``migration.py:128-134`` (``phase_correlation_spectra``),
with the same argument checks, conventions (unnormalised forward, 1/(U V)
inverse, orthonormal DCT-II, atan2 phase) and errors.  The arithmetic runs
in the C ABI's fp64 spectral operators (``fc_dft2``, ``fc_block_dct``,
``fc_amplitude_phase``, ``fc_phase_correlation_spectra``;
``csrc/fc_spectral.cuh``).  The batched decision path does not use these —
it runs packed fp32 FFTs inside ``fc_select``.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as nat
from .engine import _ptr, _stream
from .geometry import validate_frame
from .types import Displacement

# spectral.py:10 — largest tolerated imaginary residue of an inverse, relative
# to the largest output magnitude
IMAG_RESIDUE_TOL = 1e-6

_WS = {}


def _ws(kind, h, w):
    lib = nat.lib()
    nb = (lib.fc_dft2_workspace_bytes if kind == "dft" else lib.fc_phase_correlation_workspace_bytes)(h, w)
    if nb < 0:
        raise ValueError(f"unsupported grid {h}x{w}")
    key = (kind, torch.cuda.current_device())
    buf = _WS.get(key)
    if buf is None or buf.numel() < nb:
        buf = torch.empty(int(nb), dtype=torch.uint8, device="cuda")
        _WS[key] = buf
    return buf


def _validate_spectrum(spec):
    arr = np.asarray(spec, dtype=np.complex128)
    if arr.ndim != 2:
        raise ValueError(f"spectrum must be 2D, got shape {arr.shape}")
    if arr.shape[0] < 1 or arr.shape[1] < 1:
        raise ValueError(f"spectrum dimensions must be >= 1, got {arr.shape}")
    if not (np.all(np.isfinite(arr.real)) and np.all(np.isfinite(arr.imag))):
        raise ValueError("spectrum contains non-finite values")
    return arr


def _to_dev(a):
    if np.iscomplexobj(a):
        a = np.ascontiguousarray(a, dtype=np.complex128).view(np.float64)
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to("cuda")


def _complex_host(t, h, w):
    return t.cpu().numpy().view(np.complex128).reshape(h, w)


def _dft_dev(src, h, w, complex_in, inverse):
    lib = nat.lib()
    out = torch.empty(h * w * 2, dtype=torch.float64, device="cuda")
    nat.check(lib.fc_dft2(int(h), int(w), _ptr(src), 1 if complex_in else 0, 1 if inverse else 0, _ptr(out),
                          _ptr(_ws("dft", h, w)), _stream()), "fc_dft2")
    return out


def dft2(frame):
    """Forward 2-D DFT of a real frame, unnormalised (spectral.py:24-29)."""
    f = validate_frame(frame)
    h, w = f.shape
    return _complex_host(_dft_dev(_to_dev(f), h, w, False, False), h, w)


def idft2(spectrum):
    """Inverse 2-D DFT with 1/(U V), returned real; rejects spectra whose
    inverse has a non-negligible imaginary residue (spectral.py:32-46)."""
    s = _validate_spectrum(spectrum)
    h, w = s.shape
    out = _complex_host(_dft_dev(_to_dev(s), h, w, True, True), h, w)
    residue = float(np.max(np.abs(out.imag)))
    if residue > IMAG_RESIDUE_TOL * float(np.max(np.abs(out))):
        raise ValueError(f"inverse transform is not real: imaginary residue {residue:g}")
    return np.ascontiguousarray(out.real)


def amplitude_phase(spectrum):
    """Amplitude and atan2 phase of a complex grid (spectral.py:49-56)."""
    s = _validate_spectrum(spectrum)
    lib = nat.lib()
    n = s.size
    src = _to_dev(s)
    amp = torch.empty(n, dtype=torch.float64, device="cuda")
    ph = torch.empty(n, dtype=torch.float64, device="cuda")
    nat.check(lib.fc_amplitude_phase(int(n), _ptr(src), _ptr(amp), _ptr(ph), _stream()), "fc_amplitude_phase")
    return amp.cpu().numpy().reshape(s.shape), ph.cpu().numpy().reshape(s.shape)


def block_dct(patch):
    """Orthonormal 2-D DCT-II of a square patch (spectral.py:59-72)."""
    arr = np.asarray(patch, dtype=np.float64)
    if arr.ndim != 2 or arr.shape[0] != arr.shape[1]:
        raise ValueError(f"patch must be square, got shape {arr.shape}")
    if arr.shape[0] < 1:
        raise ValueError("patch must be non-empty")
    if not np.all(np.isfinite(arr)):
        raise ValueError("patch contains non-finite values")
    p = arr.shape[0]
    if p > 64:
        raise ValueError(f"patch side {p} exceeds the GPU block-DCT limit (64)")
    lib = nat.lib()
    src = _to_dev(arr)
    out = torch.empty(p * p, dtype=torch.float64, device="cuda")
    nat.check(lib.fc_block_dct(1, int(p), _ptr(src), _ptr(out), _stream()), "fc_block_dct")
    return out.cpu().numpy().reshape(p, p)


def phase_correlation_spectra(spec_prev, spec_curr, patch_size=1):
    """Phase correlation on precomputed forward spectra (migration.py:128-134):
    normalised cross-power, inverse transform, impulse peak with the
    reference's tie rule, quantised to patch units."""
    a = np.asarray(spec_prev, dtype=np.complex128)
    b = np.asarray(spec_curr, dtype=np.complex128)
    if a.ndim != 2 or a.shape != b.shape:
        raise ValueError(f"spectra must be 2D of one shape, got {a.shape} and {b.shape}")
    h, w = a.shape
    lib = nat.lib()
    d = torch.empty(2, dtype=torch.int32, device="cuda")
    nat.check(lib.fc_phase_correlation_spectra(int(h), int(w), _ptr(_to_dev(a)), _ptr(_to_dev(b)), _ptr(d),
                                               _ptr(_ws("pc", h, w)), _stream()), "fc_phase_correlation_spectra")
    di, dj = (int(v) for v in d.cpu().tolist())
    return Displacement.from_pixels(di, dj, patch_size)
