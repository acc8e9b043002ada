"""Frame ingest (§8f #4): the reference's file formats, and a device loader.

Host API with the reference's names and behaviour (frameio.py:1-219):
binary PGM / PPM (maxval 255) and the ``rawf32`` container
(``FQC1`` + u32 height, width, count, little-endian float32 payload), with
parse errors carrying the byte offset at which the file became unreadable.

Device ingest (``load_frames_device``): the payload goes to the GPU in its
compact on-disk form — 1 byte per pixel for P5, 3 for P6, 4 for rawf32 —
through pinned host memory, and the decision kernels read that layout
directly (``FC_FMT_GRAY_U8`` / ``FC_FMT_RGB_U8`` / ``FC_FMT_GRAY_F32``): the
gray value (v / 255, or BT.601 luma / 255 in fp64, frameio.py:81-88) is formed
inside the frame kernel, so no float64 frame is ever materialised.  For RGB
PPM input that is 3 bytes per pixel over PCIe and HBM instead of the 8 of a
float64 gray frame.
"""

from __future__ import annotations

import re
import struct
from pathlib import Path

import numpy as np

from .types import FrameParseError

RAWF32_MAGIC = b"FQC1"          # frameio.py:21
RAWF32_HEADER = 16              # frameio.py:22
LUMA_WEIGHTS = (0.299, 0.587, 0.114)   # frameio.py:26

# Netpbm header grammar (frameio.py:29-50): fields are runs of non-blank
# bytes; blanks and `#` comments (to end of line) separate them; exactly one
# blank byte ends the header after maxval.
_BLANKS = b" \t\n\r\x0b\x0c"
_GAP = re.compile(rb"(?:[ \t\n\r\x0b\x0c]|#[^\n\r]*)*")
_FIELD = re.compile(rb"[^ \t\n\r\x0b\x0c]+")
_CHANNELS = {b"P5": 1, b"P6": 3}


class _Fail(Exception):
    """A parse failure before the file name is attached: (message, offset)."""


def _header_fields(data, want):
    """The first ``want`` header fields and the payload offset."""
    fields, at, end = [], 0, len(data)
    for _ in range(want):
        at = _GAP.match(data, at).end()
        if at >= end:
            raise _Fail("truncated header", at)
        m = _FIELD.match(data, at)
        fields.append(m.group())
        at = m.end()
    if at >= end:
        raise _Fail("missing pixel data", at)
    return fields, at + 1


def _netpbm(data):
    """(uint8 pixels (H, W) or (H, W, 3), channels) of P5 / P6 bytes."""
    if len(data) < 2:
        raise _Fail("file too short", len(data))
    channels = _CHANNELS.get(data[:2])
    if channels is None:
        raise _Fail(f"unsupported magic {data[:2]!r}", 0)
    fields, at = _header_fields(data, 4)
    try:
        width, height, maxval = map(int, fields[1:])
    except ValueError:
        raise _Fail("non-numeric header field", 2) from None
    rules = ((width >= 1 and height >= 1, f"invalid dimensions {width}x{height}"),
             (maxval == 255, f"only maxval 255 supported, got {maxval}"))
    for ok, msg in rules:
        if not ok:
            raise _Fail(msg, 2)
    count = width * height * channels
    body = memoryview(data)[at:at + count]
    if body.nbytes < count:
        raise _Fail(f"truncated pixel data, expected {count} bytes", at + body.nbytes)
    px = np.frombuffer(body, dtype=np.uint8)
    return px.reshape((height, width) if channels == 1 else (height, width, 3)), channels


def _parse(path, parser):
    path = Path(path)
    try:
        return parser(path.read_bytes())
    except _Fail as f:
        msg, offset = f.args
        raise FrameParseError(f"{path}: {msg}", offset=offset) from None


def read_netpbm_payload(path):
    """Parse a P5 / P6 file (frameio.py:53-80): returns (uint8 pixels of
    shape (H, W) or (H, W, 3), channels)."""
    return _parse(path, _netpbm)


def read_netpbm(path):
    """P5 gray / P6 luma-reduced frame as float64 in [0, 1] (frameio.py:53-88)."""
    px, channels = read_netpbm_payload(path)
    v = px.astype(np.float64)
    if channels == 3:
        # left-to-right sum, as the reference writes it
        v = (LUMA_WEIGHTS[0] * v[..., 0] + LUMA_WEIGHTS[1] * v[..., 1]) + LUMA_WEIGHTS[2] * v[..., 2]
    return v / 255.0


def _u8_image(values):
    a = np.asarray(values)
    if a.ndim != 2:
        raise ValueError(f"image must be 2D, got shape {a.shape}")
    return a if a.dtype == np.uint8 else np.round(np.clip(a, 0.0, 1.0) * 255.0).astype(np.uint8)


def write_pgm(path, values):
    """Binary P5, maxval 255; float data clipped to [0, 1] and quantised
    (frameio.py:91-105)."""
    img = _u8_image(values)
    header = b"P5\n%d %d\n255\n" % (img.shape[1], img.shape[0])
    Path(path).write_bytes(header + img.tobytes())


def _finite_2d(f):
    a = np.asarray(f, dtype=np.float64)
    problem = ("frame must be 2D, got shape %s" % (a.shape,) if a.ndim != 2 else
               "frame dimensions must be >= 1, got %s" % (a.shape,) if min(a.shape) < 1 else
               "frame contains non-finite values" if not np.isfinite(a).all() else None)
    if problem:
        raise ValueError(problem)
    return a


def save_rawf32(path, frames):
    """rawf32 container writer (frameio.py:107-115)."""
    stack = np.stack([_finite_2d(f) for f in frames]).astype("<f4")
    t, h, w = stack.shape
    Path(path).write_bytes(RAWF32_MAGIC + struct.pack("<III", h, w, t) + stack.tobytes())


def _rawf32(data):
    """float32 [T, H, W] view of rawf32 bytes (frameio.py:118-139)."""
    if len(data) < RAWF32_HEADER:
        raise _Fail("truncated rawf32 header", len(data))
    if data[:4] != RAWF32_MAGIC:
        raise _Fail(f"bad magic {data[:4]!r}, expected {RAWF32_MAGIC!r}", 0)
    h, w, t = struct.unpack_from("<III", data, 4)
    if min(h, w, t) < 1:
        raise _Fail(f"invalid header dimensions {h}x{w}x{t}", 4)
    size = RAWF32_HEADER + 4 * h * w * t
    if len(data) != size:
        raise (_Fail(f"truncated rawf32 payload, expected {size} bytes", len(data)) if len(data) < size
               else _Fail("trailing bytes after payload", size))
    return np.frombuffer(data, dtype="<f4", count=h * w * t, offset=RAWF32_HEADER).reshape(t, h, w)


def _rawf32_payload(path):
    return _parse(path, _rawf32), Path(path)


def load_rawf32(path):
    """rawf32 reader (frameio.py:118-146): float64 frames, non-finite rejected."""
    vals, path = _rawf32_payload(path)
    bad = np.flatnonzero(~np.isfinite(vals).reshape(vals.shape[0], -1).all(axis=1))
    if bad.size:
        raise FrameParseError(f"{path}: frame {int(bad[0])} contains non-finite values")
    return list(vals.astype(np.float64))


_NETPBM_SUFFIXES = (".pgm", ".ppm")


def _resolve(path, fmt):
    """(format, files) of a rawf32 file, a netpbm file or a directory of
    netpbm files in sorted order."""
    path = Path(path)
    if fmt == "auto":
        fmt = "pgm" if (path.is_dir() or path.suffix.lower() in _NETPBM_SUFFIXES) else "rawf32"
    if fmt not in ("rawf32", "pgm"):
        raise ValueError(f"unknown format {fmt!r}")
    if fmt == "rawf32" or not path.is_dir():
        return fmt, [path]
    files = sorted(p for p in path.iterdir() if p.suffix.lower() in _NETPBM_SUFFIXES)
    if not files:
        raise FrameParseError(f"{path}: no .pgm/.ppm files found")
    return fmt, files


def load_frames(path, fmt="auto"):
    """Ordered frame list from a rawf32 file, a netpbm file or a directory of
    them in sorted order (frameio.py:149-175)."""
    fmt, files = _resolve(path, fmt)
    return load_rawf32(files[0]) if fmt == "rawf32" else list(map(read_netpbm, files))


def load_frames_device(path, fmt="auto", device=None):
    """Frames straight to the GPU in their compact on-disk layout.

    Returns ``(frames, engine_format)``: uint8 [T, H, W] ("gray_u8") for P5,
    uint8 [T, H, W, 3] ("rgb_u8") for P6, float32 [T, H, W] ("gray32") for
    rawf32 — ready for ``FreqCacheEngine(..., fmt=engine_format)`` with
    ``frames[t]`` (or a [B, ...] slice) per step.  The payload is staged in
    pinned host memory and copied asynchronously.  A directory mixing P5 and
    P6 files raises ValueError (one layout per tensor; use load_frames).
    """
    import torch

    from . import _native as nat

    nat.lib()
    dev = torch.device(device) if device is not None else torch.device("cuda")
    fmt, files = _resolve(path, fmt)
    if fmt == "rawf32":
        vals, p = _rawf32_payload(files[0])
        host = torch.empty(vals.shape, dtype=torch.float32).pin_memory()
        host.numpy()[...] = vals
        out = host.to(dev, non_blocking=True)
        bad = (~torch.isfinite(out)).flatten(1).any(dim=1)
        if bool(bad.any()):
            t = int(torch.nonzero(bad)[0, 0])
            raise FrameParseError(f"{p}: frame {t} contains non-finite values")
        return out, "gray32"
    payloads = [read_netpbm_payload(p) for p in files]
    chans = {c for _, c in payloads}
    if len(chans) != 1:
        raise ValueError("directory mixes P5 and P6 files; use load_frames for gray float64 frames")
    shapes = {px.shape for px, _ in payloads}
    if len(shapes) != 1:
        raise ValueError(f"frames differ in shape: {sorted(shapes)}")
    shape = payloads[0][0].shape
    host = torch.empty((len(payloads),) + shape, dtype=torch.uint8).pin_memory()
    hv = host.numpy()
    for t, (px, _) in enumerate(payloads):
        hv[t] = px
    out = host.to(dev, non_blocking=True)
    return out, ("gray_u8" if chans == {1} else "rgb_u8")


def export_energy_heatmap(energy_map, path):
    """Per-patch energy map as an 8-bit PGM, hottest patch = 255
    (frameio.py:178-188)."""
    e = np.asarray(energy_map.energies, dtype=np.float64)
    top = float(e.max())
    scaled = np.zeros_like(e) if top <= 0.0 else e / top
    write_pgm(path, scaled)
    return Path(path)
