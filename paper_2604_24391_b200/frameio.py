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

import struct
from pathlib import Path

import numpy as np

from .types import FrameParseError

RAWF32_MAGIC = b"FQC1"          # frameio.py:21
RAWF32_HEADER = 16              # frameio.py:22
LUMA_WEIGHTS = (0.299, 0.587, 0.114)   # frameio.py:26


def _tokenize_netpbm(data, count, path):
    """Header tokens and the payload offset (frameio.py:29-50): tokens are
    whitespace-delimited, ``#`` starts a comment that runs to end of line, and
    exactly one whitespace byte separates maxval from the payload."""
    tokens = []
    pos, n = 0, len(data)
    while len(tokens) < count:
        if pos >= n:
            raise FrameParseError(f"{path}: truncated header", offset=pos)
        c = data[pos:pos + 1]
        if c.isspace():
            pos += 1
        elif c == b"#":
            while pos < n and data[pos:pos + 1] not in (b"\n", b"\r"):
                pos += 1
        else:
            start = pos
            while pos < n and not data[pos:pos + 1].isspace():
                pos += 1
            tokens.append(data[start:pos])
    if pos >= n:
        raise FrameParseError(f"{path}: missing pixel data", offset=pos)
    return tokens, pos + 1


def read_netpbm_payload(path):
    """Parse a P5 / P6 file (frameio.py:53-80): returns (uint8 pixels of
    shape (H, W) or (H, W, 3), channels)."""
    path = Path(path)
    data = path.read_bytes()
    if len(data) < 2:
        raise FrameParseError(f"{path}: file too short", offset=len(data))
    magic = data[:2]
    if magic not in (b"P5", b"P6"):
        raise FrameParseError(f"{path}: unsupported magic {magic!r}", offset=0)
    tokens, at = _tokenize_netpbm(data, 4, path)
    try:
        width, height, maxval = (int(t) for t in tokens[1:])
    except ValueError:
        raise FrameParseError(f"{path}: non-numeric header field", offset=2)
    if width < 1 or height < 1:
        raise FrameParseError(f"{path}: invalid dimensions {width}x{height}", offset=2)
    if maxval != 255:
        raise FrameParseError(f"{path}: only maxval 255 supported, got {maxval}", offset=2)
    channels = 1 if magic == b"P5" else 3
    need = width * height * channels
    payload = data[at:at + need]
    if len(payload) < need:
        raise FrameParseError(f"{path}: truncated pixel data, expected {need} bytes",
                              offset=at + len(payload))
    px = np.frombuffer(payload, dtype=np.uint8)
    shape = (height, width) if channels == 1 else (height, width, 3)
    return px.reshape(shape), channels


def read_netpbm(path):
    """P5 gray / P6 luma-reduced frame as float64 in [0, 1] (frameio.py:53-88)."""
    px, channels = read_netpbm_payload(path)
    p = px.astype(np.float64)
    if channels == 1:
        gray = p
    else:
        gray = LUMA_WEIGHTS[0] * p[..., 0] + LUMA_WEIGHTS[1] * p[..., 1] + LUMA_WEIGHTS[2] * p[..., 2]
    return gray / 255.0


def write_pgm(path, values):
    """Binary P5, maxval 255; float data clipped to [0, 1] and quantised
    (frameio.py:91-105)."""
    arr = np.asarray(values)
    if arr.ndim != 2:
        raise ValueError(f"image must be 2D, got shape {arr.shape}")
    if arr.dtype != np.uint8:
        arr = np.round(np.clip(arr, 0.0, 1.0) * 255.0).astype(np.uint8)
    h, w = arr.shape
    with open(path, "wb") as fh:
        fh.write(f"P5\n{w} {h}\n255\n".encode("ascii"))
        fh.write(arr.tobytes())


def _validate(f):
    a = np.asarray(f, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError(f"frame must be 2D, got shape {a.shape}")
    if a.shape[0] < 1 or a.shape[1] < 1:
        raise ValueError(f"frame dimensions must be >= 1, got {a.shape}")
    if not np.all(np.isfinite(a)):
        raise ValueError("frame contains non-finite values")
    return a


def save_rawf32(path, frames):
    """rawf32 container writer (frameio.py:107-115)."""
    stack = np.stack([_validate(f) for f in frames]).astype("<f4")
    t, h, w = stack.shape
    with open(path, "wb") as fh:
        fh.write(RAWF32_MAGIC)
        fh.write(struct.pack("<III", h, w, t))
        fh.write(stack.tobytes())


def _rawf32_payload(path):
    """Header checks of frameio.py:118-139; returns float32 [T, H, W]."""
    path = Path(path)
    data = path.read_bytes()
    if len(data) < RAWF32_HEADER:
        raise FrameParseError(f"{path}: truncated rawf32 header", offset=len(data))
    if data[:4] != RAWF32_MAGIC:
        raise FrameParseError(f"{path}: bad magic {data[:4]!r}, expected {RAWF32_MAGIC!r}", offset=0)
    h, w, t = struct.unpack("<III", data[4:16])
    if h < 1 or w < 1 or t < 1:
        raise FrameParseError(f"{path}: invalid header dimensions {h}x{w}x{t}", offset=4)
    need = RAWF32_HEADER + 4 * h * w * t
    if len(data) < need:
        raise FrameParseError(f"{path}: truncated rawf32 payload, expected {need} bytes", offset=len(data))
    if len(data) > need:
        raise FrameParseError(f"{path}: trailing bytes after payload", offset=need)
    return np.frombuffer(data, dtype="<f4", count=h * w * t, offset=RAWF32_HEADER).reshape(t, h, w), path


def load_rawf32(path):
    """rawf32 reader (frameio.py:118-146): float64 frames, non-finite rejected."""
    vals, path = _rawf32_payload(path)
    frames = vals.astype(np.float64)
    for t in range(frames.shape[0]):
        if not np.all(np.isfinite(frames[t])):
            raise FrameParseError(f"{path}: frame {t} contains non-finite values")
    return [frames[t] for t in range(frames.shape[0])]


def _resolve(path, fmt):
    path = Path(path)
    if fmt == "auto":
        if path.is_dir() or path.suffix.lower() in (".pgm", ".ppm"):
            fmt = "pgm"
        else:
            fmt = "rawf32"
    if fmt not in ("rawf32", "pgm"):
        raise ValueError(f"unknown format {fmt!r}")
    if fmt == "pgm" and path.is_dir():
        files = sorted(p for p in path.iterdir() if p.suffix.lower() in (".pgm", ".ppm"))
        if not files:
            raise FrameParseError(f"{path}: no .pgm/.ppm files found")
        return fmt, files
    return fmt, [path]


def load_frames(path, fmt="auto"):
    """Ordered frame list from a rawf32 file, a netpbm file or a directory of
    them in sorted order (frameio.py:149-175)."""
    fmt, files = _resolve(path, fmt)
    if fmt == "rawf32":
        return load_rawf32(files[0])
    return [read_netpbm(p) for p in files]


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
    peak = float(e.max())
    write_pgm(path, e / peak if peak > 0.0 else np.zeros_like(e))
    return Path(path)
