"""Deterministic input recipes shared by make_golden.py and the tests.

Frames are regenerated from these recipes (and checked against the hashes
stored in the fixtures) instead of being committed.
"""

import hashlib

import numpy as np


def fhash(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def _dup_block_frame(rng, shape, p):
    curr = rng.random(shape)
    dup = np.full((p, p), 0.5)
    dup[0, 0] = 0.52
    rows, cols = shape[0] // p, shape[1] // p
    blocks = curr.reshape(rows, p, cols, p).swapaxes(1, 2)
    for bi, bj in ((0, 1), (1, min(2, cols - 1)), (min(2, rows - 1), 0)):
        blocks[bi, bj] = dup
    return curr


def small_cases():
    """(name, prev, curr, cfg-dict) over the reference test shapes/buckets."""
    out = []
    rng = np.random.default_rng(20260)
    shapes = [((16, 16), 4), ((32, 32), 8), ((48, 48), 8), ((64, 64), 8), ((64, 64), 16),
              ((96, 96), 8), ((112, 112), 8), ((224, 224), 16), ((224, 224), 14), ((64, 96), 8)]
    for (shape, p) in shapes:
        for b in range(5):
            prev = rng.random(shape)
            cfg = {"patch_size": p}
            if b == 0:
                sh = (int(rng.integers(-shape[0] // 3, shape[0] // 3 + 1)),
                      int(rng.integers(-shape[1] // 3, shape[1] // 3 + 1)))
                curr = np.roll(prev, sh, axis=(0, 1))
            elif b == 1:
                curr = rng.random(shape)
                cfg["tau_mig"] = 1.0
            elif b == 2:
                curr = np.roll(prev, (int(rng.integers(-p, p + 1)), 0), axis=(0, 1))
                cfg["edge_lambda"] = -5.0
            elif b == 3:
                curr = np.roll(prev, (0, int(rng.integers(-p, p + 1))), axis=(0, 1))
                cfg["alpha_min"], cfg["alpha_max"] = 0.1, 0.2
            else:
                curr = _dup_block_frame(rng, shape, p)
                sh = (int(rng.integers(-3, 4)), int(rng.integers(-3, 4)))
                prev = np.roll(curr, (-sh[0], -sh[1]), axis=(0, 1))
            out.append((f"{shape[0]}x{shape[1]}p{p}b{b}", prev, curr, cfg))
    # degenerate frames (test_fusion.py:102-109)
    f = np.random.default_rng(8).random((32, 32))
    out.append(("black_prev", np.zeros((32, 32)), f, {"patch_size": 8}))
    out.append(("const_prev", np.full((32, 32), 0.5), f, {"patch_size": 8}))
    out.append(("black_curr", f, np.zeros((32, 32)), {"patch_size": 8}))
    out.append(("const_curr", f, np.full((32, 32), 0.25), {"patch_size": 8}))
    tile = np.random.default_rng(17).random((8, 8))
    out.append(("tied_tiles", np.tile(tile, (2, 2)), np.tile(tile, (2, 2)), {"patch_size": 8}))
    return out


C1 = dict(seed=1000, stream=0, steps=32, size=224, patch=14, alpha=(0.5, 0.5))
C2 = dict(seed=2000, streams=2, steps=14, size=448, patch=14, refresh_shift=1)


def compare_cases():
    """(name, frames, cfg-dict, edge_labels | None) for compare_domains
    (compare.py:55-114) over the shapes of test_compare.py."""
    out = []
    rng = np.random.default_rng(4242)
    base = rng.random((64, 64))
    out.append(("translate", [np.roll(base, (3 * t, 5 * t), axis=(0, 1)) for t in range(6)],
                {"patch_size": 8}, None))
    # persistent sharp rectangle over a smooth drifting background; labels =
    # patches crossed by the rectangle's boundary
    yy, xx = np.mgrid[0:96, 0:96] / 96.0
    frames, labels = [], []
    r0, r1, c0, c1 = 20, 61, 28, 75
    edge = set()
    for i in range(12):
        for j in range(12):
            ys, xs = set(range(8 * i, 8 * i + 8)), set(range(8 * j, 8 * j + 8))
            on_r = bool(ys & {r0, r1 - 1}) and bool(xs & set(range(c0, c1)))
            on_c = bool(xs & {c0, c1 - 1}) and bool(ys & set(range(r0, r1)))
            if on_r or on_c:
                edge.add(12 * i + j)
    for t in range(12):
        f = 0.25 + 0.2 * np.sin(2 * np.pi * (xx + 0.02 * t)) * np.cos(2 * np.pi * yy)
        f = f + 0.01 * rng.standard_normal((96, 96))
        f[r0:r1, c0:c1] = 1.0
        frames.append(f)
        labels.append(sorted(edge))
    out.append(("edge", frames, {"patch_size": 8}, labels))
    st = rng.random((64, 64))
    out.append(("static", [st.copy() for _ in range(6)],
                {"patch_size": 8, "edge_lambda": 1e15, "alpha_min": 0.4, "alpha_max": 0.4}, None))
    out.append(("random", [rng.random((32, 32)) for _ in range(3)], {"patch_size": 8}, None))
    out.append(("p14", [np.roll(rng.random((112, 112)), (t, 2 * t), axis=(0, 1)) for t in range(4)],
                {"patch_size": 14}, None))
    return out


def frameio_cases():
    """(name, suffix, file bytes) for the netpbm / rawf32 readers
    (frameio.py:29-175): valid files and every parse-failure branch."""
    import struct
    rng = np.random.default_rng(99)
    out = []
    out.append(("p5_small", ".pgm", b"P5\n2 2\n255\n" + bytes([0, 255, 128, 64])))
    out.append(("p5_comments", ".pgm", b"P5\n# made by hand\n3 2\n# maxval next\n255\n" + bytes(range(10, 16))))
    out.append(("p6_rand", ".ppm", b"P6 5 4 255\n" + rng.integers(0, 256, 60, dtype=np.uint8).tobytes()))
    out.append(("p5_extra_payload", ".pgm", b"P5\n2 1\n255\n" + bytes([7, 9, 11, 13])))
    out.append(("p5_truncated", ".pgm", b"P5\n4 4\n255\n" + bytes(10)))
    out.append(("bad_magic", ".pgm", b"P7\n2 2\n255\n" + bytes(4)))
    out.append(("short", ".pgm", b"P"))
    out.append(("trunc_header", ".pgm", b"P5\n3 "))
    out.append(("zero_dims", ".pgm", b"P5\n0 2\n255\n"))
    out.append(("maxval16", ".pgm", b"P5\n2 2\n65535\n" + bytes(8)))
    out.append(("non_numeric", ".pgm", b"P5\nab 2\n255\n" + bytes(4)))
    out.append(("no_pixels", ".pgm", b"P5\n2 2\n255"))
    fr = rng.random((2, 3, 4)).astype("<f4")
    head = b"FQC1" + struct.pack("<III", 3, 4, 2)
    out.append(("raw_ok", ".raw", head + fr.tobytes()))
    out.append(("raw_magic", ".raw", b"FQC2" + head[4:] + fr.tobytes()))
    out.append(("raw_short", ".raw", head[:10]))
    out.append(("raw_zero", ".raw", b"FQC1" + struct.pack("<III", 0, 4, 2)))
    out.append(("raw_trunc", ".raw", head + fr.tobytes()[:-5]))
    out.append(("raw_trailing", ".raw", head + fr.tobytes() + b"\x00"))
    bad = fr.copy()
    bad[1, 2, 3] = np.inf
    out.append(("raw_nonfinite", ".raw", head + bad.tobytes()))
    return out
