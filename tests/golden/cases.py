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
