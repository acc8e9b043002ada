"""Frozen synthetic navigation-stream generator (BASELINE configs 1-5).

The reference ships no generator for the BASELINE workloads (its
``scenes.py`` only has cyclic-shift scenes), so this one is defined here and
frozen under ``GENERATOR_VERSION``; ``tests/golden`` pins frame hashes.
It stands in for the paper's R2R-CE observation streams (no dataset items
are used).  Parameterisation:

* scene RNG ``np.random.default_rng([seed, stream, scene])``;
* base = per channel, sum over sigma in {2, 8, 32} of N(0,1) noise blurred by
  circular convolution with the 4-sigma-truncated, normalised Gaussian
  (separable, i.e. ``gaussian_filter(mode='wrap', truncate=4)``), each
  normalised to unit std; then min-max to [0, 1] per channel;
* U{3..8} axis-aligned rectangles of constant U[0,1]^3 colour, sides
  U[H/16, H/3] (integers), PASTED (they replace the pixels);
* per step a translation U(-6, 6) px per axis and a zoom x U(1.00, 1.03),
  both cumulative, about the frame centre; bilinear sampling with
  half-sample-symmetric reflection at the border; clip to [0, 1];
* a hard cut every 12 frames (new scene, motion reset).

Two implementations share these formulas: ``numpy`` (the frozen one, used
for parity fixtures and the CPU baseline) and ``torch`` (same math on the
GPU for bulk benchmark inputs; its RNG stream differs, so its frames are a
different draw from the same distribution).
"""

from __future__ import annotations

import hashlib

import numpy as np

GENERATOR_VERSION = "fcb200-synth-v1"
SIGMAS = (2.0, 8.0, 32.0)
CUT_EVERY = 12
MAX_SHIFT = 6.0
MAX_ZOOM = 1.03


def _gauss_taps(sigma):
    radius = int(4.0 * sigma + 0.5)
    x = np.arange(-radius, radius + 1, dtype=np.float64)
    k = np.exp(-0.5 * (x / sigma) ** 2)
    return k / k.sum(), radius


def _circular_kernel_fft(n, sigma):
    """FFT of the truncated Gaussian wrapped onto a length-n circle."""
    taps, radius = _gauss_taps(sigma)
    circ = np.zeros(n, dtype=np.float64)
    for t, off in zip(taps, range(-radius, radius + 1)):
        circ[off % n] += t
    return np.fft.rfft(circ)


def _blur_wrap(img, sigma):
    h, w = img.shape
    kh = _circular_kernel_fft(h, sigma)
    kw = _circular_kernel_fft(w, sigma)
    f = np.fft.rfft(img, axis=1) * kw[None, :]
    out = np.fft.irfft(f, n=w, axis=1)
    f = np.fft.rfft(out, axis=0) * kh[:, None]
    return np.fft.irfft(f, n=h, axis=0)


def scene_params(seed, stream, scene, h, w):
    """All random draws of one scene, in a fixed order."""
    rng = np.random.default_rng([int(seed), int(stream), int(scene)])
    noise = rng.standard_normal((3, len(SIGMAS), h, w))
    n_rect = int(rng.integers(3, 9))
    lo_h, hi_h = max(1, h // 16), max(1, h // 3)
    lo_w, hi_w = max(1, w // 16), max(1, w // 3)
    rects = []
    for _ in range(n_rect):
        rh = int(rng.integers(lo_h, hi_h + 1))
        rw = int(rng.integers(lo_w, hi_w + 1))
        y0 = int(rng.integers(0, h - rh + 1))
        x0 = int(rng.integers(0, w - rw + 1))
        colour = rng.random(3)
        rects.append((y0, x0, rh, rw, colour))
    motion = [(float(rng.uniform(-MAX_SHIFT, MAX_SHIFT)),
               float(rng.uniform(-MAX_SHIFT, MAX_SHIFT)),
               float(rng.uniform(1.0, MAX_ZOOM))) for _ in range(CUT_EVERY)]
    return noise, rects, motion


def make_scene(seed, stream, scene, h, w):
    """(H, W, 3) float64 scene in [0, 1] plus its per-step motion draws."""
    noise, rects, motion = scene_params(seed, stream, scene, h, w)
    base = np.empty((h, w, 3))
    for c in range(3):
        acc = np.zeros((h, w))
        for s, sigma in enumerate(SIGMAS):
            b = _blur_wrap(noise[c, s], sigma)
            sd = b.std()
            acc += b / sd if sd > 0 else b
        lo, hi = acc.min(), acc.max()
        base[..., c] = (acc - lo) / (hi - lo) if hi > lo else 0.0
    for y0, x0, rh, rw, colour in rects:
        base[y0:y0 + rh, x0:x0 + rw, :] = colour
    return base, motion


def _reflect(idx, n):
    m = np.mod(idx, 2 * n)
    return np.where(m >= n, 2 * n - 1 - m, m)


def warp(scene, ty, tx, zoom):
    """Bilinear sample of ``scene`` at centre + (p - centre)/zoom - t."""
    h, w, _ = scene.shape
    cy, cx = (h - 1) / 2.0, (w - 1) / 2.0
    sy = cy + (np.arange(h, dtype=np.float64) - cy) / zoom - ty
    sx = cx + (np.arange(w, dtype=np.float64) - cx) / zoom - tx
    y0 = np.floor(sy)
    x0 = np.floor(sx)
    fy = (sy - y0)[:, None, None]
    fx = (sx - x0)[None, :, None]
    y0 = y0.astype(np.int64)
    x0 = x0.astype(np.int64)
    ya, yb = _reflect(y0, h), _reflect(y0 + 1, h)
    xa, xb = _reflect(x0, w), _reflect(x0 + 1, w)
    top = scene[ya][:, xa] * (1 - fx) + scene[ya][:, xb] * fx
    bot = scene[yb][:, xa] * (1 - fx) + scene[yb][:, xb] * fx
    return top * (1 - fy) + bot * fy


def motion_state(motion, k):
    """Cumulative (ty, tx, zoom) after k steps into a scene (k=0: identity)."""
    ty = tx = 0.0
    z = 1.0
    for dy, dx, dz in motion[:k]:
        ty += dy
        tx += dx
        z *= dz
    return ty, tx, z


def stream_frames(seed, stream, steps, h, w):
    """fp32 RGB frames (steps, H, W, 3) of one stream, numpy (frozen)."""
    out = np.empty((steps, h, w, 3), dtype=np.float32)
    cache = {}
    for t in range(steps):
        scene, k = divmod(t, CUT_EVERY)
        if scene not in cache:
            cache.clear()
            cache[scene] = make_scene(seed, stream, scene, h, w)
        base, motion = cache[scene]
        ty, tx, z = motion_state(motion, k)
        out[t] = np.clip(warp(base, ty, tx, z), 0.0, 1.0).astype(np.float32)
    return out


def frame_hash(frame):
    a = np.ascontiguousarray(frame)
    return hashlib.sha256(a.tobytes()).hexdigest()[:16]


# ------------------------------------------------------------------ torch --

def torch_stream_frames(streams, steps, h, w, seed, device, t0=0):
    """Same parameterisation on the GPU (torch RNG; bulk benchmark inputs).

    Returns a (steps, streams, H, W, 3) float32 tensor on ``device``.
    Frames ``t0 .. t0+steps-1`` of each stream.
    """
    import torch

    dev = torch.device(device)
    g = torch.Generator(device=dev)
    out = torch.empty((steps, streams, h, w, 3), dtype=torch.float32, device=dev)
    fy = {s: torch.as_tensor(_circular_kernel_fft(h, s), device=dev) for s in SIGMAS}
    fx = {s: torch.as_tensor(_circular_kernel_fft(w, s), device=dev) for s in SIGMAS}
    cy, cx = (h - 1) / 2.0, (w - 1) / 2.0
    ar_h = torch.arange(h, dtype=torch.float64, device=dev)
    ar_w = torch.arange(w, dtype=torch.float64, device=dev)

    def refl(i, n):
        m = torch.remainder(i, 2 * n)
        return torch.where(m >= n, 2 * n - 1 - m, m)

    scene_cache = {}
    for t in range(t0, t0 + steps):
        scene, k = divmod(t, CUT_EVERY)
        if scene not in scene_cache:
            scene_cache.clear()
            g.manual_seed(int(seed) * 1000003 + scene)
            noise = torch.randn((streams, 3, len(SIGMAS), h, w), generator=g,
                                device=dev, dtype=torch.float64)
            acc = torch.zeros((streams, 3, h, w), dtype=torch.float64, device=dev)
            for si, s in enumerate(SIGMAS):
                f = torch.fft.rfft(noise[:, :, si], dim=-1) * fx[s]
                b = torch.fft.irfft(f, n=w, dim=-1)
                f = torch.fft.rfft(b, dim=-2) * fy[s][:, None]
                b = torch.fft.irfft(f, n=h, dim=-2)
                sd = b.std(dim=(-2, -1), keepdim=True, unbiased=False)
                acc += b / sd.clamp_min(1e-300)
            lo = acc.amin(dim=(-2, -1), keepdim=True)
            hi = acc.amax(dim=(-2, -1), keepdim=True)
            base = ((acc - lo) / (hi - lo).clamp_min(1e-300)).permute(0, 2, 3, 1).contiguous()
            nrect = torch.randint(3, 9, (streams,), generator=g, device=dev)
            for r in range(8):
                rh = torch.randint(max(1, h // 16), max(1, h // 3) + 1, (streams,), generator=g, device=dev)
                rw = torch.randint(max(1, w // 16), max(1, w // 3) + 1, (streams,), generator=g, device=dev)
                y0 = (torch.rand(streams, generator=g, device=dev, dtype=torch.float64) * (h - rh + 1)).long()
                x0 = (torch.rand(streams, generator=g, device=dev, dtype=torch.float64) * (w - rw + 1)).long()
                col = torch.rand((streams, 3), generator=g, device=dev, dtype=torch.float64)
                on = (r < nrect)
                my = (ar_h[None, :] >= y0[:, None]) & (ar_h[None, :] < (y0 + rh)[:, None])
                mx = (ar_w[None, :] >= x0[:, None]) & (ar_w[None, :] < (x0 + rw)[:, None])
                m = (my[:, :, None] & mx[:, None, :] & on[:, None, None])[..., None]
                base = torch.where(m, col[:, None, None, :], base)
            mot = torch.rand((streams, CUT_EVERY, 3), generator=g, device=dev, dtype=torch.float64)
            dy = (mot[..., 0] * 2 - 1) * MAX_SHIFT
            dx = (mot[..., 1] * 2 - 1) * MAX_SHIFT
            dz = 1.0 + mot[..., 2] * (MAX_ZOOM - 1.0)
            scene_cache[scene] = (base, dy, dx, dz)
        base, dy, dx, dz = scene_cache[scene]
        ty = dy[:, :k].sum(dim=1)
        tx = dx[:, :k].sum(dim=1)
        z = dz[:, :k].prod(dim=1)
        sy = cy + (ar_h[None, :] - cy) / z[:, None] - ty[:, None]
        sx = cx + (ar_w[None, :] - cx) / z[:, None] - tx[:, None]
        y0 = torch.floor(sy)
        x0 = torch.floor(sx)
        wy = (sy - y0)[:, :, None, None]
        wx = (sx - x0)[:, None, :, None]
        y0 = y0.long()
        x0 = x0.long()
        ya, yb = refl(y0, h), refl(y0 + 1, h)
        xa, xb = refl(x0, w), refl(x0 + 1, w)
        bidx = torch.arange(streams, device=dev)[:, None, None]

        def gather(yy, xx):
            return base[bidx, yy[:, :, None], xx[:, None, :]]

        top = gather(ya, xa) * (1 - wx) + gather(ya, xb) * wx
        bot = gather(yb, xa) * (1 - wx) + gather(yb, xb) * wx
        out[t - t0] = (top * (1 - wy) + bot * wy).clamp_(0.0, 1.0).to(torch.float32)
    return out
