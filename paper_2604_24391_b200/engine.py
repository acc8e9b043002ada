"""Batched device API over the C ABI: many independent streams per GPU.

``FreqCacheEngine`` owns one ``fc_plan`` (geometry), the per-stream state
(previous-frame spectrum + flags) and the scratch workspace, all in device
memory allocated through torch.  ``select`` runs one decision step for every
stream (reference ``decide``, fusion.py:121-242, batched); ``splice`` applies
the decisions to the hidden-state cache (reference ``step``,
fusion.py:462-512).  Everything is stream-ordered on torch's current CUDA
stream, so whole steps can be captured in a CUDA graph.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

from . import _native as nat

_FORMATS = {
    "rgb": (nat.FC_FMT_RGB_F32, torch.float32, 3),
    "gray32": (nat.FC_FMT_GRAY_F32, torch.float32, 1),
    "gray64": (nat.FC_FMT_GRAY_F64, torch.float64, 1),
    "gray_u8": (nat.FC_FMT_GRAY_U8, torch.uint8, 1),   # PGM P5 payload, gray = v / 255
    "rgb_u8": (nat.FC_FMT_RGB_U8, torch.uint8, 3),     # PPM P6 payload, gray = luma / 255
}


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def _stream(device=None):
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def make_config(cfg, refresh_shift=None):
    """CacheConfig-like object -> fc_config."""
    b = getattr(cfg, "budget", None)
    amin = b.alpha_min if b is not None else getattr(cfg, "alpha_min", 0.08)
    amax = b.alpha_max if b is not None else getattr(cfg, "alpha_max", 0.5)
    rs = refresh_shift if refresh_shift is not None else getattr(cfg, "refresh_shift", None)
    return nat.Config(float(cfg.tau_mig), float(cfg.edge_lambda), float(amin), float(amax),
                      -1 if rs is None else int(rs), 0)


@dataclass
class SelectResult:
    """Device outputs of one ``select`` step (N = rows*cols tokens)."""

    results: torch.Tensor        # [B, 136] uint8 (fc_stream_result records)
    reuse_idx: torch.Tensor      # [B, N] int32, ascending (E, idx), -1 padded
    recompute_idx: torch.Tensor  # [B, N] int32 row-major, -1 padded
    src_map: torch.Tensor        # [B, N] int32 splice map
    reuse_mask: torch.Tensor     # [B, N] uint8
    refresh_mask: torch.Tensor   # [B, N] uint8
    energy: torch.Tensor         # [B, N] float64
    counters: torch.Tensor = None  # optional int64 [4]: frames, reused tokens, flushes, cold (accumulated)

    def host_results(self):
        return self.results.cpu().numpy().view(nat.RESULT_DTYPE).reshape(-1)


class FreqCacheEngine:
    """Per-GPU batch of ``batch`` independent streams of (H, W) frames."""

    def __init__(self, batch, height, width, patch_size, fmt="rgb", device=None):
        if fmt not in _FORMATS:
            raise ValueError(f"unknown frame format {fmt!r}")
        self.lib = nat.lib()
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.fmt = fmt
        self.format_code, self.dtype, self.channels = _FORMATS[fmt]
        self.batch, self.height, self.width, self.patch_size = int(batch), int(height), int(width), int(patch_size)
        geom = nat.Geometry(self.batch, self.height, self.width, self.patch_size, self.format_code)
        plan = C.c_void_p()
        with torch.cuda.device(self.device):
            rc = self.lib.fc_plan_create(C.byref(geom), C.byref(plan))
        nat.check(rc, "fc_plan_create")
        self._plan = plan
        self.rows = self.height // self.patch_size
        self.cols = self.width // self.patch_size
        self.n_tokens = self.lib.fc_plan_tokens(plan)
        self.launches_per_select = self.lib.fc_plan_launches(plan)
        # select_front + select_back of one step: K_A, K_D1 | K_B, K_C, K_D
        # over the whole batch (FC_SPLIT_LANES=1: the plan's chunks instead)
        self.launches_per_split_step = (self.launches_per_select
                                        if os.environ.get("FC_SPLIT_LANES") == "1" else 5)
        sb = self.lib.fc_plan_state_bytes(plan)
        wb = self.lib.fc_plan_workspace_bytes(plan)
        self.state = torch.zeros(sb, dtype=torch.uint8, device=self.device)
        self.workspace = torch.zeros(wb, dtype=torch.uint8, device=self.device)
        self.out = self.new_output()
        self.reset()

    def __del__(self):
        plan = getattr(self, "_plan", None)
        if plan is not None and plan.value:
            try:
                self.lib.fc_plan_destroy(plan)
            except Exception:
                pass
            self._plan = None

    # ------------------------------------------------------------------
    def new_output(self):
        B, N, dev = self.batch, self.n_tokens, self.device
        return SelectResult(
            results=torch.zeros((B, nat.RESULT_DTYPE.itemsize), dtype=torch.uint8, device=dev),
            reuse_idx=torch.empty((B, N), dtype=torch.int32, device=dev),
            recompute_idx=torch.empty((B, N), dtype=torch.int32, device=dev),
            src_map=torch.empty((B, N), dtype=torch.int32, device=dev),
            reuse_mask=torch.empty((B, N), dtype=torch.uint8, device=dev),
            refresh_mask=torch.empty((B, N), dtype=torch.uint8, device=dev),
            energy=torch.empty((B, N), dtype=torch.float64, device=dev),
        )

    def reset(self, first=0, count=None):
        """Mark streams cold (populate_cache semantics, fusion.py:450-459)."""
        count = self.batch - first if count is None else count
        with torch.cuda.device(self.device):
            nat.check(self.lib.fc_state_reset(self._plan, _ptr(self.state), int(first), int(count),
                                              _stream(self.device)), "fc_state_reset")

    def frame_shape(self):
        if self.channels == 3:
            return (self.batch, self.height, self.width, 3)
        return (self.batch, self.height, self.width)

    def _check_frames(self, frames):
        if not isinstance(frames, torch.Tensor) or frames.device != self.device:
            raise ValueError("frames must be a tensor on the engine's device")
        if frames.dtype != self.dtype or tuple(frames.shape) != self.frame_shape():
            raise ValueError(f"frames must be {self.dtype} of shape {self.frame_shape()}, "
                             f"got {frames.dtype} {tuple(frames.shape)}")
        if not frames.is_contiguous():
            raise ValueError("frames must be contiguous")

    def select(self, frames, cfg, out=None, refresh_shift=None, profile=None):
        """One decision step for every stream; returns device outputs.
        ``profile``: a list that receives per-kernel device ms (rows_fwd,
        cols, rows_inv, select, rank) — launches serially and synchronises."""
        self._check_frames(frames)
        out = self.out if out is None else out
        so = self._select_out(out)
        conf = make_config(cfg, refresh_shift)
        with torch.cuda.device(self.device):
            if profile is None:
                rc = self.lib.fc_select(self._plan, C.byref(conf), _ptr(frames), _ptr(self.state),
                                        _ptr(self.workspace), C.byref(so), _stream(self.device))
            else:
                ms = (C.c_float * 5)()
                rc = self.lib.fc_select_profile(self._plan, C.byref(conf), _ptr(frames), _ptr(self.state),
                                                _ptr(self.workspace), C.byref(so), ms, _stream(self.device))
                profile[:] = list(ms)
        nat.check(rc, "fc_select")
        return out

    def _select_out(self, out):
        if out.counters is not None and (out.counters.dtype != torch.int64 or out.counters.numel() < 4
                                         or out.counters.device != self.device):
            raise ValueError("counters must be an int64 tensor of >= 4 elements on the engine's device")
        return nat.SelectOut(out.results.data_ptr(), out.reuse_idx.data_ptr(), out.recompute_idx.data_ptr(),
                             out.src_map.data_ptr(), out.reuse_mask.data_ptr(), out.refresh_mask.data_ptr(),
                             out.energy.data_ptr(), out.counters.data_ptr() if out.counters is not None else None)

    def select_front(self, frames, cfg, out, slot, refresh_shift=None):
        """Front half of a step (``fc_select_front``): energies, refresh mask,
        token order and row spectra of ``frames`` into workspace ``slot``.
        Pair with :meth:`select_back` on the same ``out`` and ``slot``; the
        front of step t + 1 (other slot) may overlap the back of step t."""
        self._check_frames(frames)
        so = self._select_out(out)
        conf = make_config(cfg, refresh_shift)
        with torch.cuda.device(self.device):
            rc = self.lib.fc_select_front(self._plan, C.byref(conf), _ptr(frames), _ptr(self.workspace),
                                          C.byref(so), int(slot), _stream(self.device))
        nat.check(rc, "fc_select_front")
        return out

    def select_back(self, cfg, out, slot, refresh_shift=None):
        """Back half of a step (``fc_select_back``): column FFTs, state swap,
        phase correlation and the decision, from workspace ``slot``."""
        so = self._select_out(out)
        conf = make_config(cfg, refresh_shift)
        with torch.cuda.device(self.device):
            rc = self.lib.fc_select_back(self._plan, C.byref(conf), _ptr(self.state), _ptr(self.workspace),
                                         C.byref(so), int(slot), _stream(self.device))
        nat.check(rc, "fc_select_back")
        return out

    def patch_energy(self, frames, energy=None):
        self._check_frames(frames)
        if energy is None:
            energy = torch.empty((self.batch, self.n_tokens), dtype=torch.float64, device=self.device)
        with torch.cuda.device(self.device):
            rc = self.lib.fc_patch_energy(self._plan, _ptr(frames), _ptr(self.workspace), _ptr(energy),
                                          _stream(self.device))
        nat.check(rc, "fc_patch_energy")
        return energy


    def compare_cosines(self, prev, curr, visual=None, naive=None):
        """Per-patch (visual, naive_freq) cosines of this engine's B frame
        pairs (see :func:`compare_cosines`)."""
        self._check_frames(prev)
        self._check_frames(curr)
        return compare_cosines(prev, curr, self.patch_size, visual, naive)


def compare_cosines(prev, curr, patch_size, visual=None, naive=None):
    """Per-patch (visual, naive_freq) cosines of B frame pairs — the two
    position-wise baseline policies of compare.py:23-52 — as [B, N] float64
    device tensors.  Frames: [B, H, W] float64 / float32 or [B, H, W, 3]
    float32 RGB (luma adapter), contiguous on one CUDA device."""
    lib = nat.lib()
    if prev.shape != curr.shape or prev.dtype != curr.dtype or prev.device != curr.device:
        raise ValueError("prev and curr must share shape, dtype and device")
    if not (prev.is_cuda and prev.is_contiguous() and curr.is_contiguous()):
        raise ValueError("frames must be contiguous CUDA tensors")
    if prev.dim() == 4 and prev.shape[-1] == 3 and prev.dtype == torch.float32:
        fmt = nat.FC_FMT_RGB_F32
    elif prev.dim() == 3 and prev.dtype == torch.float32:
        fmt = nat.FC_FMT_GRAY_F32
    elif prev.dim() == 3 and prev.dtype == torch.float64:
        fmt = nat.FC_FMT_GRAY_F64
    elif prev.dim() == 3 and prev.dtype == torch.uint8:
        fmt = nat.FC_FMT_GRAY_U8
    elif prev.dim() == 4 and prev.shape[-1] == 3 and prev.dtype == torch.uint8:
        fmt = nat.FC_FMT_RGB_U8
    else:
        raise ValueError(f"unsupported frame layout {prev.dtype} {tuple(prev.shape)}")
    B, H, W = (int(v) for v in prev.shape[:3])
    p = int(patch_size)
    if p < 2 or H % p or W % p:
        raise ValueError(f"patch size {p} does not divide frame dimensions {H}x{W}")
    shape = (B, (H // p) * (W // p))
    if visual is None:
        visual = torch.empty(shape, dtype=torch.float64, device=prev.device)
    if naive is None:
        naive = torch.empty(shape, dtype=torch.float64, device=prev.device)
    geom = nat.Geometry(B, H, W, p, fmt)
    with torch.cuda.device(prev.device):
        rc = lib.fc_compare_cosines(C.byref(geom), _ptr(prev), _ptr(curr), _ptr(visual), _ptr(naive),
                                    _stream(prev.device))
    nat.check(rc, "fc_compare_cosines")
    return visual, naive


def gather_patches(frames, patch_size, index, out=None):
    """bf16 [T, 3 P^2] pixels of the tokens ``index`` (int64 [T], b * N + p)
    of fp32 RGB frames [B, H, W, 3], in a ViT patch embedding's (py, px, c)
    order (``fc_gather_patches``)."""
    lib = nat.lib()
    if frames.dtype != torch.float32 or frames.dim() != 4 or frames.shape[-1] != 3 or not frames.is_contiguous():
        raise ValueError("frames must be a contiguous float32 [B, H, W, 3] tensor")
    if index.dtype != torch.int64 or index.dim() != 1 or not index.is_contiguous():
        raise ValueError("index must be a contiguous int64 [T] tensor")
    B, H, W, _ = (int(v) for v in frames.shape)
    p = int(patch_size)
    if out is None:
        out = torch.empty((index.numel(), 3 * p * p), dtype=torch.bfloat16, device=frames.device)
    rc = lib.fc_gather_patches(int(index.numel()), B, H, W, p, _ptr(frames), _ptr(index), _ptr(out),
                               _stream(frames.device))
    nat.check(rc, "fc_gather_patches")
    return out


def row_cosines(a, b, out=None):
    """Row-wise cosine of two [n, d] float64 device stacks (compare.py:28-38)."""
    lib = nat.lib()
    if a.shape != b.shape or a.dim() != 2 or a.dtype != torch.float64 or b.dtype != torch.float64:
        raise ValueError("row_cosines needs two float64 [n, d] tensors of one shape")
    if not (a.is_cuda and b.is_cuda and a.is_contiguous() and b.is_contiguous()):
        raise ValueError("row_cosines operands must be contiguous CUDA tensors")
    if out is None:
        out = torch.empty(a.shape[0], dtype=torch.float64, device=a.device)
    with torch.cuda.device(a.device):
        rc = lib.fc_row_cosines(int(a.shape[0]), int(a.shape[1]), _ptr(a), _ptr(b), _ptr(out),
                                _stream(a.device))
    nat.check(rc, "fc_row_cosines")
    return out


def _status_word(device):
    return torch.zeros(1, dtype=torch.int32, device=device)


def check_status(status, what="splice"):
    """Raise the reference's AssertionError (fusion.py:488-490) if a splice
    kernel flagged an out-of-bounds source in ``status`` (synchronises)."""
    code = int(status.reshape(-1)[0].item())
    if code != nat.FC_OK:
        nat.check(code, what)


def splice(src_map, cache, cache_ages, fresh, out, out_ages, compact=False, status=None):
    """Token splice on device (fusion.py:462-512), any element type.

    src_map [B, N] int32; cache/fresh/out [B, N, D] (fresh may be [B, K, D]
    front-packed when ``compact``); ages int64 [B, N].  ``cache`` may be None
    when no entry of src_map is >= 0 (cold start / flush).

    Every row's source is bounds-checked on the device (fusion.py:488-490).
    With ``status=None`` the call allocates a status word and checks it after
    the splice (one synchronisation), raising ``AssertionError`` on a bad
    source; pass a zeroed device int32 tensor to keep the call asynchronous
    and check it later with :func:`check_status`.
    """
    lib = nat.lib()
    if src_map.dtype != torch.int32 or src_map.dim() != 2:
        raise ValueError("src_map must be an int32 [B, N] tensor")
    B, N = src_map.shape
    row_bytes = out.shape[-1] * out.element_size()
    for t in (src_map, fresh, out, out_ages) + ((cache, cache_ages) if cache is not None else ()):
        if not t.is_cuda or not t.is_contiguous():
            raise ValueError("splice operands must be contiguous CUDA tensors")
    if cache is not None and (cache.dtype != out.dtype or cache.shape != out.shape):
        raise ValueError("cache and out must share dtype and shape")
    if fresh.dtype != out.dtype or fresh.shape[-1] != out.shape[-1]:
        raise ValueError("fresh rows must match out's dtype and row width")
    if fresh.dim() != 3 or fresh.shape[0] != B or (not compact and fresh.shape[1] != N):
        raise ValueError("fresh must be [B, N, D] (dense) or [B, K, D] (compact)")
    st = _status_word(out.device) if status is None else status
    rc = lib.fc_splice(int(B), int(N), int(row_bytes), _ptr(src_map), _ptr(cache),
                       _ptr(cache_ages), _ptr(fresh),
                       nat.FC_FRESH_COMPACT if compact else nat.FC_FRESH_DENSE, int(fresh.shape[1]),
                       _ptr(out), _ptr(out_ages), _ptr(st), _stream(out.device))
    nat.check(rc, "fc_splice")
    if status is None:
        check_status(st, "fc_splice")
    return out, out_ages


def splice_packed(src_map, cache, cache_ages, fresh_values, fresh_offsets, out, out_ages, status=None):
    """Splice with ragged fresh rows: stream b's k-th recomputed token is
    ``fresh_values[fresh_offsets[b] + k]`` ([total, D]; offsets int64 [B]).
    ``status`` as in :func:`splice`."""
    lib = nat.lib()
    B, N = src_map.shape
    row_bytes = out.shape[-1] * out.element_size()
    if fresh_values.dim() != 2 or fresh_values.shape[-1] != out.shape[-1] or fresh_values.dtype != out.dtype:
        raise ValueError("fresh_values must be [total, D] with out's dtype")
    if fresh_offsets.dtype != torch.int64 or fresh_offsets.numel() < B:
        raise ValueError("fresh_offsets must be int64 [B]")
    for t in (src_map, fresh_values, fresh_offsets, out, out_ages) + ((cache, cache_ages) if cache is not None else ()):
        if not t.is_cuda or not t.is_contiguous():
            raise ValueError("splice operands must be contiguous CUDA tensors")
    if cache is not None and (cache.dtype != out.dtype or cache.shape != out.shape):
        raise ValueError("cache and out must share dtype and shape")
    st = _status_word(out.device) if status is None else status
    rc = lib.fc_splice_packed(int(B), int(N), int(row_bytes), _ptr(src_map), _ptr(cache), _ptr(cache_ages),
                              _ptr(fresh_values), _ptr(fresh_offsets), _ptr(out), _ptr(out_ages), _ptr(st),
                              _stream(out.device))
    nat.check(rc, "fc_splice_packed")
    if status is None:
        check_status(st, "fc_splice_packed")
    return out, out_ages


class SpliceState:
    """Ping-pong token cache for in-place splicing (``fc_splice_inplace``).

    ``cache`` [2, B, N, D] and ``ages`` [2, B, N]; ``slot[b]`` names the
    buffer that holds stream b's current cache (``current()`` gathers views).
    Steps stay asynchronous: a malformed ``src_map`` row is skipped on the
    device and recorded in ``status``; :meth:`check` raises the reference's
    ``AssertionError`` (fusion.py:488-490) for it.
    """

    def __init__(self, cache, ages):
        if cache.dim() != 4 or cache.shape[0] != 2 or ages.shape != cache.shape[:3]:
            raise ValueError("cache must be [2, B, N, D] and ages [2, B, N]")
        self.cache, self.ages = cache, ages
        B = cache.shape[1]
        self.slots = [torch.zeros(B, dtype=torch.uint8, device=cache.device) for _ in range(2)]
        self.k = 0
        nb = nat.lib().fc_splice_inplace_scratch_bytes(int(B), int(cache.shape[2]))
        self.scratch = torch.empty(nb, dtype=torch.uint8, device=cache.device)
        self.status = _status_word(cache.device)
        self.plan_done = None      # event after the last boostable splice's plan
        self._boost_args = None

    @property
    def slot(self):
        return self.slots[self.k]

    def step(self, src_map, fresh, compact=False, boostable=False):
        """One splice on the current stream.  ``boostable``: issued as plan +
        copy with an event between them, so :meth:`boost` can later add
        copier CTAs to this splice from another stream."""
        lib = nat.lib()
        dev = self.cache.device
        if (src_map.dtype != torch.int32 or tuple(src_map.shape) != tuple(self.cache.shape[1:3])
                or not src_map.is_contiguous() or src_map.device != dev):
            raise ValueError(f"src_map must be a contiguous int32 {tuple(self.cache.shape[1:3])} tensor "
                             "on the cache's device")
        B, N = src_map.shape
        row_bytes = self.cache.shape[-1] * self.cache.element_size()
        if fresh.dtype != self.cache.dtype or fresh.shape[-1] != self.cache.shape[-1] or fresh.shape[0] != B:
            raise ValueError("fresh must be [B, *, D] with the cache dtype")
        if fresh.dim() != 3 or not fresh.is_contiguous() or fresh.device != dev:
            raise ValueError("fresh must be a contiguous [B, *, D] tensor on the cache's device")
        if not compact and fresh.shape[1] != N:
            raise ValueError("dense fresh must be [B, N, D]")
        sin, sout = self.slots[self.k], self.slots[1 - self.k]
        layout = nat.FC_FRESH_COMPACT if compact else nat.FC_FRESH_DENSE
        args = (int(B), int(N), int(row_bytes), _ptr(src_map), _ptr(self.cache[0]), _ptr(self.cache[1]),
                _ptr(self.ages[0]), _ptr(self.ages[1]), _ptr(sin), _ptr(sout), _ptr(fresh), layout,
                int(fresh.shape[1]), _ptr(self.scratch))
        st = _stream(self.cache.device)
        if boostable:
            nat.check(lib.fc_splice_inplace_plan(*args, st), "fc_splice_inplace_plan")
            if self.plan_done is None:
                self.plan_done = torch.cuda.Event()
            self.plan_done.record(torch.cuda.current_stream(dev))
            nat.check(lib.fc_splice_inplace_copy(*args, _ptr(self.status), 0, st), "fc_splice_inplace_copy")
            self._boost_args = args
        else:
            rc = lib.fc_splice_inplace(*args, _ptr(self.status), st)
            nat.check(rc, "fc_splice_inplace")
            self._boost_args = None
        self.k = 1 - self.k
        return self.slot

    def boost(self, ctas):
        """Add ``ctas`` copier CTAs, on the current stream, to the last
        ``boostable`` splice: they wait for its plan and take only rows no
        copier has claimed yet (fc_splice_inplace_copy).  Must complete before
        the next step's splice (join the streams); that step's ``src_map`` and
        ``fresh`` tensors must stay alive until then (the launch reads them)."""
        if self._boost_args is None:
            raise RuntimeError("boost() needs a preceding step(..., boostable=True)")
        dev = self.cache.device
        torch.cuda.current_stream(dev).wait_event(self.plan_done)
        nat.check(nat.lib().fc_splice_inplace_copy(*self._boost_args, _ptr(self.status), int(ctas),
                                                   _stream(dev)), "fc_splice_inplace_copy")

    def check(self):
        """Raise AssertionError if any step so far met an out-of-bounds
        source (synchronises); clears the status word."""
        try:
            check_status(self.status, "fc_splice_inplace")
        finally:
            self.status.zero_()

    def current(self):
        """[B, N, D] tokens and [B, N] ages of every stream's current cache."""
        idx = self.slot.long()
        b = torch.arange(idx.numel(), device=idx.device)
        return self.cache[idx, b], self.ages[idx, b]


class StepGraph:
    """One captured step: everything ``fn()`` launches on the current CUDA
    stream (and on streams forked from it through events) is recorded once
    and replayed with a single graph launch (``fc_graph_*``).  ``fn`` must
    not allocate device memory (all buffers exist before capture)."""

    def __init__(self, fn, device=None):
        self.lib = nat.lib()
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        # the legacy default stream cannot be captured: capture on a side
        # stream ordered after the caller's work
        cap = torch.cuda.Stream(self.device)
        cap.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(cap):
            st = _stream(self.device)
            nat.check(self.lib.fc_graph_capture_begin(st), "fc_graph_capture_begin")
            try:
                fn()
            finally:
                ex = C.c_void_p()
                rc = self.lib.fc_graph_capture_end(st, C.byref(ex))
        nat.check(rc, "fc_graph_capture_end")
        self._exec = ex

    def replay(self):
        nat.check(self.lib.fc_graph_launch(self._exec, _stream(self.device)), "fc_graph_launch")

    def __del__(self):
        ex = getattr(self, "_exec", None)
        if ex is not None and ex.value:
            try:
                self.lib.fc_graph_destroy(ex)
            except Exception:
                pass
            self._exec = None


def splice_map(rows, cols, reuse_idx, di_patches, dj_patches, src_map=None, flag=None):
    """Device src_map for one stream from an ordered reuse list."""
    lib = nat.lib()
    dev = reuse_idx.device if reuse_idx is not None and reuse_idx.numel() else torch.device("cuda")
    if src_map is None:
        src_map = torch.empty(rows * cols, dtype=torch.int32, device=dev)
    k = 0 if reuse_idx is None else int(reuse_idx.numel())
    rc = lib.fc_splice_map(int(rows), int(cols), _ptr(reuse_idx if k else None), k, int(di_patches),
                           int(dj_patches), _ptr(src_map), _ptr(flag), _stream(dev))
    nat.check(rc, "fc_splice_map")
    return src_map
