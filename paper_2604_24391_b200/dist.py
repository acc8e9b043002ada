"""Multi-GPU plumbing: streams shard by rank, no collective on the hot path.

Each rank (one process per GPU) owns a contiguous block of independent
navigation streams; per-stream state never crosses ranks.
The only collectives are the end-of-run metric gather and the max-over-
ranks timing, both a few bytes (NCCL over NVLink on GPUs, gloo in tests).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

COUNTERS = ("frames", "tokens", "reused_tokens", "flushes", "cold")


def shard(total_streams, world, rank):
    """Contiguous block [lo, hi) of streams owned by ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(int(total_streams), int(world))
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def max_over_ranks(value, device=None):
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_counters(counts, device=None):
    """Sum per-rank decision counters (dict over COUNTERS) across ranks."""
    t = torch.tensor([float(counts.get(k, 0)) for k in COUNTERS], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return {k: float(v) for k, v in zip(COUNTERS, t.tolist())}


def step_counters(host_results):
    """Counters of one select step from the fc_stream_result records."""
    r = host_results
    n = (r["rows"] * r["cols"]).astype("int64")
    return {
        "frames": int(len(r)),
        "tokens": int(n.sum()),
        "reused_tokens": int(r["k_final"].sum()),
        "flushes": int((r["flushed"] & (r["cold"] == 0)).sum()),
        "cold": int(r["cold"].sum()),
    }
