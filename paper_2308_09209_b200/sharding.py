"""Multi-GPU plumbing for independent panorama streams.

The per-frame path has no cross-stream data (all temporal state -- 3D-M
windows, threshold history, frame counter -- is per stream,
/root/reference/proj/include/stitch/pipeline.hpp:47-63), so streams shard
one-per-GPU with no collective on the data path.  torch.distributed is used
only for the barrier around the timed region and for reducing timings and
counts across ranks (NCCL on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import List


def stream_assignment(n_streams: int, world: int, rank: int) -> List[int]:
    """Stream ids served by `rank`: s mod world == rank (round-robin)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return [s for s in range(n_streams) if s % world == rank]


def _reduce(value: float, op: str, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op={"max": dist.ReduceOp.MAX, "sum": dist.ReduceOp.SUM,
                           "min": dist.ReduceOp.MIN}[op])
    return float(t.item())


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank duration: the whole job ends when the slowest rank does."""
    return _reduce(value, "max", device)


def sum_over_ranks(value: float, device=None) -> float:
    return _reduce(value, "sum", device)


def aggregate_throughput(units_per_rank: float, seconds_per_rank: float, device=None) -> float:
    """Whole-job units/s: units processed by all ranks / max rank time."""
    total = sum_over_ranks(units_per_rank, device)
    slowest = max_over_ranks(seconds_per_rank, device)
    return total / slowest if slowest > 0 else 0.0
