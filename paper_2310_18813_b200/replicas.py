"""Data-parallel replicas (7B / OPT-6.7B targets shard by request).

Sequences are independent, so N GPUs run N independent engines with no
data-path collective.  This module holds the only host logic that crosses
ranks: the deterministic request partition and the max-over-ranks timing
reduction (torch.distributed; NCCL on GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

import torch

__all__ = ["shard_requests", "max_over_ranks", "sum_over_ranks"]


def shard_requests(requests, rank: int, world: int):
    """Round-robin partition of a request list (order preserved per rank)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank/world {rank}/{world}")
    return [r for i, r in enumerate(requests) if i % world == rank]


def _reduce(value: float, op, device=None) -> float:
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=op)
    return float(t.item())


def max_over_ranks(value: float, device=None) -> float:
    """Job time = the slowest rank's time (the bench's timing rule)."""
    import torch.distributed as dist

    return _reduce(value, dist.ReduceOp.MAX, device)


def sum_over_ranks(value: float, device=None) -> float:
    import torch.distributed as dist

    return _reduce(value, dist.ReduceOp.SUM, device)
