"""Sharding of independent matrices across GPUs (one process per GPU).

The hot path does not partition a single matrix in this round (SURVEY.md
8(e): the reference elimination order is a sequential column chain); what
shards naturally is a batch of independent matrices -- an INLA
hyper-parameter sweep (BASELINE config 5) -- so each rank factors and inverts
its own contiguous slice with the batched device sweep, and the only
collectives are host-side plumbing (a barrier and a MAX of the per-rank time)
through torch.distributed.  No data-path collective exists.
"""
from __future__ import annotations


def shard_range(count: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [start, end) slice of `count` items for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank must satisfy 0 <= rank < world")
    base, extra = divmod(count, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def batch_seeds(first_seed: int, count: int, rank: int, world: int) -> list[int]:
    """Seeds of this rank's matrices in a sweep of `count` matrices seeded
    first_seed, first_seed + 1, ... (BASELINE config 5 uses 1000..1063)."""
    s, e = shard_range(count, rank, world)
    return [first_seed + k for k in range(s, e)]


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """MAX of a per-rank scalar (the bench reports the slowest rank's time)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
