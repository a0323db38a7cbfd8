"""Batch sharding across ranks: independent media need no collective on the
data path.  Each rank takes a contiguous slice of the members; torch.distributed is used only
for the barrier, the max-over-ranks time and gathering per-member traces at the end."""
from __future__ import annotations


def shard_members(total: int, world: int, rank: int) -> tuple[int, int]:
    """(first member, count) of this rank's slice; every member is owned by exactly one rank.
    Uneven totals put the remainder on the lowest ranks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if total < world:
        raise ValueError(f"{total} members cannot be sharded over {world} ranks")
    base, rem = divmod(total, world)
    count = base + (1 if rank < rem else 0)
    first = rank * base + min(rank, rem)
    return first, count


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_traces(iters, device=None):
    """All ranks' per-member iteration counts, in member order (rank 0 gets the full list)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(iters)
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, list(iters))
    return [x for part in out for x in part]
