"""Multi-GPU scenario sharding.

Scenarios are independent, so each rank owns a contiguous slice of
the global scenario range, generates it itself with the counter-based
generator (no data movement, identical data for every world size) and runs the
split sweep locally.  The only exchange step is ONE all-reduce(SUM) of the
int64 SAA partials (48 bytes per tour) over the process group -- NCCL over
NVLink/NVSwitch on GPUs, gloo in the CPU tests.  Integer partials make the
result bit-identical for every world size.
"""
from __future__ import annotations


def shard_range(S: int, rank: int, world: int) -> tuple[int, int]:
    """[begin, end) of the global scenarios owned by `rank`: floor(r S / R) .. floor((r+1) S / R)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return (rank * S) // world, ((rank + 1) * S) // world


def allreduce_partials(partial, group=None):
    """SUM the int64 partial tensor(s) across ranks, in place (one collective)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(partial, op=dist.ReduceOp.SUM, group=group)
    return partial


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a scalar over ranks (for device-timed multi-GPU numbers)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
