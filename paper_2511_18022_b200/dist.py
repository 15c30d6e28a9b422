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


def saa_estimate_f32(cost, group=None, moments_fn=None) -> dict:
    """fp32-mode SAA estimate over the costs of ALL ranks (DESIGN R25): two passes, each one
    all-reduce(SUM) of 4 doubles -- {m, sum} gives the global mean (spdp_saa_finalize_f32), then
    the squared deviations about it; the estimate itself is spdp_saa_finalize_f32 of the two
    summed passes (this function only moves the moments).  moments_fn(cost, center) -> float64
    tensor [4] defaults to the device kernel (spdp_saa_f32_moments)."""
    import torch.distributed as dist

    from paper_2511_18022_b200 import saa_finalize_f32
    if moments_fn is None:
        from paper_2511_18022_b200 import saa_f32_moments as moments_fn
    multi = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
    m1 = moments_fn(cost, 0.0)
    if multi:
        dist.all_reduce(m1, op=dist.ReduceOp.SUM, group=group)
    center = saa_finalize_f32(m1)["mean"]
    m2 = moments_fn(cost, center)
    if multi:
        dist.all_reduce(m2, op=dist.ReduceOp.SUM, group=group)
    return saa_finalize_f32(m1, m2)
