"""Multi-GPU partitioning of the LLSA path.

Every (batch, head) unit runs the whole path independently, so units are
split into contiguous per-rank ranges with NO collective on the data path
(no NCCL traffic between compress, select, attention and backward).  The
only cross-rank operation is the max-over-ranks reduction of the step time
in bench.py.
"""
from __future__ import annotations


def shard_units(total_units: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, start+count) of `total_units` for `rank`; the first
    total_units % world ranks take one extra unit."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(total_units, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def max_over_ranks(value: float, group=None) -> float:
    """Step time as the maximum over ranks (any torch.distributed backend)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
