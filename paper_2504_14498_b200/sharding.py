"""Sharding of independent systems across ranks.

Batched independent systems (BASELINE.json cfg5) are the only workload on
this path that partitions without changing the preconditioner: each rank
(one process per GPU) solves a contiguous block of systems, and nothing is
exchanged until the final gather of the per-system reports to rank 0.
Single-system solves run as replicas.
"""

from __future__ import annotations

__all__ = ["shard", "gather_reports"]


def shard(n_units: int, rank: int, world: int) -> range:
    """Contiguous block of unit indices owned by `rank` (sizes differ by at
    most one, lower ranks take the remainder)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, rem = divmod(n_units, world)
    lo = rank * base + min(rank, rem)
    hi = lo + base + (1 if rank < rem else 0)
    return range(lo, hi)


def gather_reports(local: dict, world: int):
    """Gather {unit_index: report_dict} from every rank (torch.distributed
    must be initialised); returns the merged reports ordered by unit on
    every rank."""
    import torch.distributed as dist

    if world == 1:
        return [local[k] for k in sorted(local)]
    parts = [None] * world
    dist.all_gather_object(parts, local)
    merged = {}
    for p in parts:
        merged.update(p)
    return [merged[k] for k in sorted(merged)]
