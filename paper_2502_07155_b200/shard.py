"""Multi-rank orchestration of the node-parallel path (host logic only; no arithmetic of the method).

Algorithm 2's outputs are independent per node once the grid theta exists (step 3), so N
ranks each run their own plan on their own node shard with a replicated grid: no
data-path collective.  The only cross-rank operations are the timing reduction (max over ranks) and,
for strong-scaling use, the contiguous split of one node set.
"""
from __future__ import annotations


def node_shard(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [start, stop) slice of n_total nodes for `rank` (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def max_over_ranks(value: float, device=None) -> float:
    """All-reduce MAX of a per-rank time (torch.distributed, any backend); identity without a group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_rate(units_per_rank: int, world: int, max_ms: float) -> float:
    """Whole-job throughput: all units processed by all ranks / the slowest rank's time."""
    return units_per_rank * world / (max_ms * 1e-3)
