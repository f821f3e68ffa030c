"""Data-parallel plumbing of the verify path (SURVEY §8 e): one process per GPU, independent
request cohorts per rank (weak scaling, no data-path collective).

The verify step is per-request independent (Alg. 2), so ranks shard requests with
no exchange.  Each rank draws its Philox streams from a disjoint request-id range
(request_id_base = rank << 32, reading C-8), so no two ranks ever reuse a uniform.  The only
collectives are the bench's timing/accounting reductions below (max time, summed units).
"""
from __future__ import annotations

import torch


def request_id_base(rank: int) -> int:
    """Disjoint 2^32-request Philox id range of `rank` (reading C-8)."""
    if rank < 0 or rank >= 1 << 31:
        raise ValueError("rank out of range")
    return rank << 32


def reduce_max_sum(values_max: list[float], values_sum: list[float], device=None):
    """All-reduce over the default group: MAX of values_max (per-rank device times -> the job's
    time), SUM of values_sum (units processed by all ranks).  Single-process: identity."""
    import torch.distributed as dist
    mx = torch.tensor(values_max, dtype=torch.float64, device=device)
    sm = torch.tensor(values_sum, dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    return mx.tolist(), sm.tolist()
