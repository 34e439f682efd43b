"""Multi-GPU plumbing of the pass: tuples shard across ranks, each rank scores its
own shard from its own pool, and the only exchange is one all-reduce(SUM) of the int64 count
vector.  Integer sums make N-rank counts bit-identical to one rank.  torch.distributed supplies
the process group (NCCL on B200; gloo in the CPU tests)."""
from __future__ import annotations

from typing import Tuple


def shard_range(n_total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous tuple range [begin, end) of `rank` (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_total, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def shard_by_cost(costs, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous tuple range [begin, end) of `rank` balanced by per-tuple cost (SURVEY §8(e):
    algorithmic bytes, the full-read upper bound Σ_l Hkv·4·d·need(t, l) — it matters for variable
    lengths).  Rank r's range ends at the first tuple whose inclusive cost prefix reaches
    (r + 1)/world of the total, so every boundary is within one tuple's cost of the ideal split;
    the ranges are contiguous, disjoint and cover every tuple."""
    import numpy as np
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    c = np.asarray(costs, dtype=np.float64)
    if c.ndim != 1 or (c < 0).any():
        raise ValueError("costs must be a non-negative vector")
    n = len(c)
    pre = np.cumsum(c)
    total = pre[-1] if n else 0.0

    def cut(k):
        if k <= 0:
            return 0
        if k >= world or total == 0:
            return n if k >= world else (n * k) // world
        return int(np.searchsorted(pre, total * k / world, side="left")) + 1

    return min(cut(rank), n), min(cut(rank + 1), n)


def weak_shard(n_per_rank: int, rank: int) -> Tuple[int, int]:
    """Weak scaling: rank r owns tuple ids r·n .. r·n + n − 1 of an N·n-tuple dataset."""
    return rank * n_per_rank, (rank + 1) * n_per_rank


def combine_counts(counts, group=None):
    """In-place all-reduce(SUM) of an int64 count tensor across the process group."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return counts


def combine_soft(out, group=None):
    """In-place all-reduce(SUM) of a ko_soft_stats fp64 output vector across ranks: the relaxed
    TP/FP/FN/cost and every Jacobian entry are sums over tuples, so each rank
    evaluates its own tuple shard and one all-reduce per optimizer iteration combines them."""
    return combine_counts(out, group)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (device time) over the group — the timing rule of bench.py."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
