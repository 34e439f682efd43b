"""N > 1 path on CPU (gloo, world size 2): tuple sharding + the count all-reduce give exactly the
1-rank counts, and the timing combine is a max over ranks.  The per-rank counts come from the
oracle's plan evaluation on that rank's shard (the GPU path's counts obey the same contract,
checked on the GPU by test_sharded_counts_add_up)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2602_04430_b200 import dist as kodist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(n=1001):
    rng = np.random.default_rng(42)
    m = rng.normal(0, 2, size=(2, 3, n))
    gold = (rng.random((2, n)) < 0.45).astype(np.uint8)
    plans = [[(0, 0, -1.0, 1.0, 0), (0, 2, 0.0, 0.0, 1), (1, 1, -0.5, 0.5, 0), (1, 2, 0.0, 0.0, 1)],
             [(1, 2, 0.0, 0.0, 1), (0, 0, 0.0, 0.0, 1)]]
    return m, gold, plans


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m, gold, plans = _problem()
    b, e = kodist.shard_range(m.shape[2], rank, world)
    c = oracle.run_plans(plans, m[:, :, b:e], np.zeros((2, 3, e - b), np.int32), [1, 1],
                         gold[:, b:e])
    t = torch.from_numpy(c)
    kodist.combine_counts(t)
    tmax = kodist.max_over_ranks(float(rank + 1))
    if rank == 0:
        out.put((t.numpy().tolist(), tmax))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_counts_equal_single_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    counts, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m, gold, plans = _problem()
    full = oracle.run_plans(plans, m, np.zeros(m.shape, np.int32), [1, 1], gold)
    assert np.array_equal(np.array(counts), full)
    assert tmax == 2.0


@pytest.mark.parametrize("n,world", [(10, 3), (7, 7), (0, 2), (1000, 8)])
def test_shard_range_partitions(n, world):
    seen = []
    for r in range(world):
        b, e = kodist.shard_range(n, r, world)
        seen += list(range(b, e))
        assert e - b in (n // world, n // world + 1)
    assert seen == list(range(n))


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_by_cost_contiguous_cover_and_balanced(world):
    """Byte-balanced sharding: contiguous, disjoint, covering ranges whose costs
    differ from the ideal share by at most one tuple's cost (log-uniform C3-like lengths)."""
    rng = np.random.default_rng(world)
    L = np.exp(rng.uniform(np.log(256), np.log(4096), size=5000)).astype(np.int64)
    cost = L * 2 * 8 * 4 * 128.0                     # bytes: layers · heads · (K+V, bf16) · d
    ranges = [kodist.shard_by_cost(cost, r, world) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == len(cost)
    for (a, b), (c, d) in zip(ranges, ranges[1:]):
        assert b == c and a <= b
    share = cost.sum() / world
    for a, b in ranges:
        assert abs(cost[a:b].sum() - share) <= 2 * cost.max()
    # equal costs reduce to an equal split
    eq = [kodist.shard_by_cost(np.ones(12), r, 4) for r in range(4)]
    assert eq == [(0, 3), (3, 6), (6, 9), (9, 12)]


def _soft_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import soft
    rng = np.random.default_rng(5)
    n = 701
    m = torch.from_numpy(rng.normal(0, 2, size=(2, 2, n)))
    gold = torch.from_numpy((rng.random((2, n)) < 0.4).astype(np.float64))
    plan = [(0, 0, -0.5, 0.5, 0), (0, 1, 0.0, 0.0, 1), (1, 0, -1.0, 1.0, 0), (1, 1, 0.0, 0.0, 1)]
    s = torch.tensor([0.3, 0.0, -0.2, 0.0], dtype=torch.float64)
    lo = torch.tensor([st[2] for st in plan], dtype=torch.float64)
    hi = torch.tensor([st[3] for st in plan], dtype=torch.float64)
    cost = torch.tensor([1.0, 4.0, 1.0, 4.0], dtype=torch.float64)
    b, e = kodist.shard_range(n, rank, world)
    part = torch.stack(list(soft.soft_forward(plan, s, lo, hi, 0.5, m[:, :, b:e], gold[:, b:e], cost)))
    kodist.combine_soft(part)
    full = torch.stack(list(soft.soft_forward(plan, s, lo, hi, 0.5, m, gold, cost)))
    if rank == 0:
        out.put((part.numpy().tolist(), full.numpy().tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_soft_relaxation_sums_equal_single_rank():
    """NEXT-1 sharded: per-rank relaxed TP/FP/FN/cost all-reduced over gloo = the 1-rank values."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_soft_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    part, full = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    assert np.allclose(part, full, rtol=1e-12, atol=1e-9)
