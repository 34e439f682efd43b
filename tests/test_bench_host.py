"""Host logic of bench.py (no GPU): weak-scaling rank ranges cover the world·n dataset with
contiguous, disjoint ranges, byte-balanced for variable lengths."""
import importlib.util
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


@pytest.mark.parametrize("cfg,world", [("C2", 1), ("C2", 8), ("C3", 2), ("C3", 8), ("C5", 4)])
def test_rank_ranges_cover_dataset(cfg, world):
    b = _bench()
    from kogen import workloads
    wl = workloads.get(cfg)
    n_per = 2000
    rr = [b.rank_range(wl, n_per, r, world) for r in range(world)]
    assert rr[0][0] == 0
    assert sum(n for _, n in rr) == world * n_per
    for (a, n), (c, _) in zip(rr, rr[1:]):
        assert a + n == c
    if wl.spec.len_min != wl.spec.len_max and world > 1:
        sl = wl.spec.seq_len(0, world * n_per).astype(np.int64)
        shares = [sl[a:a + n].sum() for a, n in rr]
        assert max(shares) - min(shares) <= 2 * sl.max()    # balanced by bytes, not by count


def test_algorithmic_bytes_c2_matches_closed_form():
    """C2 grid: every tuple needs its full 512-token cache in all 4 layers, 8 kv-heads, d 128."""
    b = _bench()
    from kogen import workloads
    wl = workloads.get("C2")
    sl = np.full(10, 512, np.int64)
    total, kv = b.algorithmic_bytes(wl, sl, len(wl.plans))
    assert kv == 10 * 4 * 512 * 8 * 4 * 128
    assert total == kv + 4 * 10 * 32 + 12 * 10 + 2 * 10 + 8 * 2 * 3 * 10
