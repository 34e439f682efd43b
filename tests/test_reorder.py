"""Algorithm 1 (DP operator reordering): SPEC's worked example and brute force."""
import itertools

import numpy as np
import pytest

from paper_2602_04430_b200 import reorder


def test_spec_two_filter_example():
    """two logical ops, one stage each, costs (1, 10), sel_inter (0.1, 0.5), N = 100:
    cheap-selective first costs 1·100 + 10·10 = 200 (SPEC prints 110: arithmetic slip), the other
    order 10·100 + 1·50 = 1050."""
    impl, cost = [0, 1], [1.0, 10.0]
    inter, intra = [0.1, 0.5], [0.0, 0.0]
    best, order = reorder.dp_reorder(impl, cost, inter, intra, 100)
    assert order == [0, 1]
    assert best == pytest.approx(1.0 * 100 + 10.0 * 100 * 0.1)       # 200
    worst = reorder.order_cost([1, 0], impl, cost, inter, intra, 100)
    assert worst == pytest.approx(10.0 * 100 + 1.0 * 100 * 0.5)       # 1050


@pytest.mark.parametrize("seed", range(6))
def test_dp_matches_brute_force(seed):
    rng = np.random.default_rng(seed)
    m = int(rng.integers(2, 8))
    impl = sorted(rng.integers(0, 3, size=m).tolist())
    cost = rng.uniform(0.5, 10, size=m).tolist()
    inter = rng.uniform(0.05, 1.0, size=m).tolist()
    intra = [x * rng.uniform(0, 1) for x in inter]
    for keep in (True, False):
        best, order = reorder.dp_reorder(impl, cost, inter, intra, 1000, keep_cascade_order=keep)
        assert sorted(order) == list(range(m))
        assert reorder.order_cost(order, impl, cost, inter, intra, 1000) == pytest.approx(best)
        brute = min(
            reorder.order_cost(p, impl, cost, inter, intra, 1000)
            for p in itertools.permutations(range(m))
            if not keep or all(p.index(a) < p.index(b) for a in range(m) for b in range(m)
                               if a < b and impl[a] == impl[b]))
        assert best == pytest.approx(brute)
