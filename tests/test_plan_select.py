"""Host derivations (row a12 / NEXT-2): cost, selectivities, Beta lower bounds and the cheapest
feasible plan — checked against independent computations (scipy's betaincinv via the oracle,
brute-force selection)."""
import numpy as np

import oracle
from paper_2602_04430_b200 import plan_select


def test_stats_and_selection_against_brute_force():
    rng = np.random.default_rng(3)
    n = 4000
    m = rng.normal(0, 2, size=(2, 3, n))
    gold = ((m[:, 2] + rng.normal(0, 0.3, size=(2, n))) > 0).astype(np.uint8)
    variants = [(200, 1), (500, 2), (1000, 2)]
    plans = []
    for h1 in (0.25, 1.0, 3.0):
        for h2 in (0.25, 1.0, 3.0):
            plans.append([(0, 0, -h1, h1, 0), (0, 2, 0.0, 0.0, 1), (1, 1, -h2, h2, 0),
                          (1, 2, 0.0, 0.0, 1)])
    counts = oracle.run_plans(plans, m, np.zeros(m.shape, np.int32), [1, 1], gold)
    _, stats0 = plan_select.select_plan(plans, counts, variants, target_recall=0.0)
    target = float(np.median([s.recall_lb for s in stats0]))
    best, stats = plan_select.select_plan(plans, counts, variants, target_recall=target)
    vc = plan_select.variant_costs(variants)
    assert vc == [0.1, 0.5, 1.0]
    feasible = []
    for g, pl in enumerate(plans):
        c = counts[g]
        cost = sum(c[5 + 4 * s] * vc[st[1]] for s, st in enumerate(pl))
        lb = oracle.beta_lower_bound(int(c[0]), int(c[2]), 0.95)
        assert abs(stats[g].cost - cost) < 1e-9 and abs(stats[g].recall_lb - lb) < 1e-10
        # conditional selectivities (Q11) from the raw counts
        for s in range(len(pl)):
            n_in, a, r, u = c[5 + 4 * s: 9 + 4 * s]
            if n_in:
                assert abs(stats[g].sel_inter[s] - (a + u) / n_in) < 1e-12
                assert abs(stats[g].sel_intra[s] - u / n_in) < 1e-12
        if lb >= target:
            feasible.append((cost, g))
    assert best is not None and (best.cost, best.index) == min(feasible)
    # wider cheap-stage bands send more tuples on: more cost, more recall
    assert stats[8].cost > stats[0].cost


def test_infeasible_returns_none():
    counts = np.zeros((1, 37), np.int64)
    counts[0, :5] = [1, 0, 99, 1, 100]
    counts[0, 5] = 100
    best, _ = plan_select.select_plan([[(0, 0, 0.0, 0.0, 1)]], counts, [(1000, 1)], 0.9)
    assert best is None


def test_selection_carries_loss_and_target_met():
    """Every plan's loss (eqn:loss) and Target Met on its hard counts equal the loss
    oracle's, with cost = Σ_s n_in[s]·cost_s and Σ_i cost_{o_i} over the plan's stages."""
    from oracle import loss
    rng = np.random.default_rng(9)
    n = 3000
    m = rng.normal(0, 2, size=(2, 3, n))
    gold = ((m[:, 2] + rng.normal(0, 0.3, size=(2, n))) > 0).astype(np.uint8)
    variants = [(200, 1), (500, 2), (1000, 2)]
    plans = [[(0, 0, -h, h, 0), (0, 2, 0.0, 0.0, 1), (1, 1, -h, h, 0), (1, 2, 0.0, 0.0, 1)]
             for h in (0.25, 1.0, 3.0)]
    counts = oracle.run_plans(plans, m, np.zeros(m.shape, np.int32), [1, 1], gold)
    best, stats = plan_select.select_plan(plans, counts, variants, target_recall=0.9,
                                          target_precision=0.8, n_tuples=n)
    vc = plan_select.variant_costs(variants)
    for st, pl, c in zip(stats, plans, counts):
        sc = [vc[s[1]] for s in pl]
        cost = sum(c[5 + 4 * k] * sc[k] for k in range(len(pl)))
        exp = loss.loss(c[0], c[1], c[2], cost, n, sc, 0.9, 0.8, 0.95, 10.0)
        for k, v in exp.items():
            assert abs(st.loss[k] - v) <= 1e-10 * max(1.0, abs(v)), k
        assert abs(st.loss["target_met_recall"] - st.recall / 0.9) < 1e-12
