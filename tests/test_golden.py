"""The paper's (and SPEC's) printed worked examples, read from tests/golden/paper_examples.json,
reproduced by the oracle and by the product's host helpers."""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import soft

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


def _product_grid(kept, n):
    m1 = np.array([1.0] * kept[0] + [-1.0] * (n - kept[0]))
    m2 = np.array([1.0] * kept[1] + [-1.0] * (n - kept[1]))
    m = np.zeros((2, 1, n * n))
    m[0, 0] = np.repeat(m1, n)
    m[1, 0] = np.tile(m2, n)
    gold = np.ones((2, n * n), np.uint8)
    plan = [(0, 0, 0.0, 0.0, 1), (1, 0, 0.0, 0.0, 1)]
    return oracle.run_plans([plan], m, np.zeros(m.shape, np.int32), [1, 1], gold)[0]


def test_symmetric_split_and_budget_shift():
    g = GOLDEN["symmetric_split"]
    assert abs(np.sqrt(g["target"]) - g["per_op_symmetric"]) < 1e-6
    for case in g["cases"]:
        c = _product_grid(case["per_op_kept"], case["per_op_n"])
        assert c[0] == case["global_tp"] and c[4] == case["global_gold"]
        assert (c[0] / c[4] >= g["target"]) == case["meets"]
    b = GOLDEN["budget_shift"]
    c = _product_grid(b["per_op_kept"], b["per_op_n"])
    assert c[0] == b["global_tp"] and c[4] == b["global_gold"] and c[0] / c[4] == b["recall"]


def test_fever_coughing():
    g = GOLDEN["fever_coughing"]
    m = np.array([[[2.0], [3.0]]])
    cls = np.array([[[0], [1]]], np.int32)            # variant 0 = o1 ('fever'), 1 = o2
    gold = np.array([[1]], np.uint8)                  # gold value: 'coughing'
    for key, var in (("choose_o2", 1), ("choose_o1", 0)):
        c = oracle.run_plans([[(0, var, 0.0, 0.0, 1)]], m, cls, [2], gold)[0]
        assert c[:3].tolist() == [g[key]["tp"], g[key]["fp"], g[key]["fn"]]


def test_fig3_walkthrough():
    g = GOLDEN["fig3_walkthrough"]
    tau = 1e-3
    s1 = tau * np.log(g["sigma1"] / (1 - g["sigma1"]))
    plan = [(0, 0, -1.0, 1.0, 0), (0, 1, -1.0, 1.0, 0), (0, 2, 0.0, 0.0, 1)]
    m = np.array([[[-5.0], [5.0], [5.0]]])
    for label, key in ((1, "positive"), (0, "negative")):
        v = soft.soft_stats(plan, [s1, 50.0, 0.0], tau, m, np.array([[label]]), [1, 2, 10])["values"]
        assert np.allclose(v[:3], [g[key]["tp"], g[key]["fp"], g[key]["fn"]], atol=1e-9)


def test_selectivity_30_40_30():
    from paper_2602_04430_b200 import plan_select
    g = GOLDEN["selectivity_30_40_30"]
    n = g["accept"] + g["unsure"] + g["reject"]
    m = np.array([5.0] * g["accept"] + [0.0] * g["unsure"] + [-5.0] * g["reject"])[None, None, :]
    plan = [(0, 0, -1.0, 1.0, 0), (0, 0, 0.0, 0.0, 1)]
    c = oracle.run_plans([plan], m, np.zeros(m.shape, np.int32), [1])
    st = plan_select.plan_stats(0, plan, c[0], [1.0])
    assert st.sel_inter[0] == pytest.approx(g["sel_inter"]) and st.sel_intra[0] == pytest.approx(g["sel_intra"])
    assert c[0][5] == n


def test_dp_two_filters():
    from paper_2602_04430_b200 import reorder
    g = GOLDEN["dp_two_filters"]
    best, order = reorder.dp_reorder([0, 1], g["cost"], g["sel_inter"], [0.0, 0.0], g["n"])
    assert order == g["order"] and best == pytest.approx(g["best"])
    assert reorder.order_cost(order[::-1], [0, 1], g["cost"], g["sel_inter"], [0.0, 0.0],
                              g["n"]) == pytest.approx(g["worst"])


def test_beta_flat_prior():
    g = GOLDEN["beta_flat_prior"]
    assert abs(oracle.beta_lower_bound(g["tp"], g["fn"], g["alpha"]) - g["bound"]) < 1e-12
    import paper_2602_04430_b200 as ko
    assert abs(ko.beta_lower_bound(g["tp"], g["fn"], g["alpha"]) - g["bound"]) < 1e-12
