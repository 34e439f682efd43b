"""ko_plan_loss / ko_beta_lower_bound_real (host C of libko.so; NEXT-2: eqn:cost-loss … eqn:loss
P:439-442, Eqs. 8–9, Target Met P:765) against the loss oracle (oracle/loss.py) and
closed forms.  CPU only (host entry points; the Jacobian comes from the relaxation oracle here,
from ko_soft_stats on the GPU in test_soft_gpu.py)."""
import math

import numpy as np
import pytest

import paper_2602_04430_b200 as ko
from oracle import loss, soft

ALPHA = 0.95


@pytest.mark.parametrize("a,b", [(0.0, 0.0), (19.0, 0.0), (0.0, 9.0), (19.0, 1.0), (90.0, 10.5),
                                 (3.25, 0.75), (4500.0, 310.0), (30000.0, 2.0)])
def test_bound_and_partials_vs_oracle(a, b):
    v, da, db = ko.beta_lower_bound_real(a, b, ALPHA)
    assert abs(v - loss.bound(a, b, ALPHA)) < 1e-10
    oa, ob = loss.bound_grad(a, b, ALPHA)
    assert abs(da - oa) <= 1e-6 * max(abs(oa), 1e-3) and abs(db - ob) <= 1e-6 * max(abs(ob), 1e-3)
    assert da > 0 > db                                   # more TP raises ℓ, more FN lowers it


def test_bound_closed_form_partials():
    A = 20.0
    l = 0.05 ** (1 / A)
    v, da, db = ko.beta_lower_bound_real(A - 1, 0.0, ALPHA)
    assert abs(v - l) < 1e-12 and abs(da - (-l * math.log(0.05) / A ** 2)) < 1e-8
    B = 10.0
    v, da, db = ko.beta_lower_bound_real(0.0, B - 1, ALPHA)
    assert abs(v - (1 - ALPHA ** (1 / B))) < 1e-12
    assert abs(db - ALPHA ** (1 / B) * math.log(ALPHA) / B ** 2) < 1e-8
    assert math.isnan(ko.beta_lower_bound_real(-1.0, 0.0, ALPHA)[0])


def test_hand_computed_and_target_met():
    v, g = ko.plan_loss([19, 1, 0, 10.0], [1.0, 1.0], 10, target_recall=0.9, beta=10.0)
    assert abs(v["recall_lb"] - 0.8608916593) < 1e-10
    assert abs(v["loss"] - 0.891083407) < 1e-9 and v["l_cost"] == 0.5 and g is None
    assert abs(v["target_met_recall"] - 1 / 0.9) < 1e-15 and math.isnan(v["target_met_precision"])
    e, _ = ko.plan_loss([0, 0, 5, 0.0], [1.0], 5, target_recall=0.5, target_precision=0.5)
    assert e["precision"] == 1.0 and e["recall"] == 0.0   # empty output: precision 1 (Q20)


@pytest.mark.parametrize("tr,tpr", [(0.05, 0.05), (0.99, 0.0), (0.0, 0.99), (0.99, 0.99)])
def test_soft_loss_and_gradient_vs_oracle(tr, tpr):
    rng = np.random.default_rng(5)
    n = 4000
    m = rng.normal(0, 2, size=(2, 2, n))
    gold = (rng.random((2, n)) < 0.5).astype(np.uint8)
    plan = [(0, 0, -0.8, 0.6, 0), (0, 1, 0.0, 0.0, 1), (1, 0, -0.4, 0.9, 0), (1, 1, 0.1, 0.1, 1)]
    pick, cost = [0.2, 0.0, -0.1, 0.0], [0.25, 1.0, 0.3, 1.0]
    vals_or, grad_or, r = loss.soft_loss(plan, pick, 0.3, m, gold, cost, tr, tpr, ALPHA, 10.0)
    v, g = ko.plan_loss(r["values"], cost, n, tr, tpr, ALPHA, 10.0, jacobian=r["jacobian"])
    for k in ko.LOSS_FIELDS:
        if math.isnan(vals_or[k]):
            assert math.isnan(v[k])
        else:
            assert abs(v[k] - vals_or[k]) <= 1e-10 * max(1.0, abs(vals_or[k])), k
    scale = np.abs(grad_or).max()
    assert np.allclose(g, grad_or, rtol=1e-6, atol=1e-9 * scale)


def test_constraint_exactly_at_target_is_inactive():
    """the constraint's gradient is nonzero only if the target is VIOLATED (T > ℓ)."""
    stats = [50.0, 5.0, 7.0, 30.0]
    J = np.arange(16, dtype=np.float64).reshape(4, 4) + 1.0
    lr = ko.beta_lower_bound_real(50.0, 7.0, ALPHA)[0]
    v, g = ko.plan_loss(stats, [1.0, 2.0], 100, target_recall=lr, beta=10.0, jacobian=J)
    assert v["l_recall"] == 0.0
    assert np.array_equal(np.array(g), J[3] / 300.0)


def test_errors():
    with pytest.raises(ko.KoError, match="alpha"):
        ko.plan_loss([1, 1, 1, 1.0], [1.0], 3, alpha=1.0)
    with pytest.raises(ko.KoError, match="negative"):
        ko.plan_loss([-1, 1, 1, 1.0], [1.0], 3)
    with pytest.raises(ko.KoError, match="n_tuples"):
        ko.plan_loss([1, 1, 1, 1.0], [1.0], 0)
