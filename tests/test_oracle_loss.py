"""Pins of the loss oracle (oracle/loss.py; NEXT-2, Eqs. 8–9, Target Met
P:765).  CPU only."""
import math

import numpy as np
import pytest

from oracle import loss, soft

ALPHA = 0.95


@pytest.mark.parametrize("a", [0.0, 0.5, 19.0, 250.3])
def test_bound_closed_form_b1(a):
    """FN = 0 ⇒ I_x(A, 1) = x^A ⇒ ℓ = (1−α)^{1/A}, dℓ/da = −ℓ·ln(1−α)/A² (A = 1 + a)."""
    A = 1.0 + a
    l = (1 - ALPHA) ** (1 / A)
    assert abs(loss.bound(a, 0.0, ALPHA) - l) < 1e-12
    da, _ = loss.bound_grad(a, 0.0, ALPHA)
    assert abs(da - (-l * math.log(1 - ALPHA) / A ** 2)) < 1e-7 * max(1.0, abs(da))


@pytest.mark.parametrize("b", [0.0, 0.7, 9.0, 120.0])
def test_bound_closed_form_a1(b):
    """TP = 0 ⇒ I_x(1, B) = 1 − (1−x)^B ⇒ ℓ = 1 − α^{1/B}, dℓ/db = α^{1/B}·ln α / B²."""
    B = 1.0 + b
    assert abs(loss.bound(0.0, b, ALPHA) - (1 - ALPHA ** (1 / B))) < 1e-12
    _, db = loss.bound_grad(0.0, b, ALPHA)
    assert abs(db - ALPHA ** (1 / B) * math.log(ALPHA) / B ** 2) < 1e-7 * max(1.0, abs(db))


def test_hand_computed_loss():
    """TP 19, FP 1, FN 0; cost 10 over |S| = 10 tuples and stage costs (1, 1); T_R = 0.9, no
    precision target, β = 10: ℓ_R = 0.05^{1/20} = 0.8608916593, L_cost = 10/(10·2) = 0.5,
    L_R = 0.9 − 0.8608916593 = 0.0391083407, L = 0.5 + 10·0.0391083407 = 0.891083407;
    Target Met recall = 1/0.9, precision = 19/20."""
    v = loss.loss(19, 1, 0, 10.0, 10, [1.0, 1.0], 0.9, 0.0, ALPHA, 10.0)
    assert abs(v["recall_lb"] - 0.8608916593) < 1e-10
    assert v["l_cost"] == 0.5 and v["l_precision"] == 0.0
    assert abs(v["l_recall"] - 0.0391083407) < 1e-10
    assert abs(v["loss"] - 0.891083407) < 1e-9
    assert abs(v["target_met_recall"] - 1 / 0.9) < 1e-15 and v["precision"] == 0.95


def _soft_problem(seed=0, n=3000):
    rng = np.random.default_rng(seed)
    m = rng.normal(0, 2, size=(2, 2, n))
    gold = (rng.random((2, n)) < 0.5).astype(np.uint8)
    plan = [(0, 0, -0.8, 0.6, 0), (0, 1, 0.0, 0.0, 1), (1, 0, -0.4, 0.9, 0), (1, 1, 0.1, 0.1, 1)]
    pick = [0.2, 0.0, -0.1, 0.0]
    cost = [0.25, 1.0, 0.3, 1.0]
    return plan, pick, m, gold, cost


def test_inactive_constraints_give_cost_gradient_only():
    plan, pick, m, gold, cost = _soft_problem()
    vals, grad, r = loss.soft_loss(plan, pick, 0.5, m, gold, cost, 0.05, 0.05, ALPHA, 10.0)
    assert vals["l_recall"] == 0.0 and vals["l_precision"] == 0.0
    assert np.array_equal(grad, r["jacobian"][3] / (m.shape[2] * sum(cost)))


def _loss_at(plan, pick, tau, m, gold, cost, tr, tpr, beta):
    r = soft.soft_stats(plan, pick, tau, m, gold, cost)
    return loss.loss(*r["values"], m.shape[2], cost, tr, tpr, ALPHA, beta)["loss"]


def test_gradient_against_finite_differences():
    """Active recall AND precision constraints: dL/d(s, θ⁻, θ⁺) by the chain rule equals central
    differences of L recomputed from scratch (forward relaxation + library quantile)."""
    plan, pick, m, gold, cost = _soft_problem(1)
    tau, tr, tpr, beta = 0.5, 0.99, 0.99, 10.0
    vals, grad, _ = loss.soft_loss(plan, pick, tau, m, gold, cost, tr, tpr, ALPHA, beta)
    assert vals["l_recall"] > 0 and vals["l_precision"] > 0
    fd = np.zeros_like(grad)
    for i, st in enumerate(plan):
        for k in range(3):
            if st[4] and k != 2:
                continue                           # finals: only θ (reported on θ⁺)
            def at(delta):
                p2 = [list(x) for x in plan]
                pk = list(pick)
                if k == 0:
                    pk[i] += delta
                    return _loss_at(plan, pk, tau, m, gold, cost, tr, tpr, beta), delta
                j = 1 + k                                      # θ⁻ at index 2, θ⁺ at 3
                new = float(np.float32(p2[i][j] + delta))          # thresholds are fp32
                eff = new - float(np.float32(p2[i][j]))
                p2[i][j] = new
                if st[4]:
                    p2[i][2] = p2[i][3] = new
                return _loss_at([tuple(x) for x in p2], pk, tau, m, gold, cost, tr, tpr, beta), eff
            (lp, hp), (lm, hm) = at(1e-3), at(-1e-3)
            fd[3 * i + k] = (lp - lm) / (hp - hm)
    assert np.allclose(grad, fd, rtol=2e-3, atol=1e-6), np.c_[grad, fd]
