"""Oracle of the operator-selection objective (NEXT-2) — TEST INFRASTRUCTURE ONLY (see
oracle/__init__.py): plain fp64, each step as the paper writes it.

  ℓ_α^R = I⁻¹(1 − α; 1 + TP, 1 + FN),  ℓ_α^P = I⁻¹(1 − α; 1 + TP, 1 + FP)     (Eqs. 8–9; Q7)
      by the library routine scipy.special.betaincinv; real-valued (soft) counts allowed
  L_cost = Σ_t cost_Σ(t) / (|S| · Σ_i cost_{o_i})                              (eqn:cost-loss)
  L_R = ReLU(T_R − ℓ_α^R),  L_P = ReLU(T_P − ℓ_α^P)
  L = L_cost + β L_P + β L_R                                                  (eqn:loss)
  Target Met = achieved / target, for recall and for precision
  dL/dθ: chain rule — dℓ/d(count) by central differences of betaincinv (a library routine as the
  step), d(count)/dθ by torch autograd through oracle/soft.py's relaxation; the
  constraint terms are "only active (i.e., gradient ≠ 0) if the current pipeline violates the
  respective target".

Pinned in tests/test_oracle_loss.py: closed forms of the bound and of its derivatives (b = 1 and
a = 1 special cases of I_x), a hand-computed loss, the inactive-constraint case, and the gradient
against finite differences of the loss recomputed from scratch.
"""
from __future__ import annotations

from typing import Dict, Sequence, Tuple

import numpy as np


def bound(a: float, b: float, alpha: float) -> float:
    """ℓ = I⁻¹(1 − α; 1 + a, 1 + b) for real counts a, b ≥ 0."""
    from scipy.special import betaincinv
    return float(betaincinv(1.0 + a, 1.0 + b, 1.0 - alpha))


def bound_grad(a: float, b: float, alpha: float, rel: float = 1e-6) -> Tuple[float, float]:
    """(dℓ/da, dℓ/db) by central differences of the library quantile."""
    ha, hb = rel * max(1.0, 1.0 + a), rel * max(1.0, 1.0 + b)
    da = (bound(a + ha, b, alpha) - bound(a - ha, b, alpha)) / (2 * ha)
    db = (bound(a, b + hb, alpha) - bound(a, b - hb, alpha)) / (2 * hb)
    return da, db


def loss(tp: float, fp: float, fn: float, cost: float, n_tuples: float,
         stage_cost: Sequence[float], target_recall: float, target_precision: float,
         alpha: float, beta: float) -> Dict[str, float]:
    lr = bound(tp, fn, alpha)
    lpr = bound(tp, fp, alpha)
    l_cost = cost / (n_tuples * sum(stage_cost))
    l_r = max(0.0, target_recall - lr)
    l_p = max(0.0, target_precision - lpr)
    recall = tp / (tp + fn) if tp + fn > 0 else 1.0
    precision = tp / (tp + fp) if tp + fp > 0 else 1.0            # Q20
    return {"loss": l_cost + beta * l_p + beta * l_r, "l_cost": l_cost, "l_recall": l_r,
            "l_precision": l_p, "recall_lb": lr, "precision_lb": lpr, "recall": recall,
            "precision": precision,
            "target_met_recall": recall / target_recall if target_recall > 0 else float("nan"),
            "target_met_precision": (precision / target_precision if target_precision > 0
                                     else float("nan"))}


def loss_grad(values: Sequence[float], jacobian: np.ndarray, n_tuples: float,
              stage_cost: Sequence[float], target_recall: float, target_precision: float,
              alpha: float, beta: float) -> np.ndarray:
    """dL/dparams from the soft counts' values (TP, FP, FN, cost) and Jacobian [4][n_params]."""
    tp, fp, fn, cost = (float(x) for x in values[:4])
    J = np.asarray(jacobian, np.float64).reshape(4, -1)
    g = J[3] / (n_tuples * sum(stage_cost))
    lr, lpr = bound(tp, fn, alpha), bound(tp, fp, alpha)
    if target_recall > lr:
        da, db = bound_grad(tp, fn, alpha)
        g = g - beta * (da * J[0] + db * J[2])
    if target_precision > lpr:
        da, db = bound_grad(tp, fp, alpha)
        g = g - beta * (da * J[0] + db * J[1])
    return g


def soft_loss(plan, pick, tau, margins, gold, stage_cost, target_recall, target_precision,
              alpha, beta):
    """L and dL/d(s_i, θ⁻_i, θ⁺_i) of a relaxed plan on margins (oracle/soft.py + the above)."""
    from . import soft
    r = soft.soft_stats(plan, pick, tau, margins, gold, stage_cost)
    n = margins.shape[2]
    vals = loss(*r["values"], n, stage_cost, target_recall, target_precision, alpha, beta)
    grad = loss_grad(r["values"], r["jacobian"], n, stage_cost, target_recall, target_precision,
                     alpha, beta)
    return vals, grad, r
