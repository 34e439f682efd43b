"""Host derivations from the pass's integer counts.

From a plan's count row (TP, FP, FN, |P_o|, |P_g|, per-stage n_in/n_acc/n_rej/n_uns):
  * cost        = Σ_s n_in[s] · cost_s                       (Eq. cost; Q22)
  * sel_inter_s = (n_acc + n_uns) / n_in,  sel_intra_s = n_uns / n_in   (Q11,
                  conditional form used by Algorithm 1)
  * ℓ_α^R = I⁻¹(1 − α; 1 + TP, 1 + FN),  ℓ_α^P = I⁻¹(1 − α; 1 + TP, 1 + FP)   (Q7)
and the grid selection: the cheapest plan whose recall and precision lower bounds meet the
targets (the discrete analogue of the constrained objective), with the loss of
eqn:cost-loss … eqn:loss and Target Met of every plan from the library's host
helper ko_plan_loss.  The Beta quantile is the library's host helper ko_beta_lower_bound.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import C_FN, C_FP, C_GOLD, C_OUT, C_TP, beta_lower_bound, plan_loss


def variant_costs(variants: Sequence[Tuple[int, int]]) -> List[float]:
    """Q22 default: cost of a variant ∝ the KV bytes it reads (keep‰ × layers), gold = 1."""
    b = [k * c for k, c in variants]
    top = max(b)
    return [x / top for x in b]


@dataclass
class PlanStats:
    index: int
    tp: int
    fp: int
    fn: int
    n_out: int
    n_gold: int
    cost: float
    recall: float
    precision: float
    recall_lb: float
    precision_lb: float
    sel_inter: List[float]
    sel_intra: List[float]
    loss: Optional[dict] = None     # ko_plan_loss fields (L, L_cost, L_R, L_P, …, Target Met)


def plan_stats(g: int, plan: Sequence[Tuple], row: np.ndarray, variant_cost: Sequence[float],
               alpha: float = 0.95) -> PlanStats:
    tp, fp, fn, n_out, n_gold = (int(row[k]) for k in (C_TP, C_FP, C_FN, C_OUT, C_GOLD))
    cost, inter, intra = 0.0, [], []
    for s, st in enumerate(plan):
        n_in, n_acc, n_rej, n_uns = (int(x) for x in row[5 + 4 * s: 9 + 4 * s])
        cost += n_in * variant_cost[st[1]]
        inter.append((n_acc + n_uns) / n_in if n_in else 1.0)
        intra.append(n_uns / n_in if n_in else 0.0)
    return PlanStats(g, tp, fp, fn, n_out, n_gold, cost,
                     tp / n_gold if n_gold else 1.0, tp / n_out if n_out else 1.0,  # Q20
                     beta_lower_bound(tp, fn, alpha), beta_lower_bound(tp, fp, alpha), inter, intra)


def hard_loss(plan: Sequence[Tuple], row: np.ndarray, variant_cost: Sequence[float],
              n_tuples: int, target_recall: float, target_precision: float, alpha: float = 0.95,
              beta: float = 10.0) -> dict:
    """ko_plan_loss on a plan's integer counts (the τ = 0 extraction of the relaxation)."""
    sc = [variant_cost[st[1]] for st in plan]
    cost = sum(int(row[5 + 4 * s]) * sc[s] for s in range(len(plan)))
    v, _ = plan_loss([int(row[C_TP]), int(row[C_FP]), int(row[C_FN]), cost], sc, n_tuples,
                     target_recall, target_precision, alpha, beta)
    return v


def select_plan(plans: Sequence[Sequence[Tuple]], counts: np.ndarray,
                variants: Sequence[Tuple[int, int]], target_recall: float = 0.9,
                target_precision: float = 0.0, alpha: float = 0.95, n_tuples: int = 0,
                beta: float = 10.0) -> Tuple[Optional[PlanStats], List[PlanStats]]:
    """Cheapest plan with ℓ_α^R ≥ T_R and ℓ_α^P ≥ T_P (ties: lower index); None if infeasible
    (SPEC's infeasible_sample: the caller falls back to the gold plan).  With n_tuples > 0 each
    plan also carries its loss and Target Met (ko_plan_loss)."""
    vc = variant_costs(variants)
    stats = [plan_stats(g, plans[g], counts[g], vc, alpha) for g in range(len(plans))]
    if n_tuples > 0:
        for st in stats:
            st.loss = hard_loss(plans[st.index], counts[st.index], vc, n_tuples, target_recall,
                                target_precision, alpha, beta)
    ok = [s for s in stats if s.recall_lb >= target_recall and s.precision_lb >= target_precision]
    best = min(ok, key=lambda s: (s.cost, s.index)) if ok else None
    return best, stats
