"""Oracle of the continuous relaxation (NEXT-1, SPEC soft_pipeline S:197-282).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain PyTorch CPU fp64, vectorised over
tuples, following the paper's equations in order; gradients by torch autograd (a library
routine), pinned against finite differences in tests/test_oracle_soft.py.

For a plan of filter stages i (plan order) with pick scores s_i, thresholds θ⁻_i ≤ θ⁺_i and
per-tuple cost c_i, temperature τ > 0, margins m_i(t) of stage i's (op, variant):
  σ_i = sigmoid(s_i / τ)                       pick factor; final stages σ = 1
  π_i = softmax([m − θ⁺, θ⁻ − m, 0] / τ)       soft accept / reject / unsure
        final stages: π_acc = sigmoid((m − θ)/τ), π_rej = 1 − π_acc, π_uns = 0 (the gold stage
        resolves every tuple)
  per op o, over its stages in plan order (Eqs. accept-i / reject-i / unsure-i, P:323-327 with
  𝟙^selected → σ_i, 𝟙^{accept/reject} → π_i):
        a_i = a_{i−1} + u_{i−1} σ_i π_acc,   r_i = r_{i−1} + u_{i−1} σ_i π_rej,   u_i = 1 − a_i − r_i
  plan accept mass  A(t) = Π_o a_o(t)          (soft AND)
  TP = Σ A g,  FP = Σ A (1 − g),  FN = Σ (1 − A) g,  g(t) = Π_o gold_o(t)     (Eqs. 5–7)
  cost = Σ_t Σ_i σ_i c_i u_{op_i}(t, before i) Π_{o' ≠ op_i} (1 − r_{o'}(t, before i))
        (Eq. cost P:338 with σ-scaling per the Fig. 3 narrative, P:417 / Q10; the product is the
        soft form of "reached": alive w.r.t. the other operators' earlier stages)
Map-classify operators ("choosing a particular map operator is equivalent to selecting
a subset of R_t"; reading Q13: maps never reject, a non-final map stage resolves iff its top-1/top-2
gap m > θ⁺): stage i of map op o resolves the mass u σ_i ρ_i with ρ_i = sigmoid((m − θ⁺)/τ)
(finals: σ = ρ = 1), carrying the value class_i(t); the op's correct mass
κ_o = Σ_i u σ_i ρ_i [class_i(t) = gold_o(t)].  Maps keep every tuple (r = 0).  Then
  A(t) = Π_o a_o (plan output mass),  T(t) = Π_filters a_o · Π_maps κ_o,  g(t) = Π_filters gold_o
  TP = Σ T g,  FP = Σ (A − T g),  FN = Σ (g − T g)
(for filter-only plans T = A and these are the three sums above; a wrong map value is one FP and one
FN, the fever/coughing example S:249-251).
As τ → 0 with s = ±∞ these are the hard counts of the extracted plan (tested).
"""
from __future__ import annotations

from typing import Dict, Sequence, Tuple

import numpy as np
import torch


def soft_forward(plan, s, lo, hi, tau, margins, gold, stage_cost, classes=None, n_classes=None):
    """Torch fp64 forward.  plan: [(op, var, θlo, θhi, final)]; s, lo, hi: tensors [S];
    margins: tensor [n_ops][n_var][n]; gold: tensor [n_ops][n] (filters 0/1, maps the class);
    classes: int tensor like margins (maps' argmax classes) or None; n_classes: per op (1 =
    filter).  Returns (tp, fp, fn, cost)."""
    n = margins.shape[2]
    ops = sorted({st[0] for st in plan})
    ncls = list(n_classes) if n_classes is not None else [1] * margins.shape[0]
    a = {o: torch.zeros(n, dtype=torch.float64) for o in ops}
    r = {o: torch.zeros(n, dtype=torch.float64) for o in ops}
    kappa = {o: torch.zeros(n, dtype=torch.float64) for o in ops if ncls[o] > 1}
    cost = torch.zeros((), dtype=torch.float64)
    for i, (o, v, _, _, fin) in enumerate(plan):
        m = margins[o, v]
        u_prev = 1.0 - a[o] - r[o]
        alive_other = torch.ones(n, dtype=torch.float64)
        for o2 in ops:
            if o2 != o:
                alive_other = alive_other * (1.0 - r[o2])
        if ncls[o] > 1:                                  # map stage: resolve or stay unsure
            if fin:
                sig = torch.ones((), dtype=torch.float64)
                p_acc = torch.ones(n, dtype=torch.float64)
            else:
                sig = torch.sigmoid(s[i] / tau)
                p_acc = torch.sigmoid((m - hi[i]) / tau)
            p_rej = torch.zeros(n, dtype=torch.float64)
            correct = (classes[o, v] == gold[o]).to(torch.float64)
            kappa[o] = kappa[o] + u_prev * sig * p_acc * correct
        elif fin:
            sig = torch.ones((), dtype=torch.float64)
            p_acc = torch.sigmoid((m - hi[i]) / tau)
            p_rej = 1.0 - p_acc
        else:
            sig = torch.sigmoid(s[i] / tau)
            logits = torch.stack([m - hi[i], lo[i] - m, torch.zeros_like(m)]) / tau
            pi = torch.softmax(logits, dim=0)
            p_acc, p_rej = pi[0], pi[1]
        cost = cost + (sig * stage_cost[i] * u_prev * alive_other).sum()
        a[o] = a[o] + u_prev * sig * p_acc
        r[o] = r[o] + u_prev * sig * p_rej
    A = torch.ones(n, dtype=torch.float64)
    T = torch.ones(n, dtype=torch.float64)
    g = torch.ones(n, dtype=torch.float64)
    for o in ops:
        A = A * a[o]
        if ncls[o] > 1:
            T = T * kappa[o]
        else:
            T = T * a[o]
            g = g * gold[o]
    tg = T * g
    tp = tg.sum()
    fp = (A - tg).sum()
    fn = (g - tg).sum()
    return tp, fp, fn, cost


def soft_stats(plan: Sequence[Tuple], pick: Sequence[float], tau: float, margins: np.ndarray,
               gold: np.ndarray, stage_cost: Sequence[float], classes: np.ndarray = None,
               n_classes: Sequence[int] = None) -> Dict[str, np.ndarray]:
    """Values [tp, fp, fn, cost] and Jacobian [4][3·S] w.r.t. (s_i, θ⁻_i, θ⁺_i) per stage
    (final stages: d/ds = 0, the threshold derivative is reported on θ⁺, d/dθ⁻ = 0; map stages:
    d/dθ⁻ = 0, final map stages have no parameters)."""
    S = len(plan)
    s = torch.tensor([float(x) for x in pick], dtype=torch.float64, requires_grad=True)
    # thresholds are fp32 in a plan (ko.h ko_stage): widened exactly, as in the hard oracle
    lo = torch.tensor([float(np.float32(st[2])) for st in plan], dtype=torch.float64,
                      requires_grad=True)
    hi = torch.tensor([float(np.float32(st[3])) for st in plan], dtype=torch.float64,
                      requires_grad=True)
    mt = torch.from_numpy(np.asarray(margins, np.float64))
    gt = torch.from_numpy(np.asarray(gold, np.float64))
    ct = [float(c) for c in stage_cost]
    cl = None if classes is None else torch.from_numpy(np.asarray(classes, np.int64))
    outs = soft_forward(plan, s, lo, hi, tau, mt, gt, ct, cl, n_classes)
    vals = np.array([float(x.detach()) for x in outs])
    jac = np.zeros((4, 3 * S))
    for k, out in enumerate(outs):
        gs, gl, gh = torch.autograd.grad(out, (s, lo, hi), retain_graph=True, allow_unused=True)
        for i in range(S):
            jac[k, 3 * i + 0] = 0.0 if gs is None else float(gs[i])
            jac[k, 3 * i + 1] = 0.0 if gl is None else float(gl[i])
            jac[k, 3 * i + 2] = 0.0 if gh is None else float(gh[i])
    return {"values": vals, "jacobian": jac}
