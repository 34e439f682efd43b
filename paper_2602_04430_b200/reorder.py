"""Operator reordering by dynamic programming (Algorithm 1; NEXT-4 host part).

Host-side, m ≤ 20 physical operators; fed by the pass's selectivity counts (plan_select:
sel_inter = (n_acc + n_uns)/n_in, sel_intra = n_uns/n_in, Q11).  For every subset S of the
physical operators, DP[S] = (C_S, N_1..N_n): the minimum cost of executing exactly S and the
tuples still to be processed by each logical operator afterwards.  Transition S → S ∪ {o_k} with
O_j = impl(o_k): c = C_S + cost(o_k)·N_j^S; N_j ← N_j·sel_intra(o_k), N_ℓ ← N_ℓ·sel_inter(o_k)
for ℓ ≠ j; keep the minimum-cost transition; parent pointers give the order.

Cascade constraint: operators of the same logical operator keep their relative (cost) order, as
a cascade passes unsure tuples from cheaper to more expensive stages; Algorithm 1
as printed does not state it, the SPEC reading leaves interleaving free — both are
available (`keep_cascade_order`).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple


def dp_reorder(impl: Sequence[int], cost: Sequence[float], sel_inter: Sequence[float],
               sel_intra: Sequence[float], n_tuples: float, keep_cascade_order: bool = True
               ) -> Tuple[float, List[int]]:
    """Returns (minimum cost, execution order as indices into the physical operators)."""
    m = len(impl)
    if m == 0:
        return 0.0, []
    if m > 20:
        raise ValueError("dp_reorder: at most 20 physical operators")
    logical = sorted(set(impl))
    lidx = {o: i for i, o in enumerate(logical)}
    full = (1 << m) - 1
    INF = float("inf")
    best = [INF] * (1 << m)
    remain: List[Tuple[float, ...]] = [()] * (1 << m)
    parent = [-1] * (1 << m)
    best[0] = 0.0
    remain[0] = tuple(float(n_tuples) for _ in logical)
    # predecessors within a cascade (same logical operator, listed earlier)
    pred_mask = [0] * m
    if keep_cascade_order:
        for k in range(m):
            for k2 in range(k):
                if impl[k2] == impl[k]:
                    pred_mask[k] |= 1 << k2
    # process subsets in increasing cardinality
    order = sorted(range(1 << m), key=lambda s: bin(s).count("1"))
    for S in order:
        if best[S] == INF or S == full:
            continue
        C, N = best[S], remain[S]
        for k in range(m):
            if S >> k & 1 or (pred_mask[k] & S) != pred_mask[k]:
                continue
            j = lidx[impl[k]]
            c = C + cost[k] * N[j]
            S2 = S | (1 << k)
            if best[S2] == INF or c < best[S2]:
                best[S2] = c
                remain[S2] = tuple(N[l] * (sel_intra[k] if l == j else sel_inter[k])
                                   for l in range(len(logical)))
                parent[S2] = k
    seq = []
    S = full
    while S:
        k = parent[S]
        seq.append(k)
        S &= ~(1 << k)
    return best[full], seq[::-1]


def order_cost(order: Sequence[int], impl, cost, sel_inter, sel_intra, n_tuples) -> float:
    """Cost of executing the physical operators in a given order (the DP's cost model)."""
    logical = sorted(set(impl))
    N = {o: float(n_tuples) for o in logical}
    total = 0.0
    for k in order:
        total += cost[k] * N[impl[k]]
        for o in logical:
            N[o] *= sel_intra[k] if o == impl[k] else sel_inter[k]
    return total
