"""Pins of the oracle's decisions, cascade routing and counts (SURVEY §8(c) steps 5–9):
brute force against an independent per-operator formulation of Eqs. (accept-i)/(reject-i)/
(unsure-i), the paper's worked examples, the
product-of-recalls identity, the τ → 0 limit of the soft decision and
count identities.  CPU only."""
import itertools
import math

import numpy as np
import pytest

import oracle

ACC, REJ, UNS = 0, 1, 2


def outcome_margin(o):
    return {ACC: 5.0, REJ: -5.0, UNS: 0.0}[o]


def per_op_recurrence(decisions):
    """Eqs. (accept-i)/(reject-i)/(unsure-i) with every stage selected: decisions is the list of
    per-stage indicator outcomes of ONE op's cascade; returns (accept, reject, unsure) after each
    stage as 0/1 ints, starting from unsure_0 = 1."""
    a, r, u = 0, 0, 1
    out = []
    for d in decisions:
        a = a + u * (1 if d == ACC else 0)
        r = r + u * (1 if d == REJ else 0)
        u = 1 - a - r
        out.append((a, r, u))
    return out


def brute_force_counts(plan_ops, finals, outcomes, gold):
    """Independent count computation.  plan_ops[s] = op of stage s, outcomes[t][s] = the stage-s
    decision of tuple t, gold[t][o] = gold bit.  Reach of stage s: unsure in op_s's cascade
    before s AND not rejected by any other op's stages that precede s (set algebra)."""
    S = len(plan_ops)
    ops = sorted(set(plan_ops))
    n_in = [0] * S; n_acc = [0] * S; n_rej = [0] * S; n_uns = [0] * S
    tp = n_out = n_gold = 0
    codes = np.zeros((S, len(outcomes)), np.int8)      # per-tuple stage outcome (0 = not reached)
    alive = np.zeros(len(outcomes), np.uint8)
    for t, dec in enumerate(outcomes):
        def state(o, upto):
            idx = [s for s in range(upto) if plan_ops[s] == o]
            rec = per_op_recurrence([dec[s] for s in idx])
            return rec[-1] if rec else (0, 0, 1)
        for s in range(S):
            o = plan_ops[s]
            reach = state(o, s)[2] == 1 and all(state(o2, s)[1] == 0 for o2 in ops if o2 != o)
            if reach:
                n_in[s] += 1
                d = dec[s]
                n_acc[s] += d == ACC; n_rej[s] += d == REJ; n_uns[s] += d == UNS
                codes[s, t] = {ACC: 1, REJ: 2, UNS: 3}[d]
        in_out = all(state(o, S)[0] == 1 for o in ops)      # conjunctive AND of each cascade
        alive[t] = in_out
        in_gold = all(gold[t][o] == 1 for o in ops)
        n_out += in_out; n_gold += in_gold; tp += in_out and in_gold
    row = [tp, n_out - tp, n_gold - tp, n_out, n_gold]
    for s in range(S):
        row += [n_in[s], n_acc[s], n_rej[s], n_uns[s]]
    return row, codes, alive


PLAN_SHAPES = [
    [0],                     # single final
    [0, 0],                  # cascade small -> final
    [0, 0, 0],
    [0, 1],                  # two single-stage filters
    [0, 0, 1, 1],            # two cascades
    [0, 1, 0, 1],            # interleaved (Algorithm 1 may interleave, Q23)
    [1, 0, 0, 1],
    [0, 1, 2],
    [0, 0, 1, 2],
    [2, 0, 1, 1],
]


@pytest.mark.parametrize("plan_ops", PLAN_SHAPES)
def test_routing_brute_force(plan_ops):
    S = len(plan_ops)
    ops = sorted(set(plan_ops))
    finals = [s == max(i for i in range(S) if plan_ops[i] == plan_ops[s]) for s in range(S)]
    choices = [[ACC, REJ] if finals[s] else [ACC, REJ, UNS] for s in range(S)]
    patterns = list(itertools.product(*choices))
    gold_patterns = list(itertools.product([0, 1], repeat=len(ops)))
    outcomes = [p for p in patterns for _ in gold_patterns]
    gold = [dict(zip(ops, g)) for _ in patterns for g in gold_patterns]
    n = len(outcomes)
    n_ops = max(ops) + 1
    # one variant per stage so each stage's margin is independent
    margins = np.zeros((n_ops, S, n))
    for t, dec in enumerate(outcomes):
        for s in range(S):
            margins[plan_ops[s], s, t] = outcome_margin(dec[s])
    classes = np.zeros(margins.shape, np.int32)
    g = np.zeros((n_ops, n), np.uint8)
    for t in range(n):
        for o in ops:
            g[o, t] = gold[t][o]
    plan = [(plan_ops[s], s, 0.0 if finals[s] else -1.0, 0.0 if finals[s] else 1.0, int(finals[s]))
            for s in range(S)]
    counts, alive, stages = oracle.run_plans([plan], margins, classes, [1] * n_ops, g,
                                             want_alive=True, want_stages=True)
    expect, codes, alive_bf = brute_force_counts(plan_ops, finals, outcomes, gold)
    assert list(counts[0, :len(expect)]) == expect
    assert not counts[0, len(expect):].any()
    # per-tuple decisions: each stage's outcome (reached or not) and P_o membership
    assert np.array_equal(stages[0, :S], codes)
    assert not stages[0, S:].any()
    assert np.array_equal(alive[0], alive_bf)


def test_count_identities_random():
    rng = np.random.default_rng(0)
    n = 2000
    m = rng.normal(0, 2, size=(2, 3, n))
    gold = (rng.random((2, n)) < 0.4).astype(np.uint8)
    plan = [(0, 0, -1.0, 1.0, 0), (0, 1, -0.5, 0.5, 0), (0, 2, 0.0, 0.0, 1),
            (1, 0, -2.0, 2.0, 0), (1, 2, 0.0, 0.0, 1)]
    c = oracle.run_plans([plan], m, np.zeros(m.shape, np.int32), [1, 1], gold)[0]
    tp, fp, fn, n_out, n_gold = c[:5]
    assert tp + fp == n_out and tp + fn == n_gold
    rej = 0
    for s in range(len(plan)):
        n_in, a, r, u = c[5 + 4 * s: 9 + 4 * s]
        assert n_in == a + r + u
        rej += r
    assert n_out == n - rej                                  # |P_o| = N − Σ n_rej
    # same-op adjacent stages: tuples entering stage s+1 are exactly stage s's unsure ones
    assert c[5 + 4 * 1] == c[8 + 4 * 0] and c[5 + 4 * 2] == c[8 + 4 * 1]
    # inter-operator order changes only n_in, never TP/FP/FN (Q12)
    plan2 = plan[3:] + plan[:3]
    c2 = oracle.run_plans([plan2], m, np.zeros(m.shape, np.int32), [1, 1], gold)[0]
    assert list(c2[:5]) == list(c[:5])


def test_gold_plan_is_exact():
    """Gold plan with gold = its own decisions ⇒ P = R = 1 (FP = FN = 0)."""
    rng = np.random.default_rng(1)
    m = rng.normal(0, 2, size=(2, 1, 500))
    gold = (m[:, 0] > 0).astype(np.uint8)
    plan = [(0, 0, 0.0, 0.0, 1), (1, 0, 0.0, 0.0, 1)]
    c = oracle.run_plans([plan], m, np.zeros(m.shape, np.int32), [1, 1], gold)[0]
    assert c[1] == 0 and c[2] == 0 and c[0] == np.sum(gold[0] & gold[1])


def test_fig3_hard_analogue():
    """P:413-419 at σ ∈ {0,1}: a selected first stage that rejects ⇒ rejected; with the first
    stage deselected (absent) and later stages accepting ⇒ accepted (counts as TP if labelled
    positive, else FP — the garbled '0.8 FP' of P:419 read as Q9)."""
    m = np.zeros((1, 3, 2)); m[0, 0] = -5.0; m[0, 1] = 5.0; m[0, 2] = 5.0
    gold = np.array([[1, 0]], np.uint8)
    sel = [(0, 0, -1.0, 1.0, 0), (0, 1, -1.0, 1.0, 0), (0, 2, 0.0, 0.0, 1)]
    c = oracle.run_plans([sel], m, np.zeros(m.shape, np.int32), [1], gold)[0]
    assert c[3] == 0 and c[0] == 0 and c[2] == 1            # rejected by o1: FN for positive
    desel = sel[1:]
    c = oracle.run_plans([desel], m, np.zeros(m.shape, np.int32), [1], gold)[0]
    assert c[3] == 2 and c[0] == 1 and c[1] == 1 and c[2] == 0


def test_always_accepting_first_stage_costs_only_itself():
    """an always-accepting stage 1 ⇒ later stages of the op see n_in = 0 (cost = c_1)."""
    m = np.zeros((1, 2, 50)); m[0, 0] = 3.0; m[0, 1] = -3.0
    plan = [(0, 0, -1.0, 1.0, 0), (0, 1, 0.0, 0.0, 1)]
    c = oracle.run_plans([plan], m, np.zeros(m.shape, np.int32), [1])[0]
    assert c[5] == 50 and c[6] == 50 and c[9] == 0
    cost = c[5] * 1.0 + c[9] * 10.0
    assert cost == 50 * 1.0


def test_threshold_boundaries_strict():
    """Q5/Q6: m = θ± ⇒ unsure; nextafter outward ⇒ accept / reject; final tie rejects."""
    lo, hi = np.float32(-0.75), np.float32(1.25)
    vals = [float(hi), np.nextafter(float(hi), np.inf), float(lo), np.nextafter(float(lo), -np.inf),
            0.0]
    m = np.array(vals)[None, None, :]
    c = oracle.run_plans([[(0, 0, float(lo), float(hi), 0), (0, 0, 0.0, 0.0, 1)]], m,
                         np.zeros(m.shape, np.int32), [1], want_alive=True)
    counts, alive = c
    assert counts[0, 5:9].tolist() == [5, 1, 1, 3]          # n_in, acc, rej, uns
    st = oracle.run_plans([[(0, 0, float(lo), float(hi), 0), (0, 0, 0.0, 0.0, 1)]], m,
                          np.zeros(m.shape, np.int32), [1], want_stages=True)[1]
    assert st[0, 0].tolist() == [3, 1, 3, 2, 3]              # unsure at θ±, strict outward
    assert st[0, 1].tolist() == [1, 0, 2, 0, 2]              # final θ_f = 0 (0: not reached; tie rejects)
    fin = oracle.run_plans([[(0, 0, 1.25, 1.25, 1)]], m, np.zeros(m.shape, np.int32), [1],
                           want_alive=True)[1]
    assert fin[0].tolist() == [0, 1, 0, 0, 0]                 # only m > θ_f accepted


def test_tau_to_zero_limit_of_soft_decision():
    """π = softmax_τ([m − θ⁺, θ⁻ − m, 0]); as τ → 0 its argmax is the hard decision."""
    rng = np.random.default_rng(2)
    m = rng.normal(0, 2, size=400)
    lo, hi = -0.5, 0.8
    m = m[(np.abs(m - lo) > 1e-3) & (np.abs(m - hi) > 1e-3)]
    logits = np.stack([m - hi, lo - m, np.zeros_like(m)], axis=1) / 1e-4
    soft = np.argmax(logits, axis=1)          # 0 accept, 1 reject, 2 unsure
    marg = m[None, None, :]
    counts = oracle.run_plans([[(0, 0, lo, hi, 0), (0, 0, 0.0, 0.0, 1)]], marg,
                              np.zeros(marg.shape, np.int32), [1])[0]
    assert counts[6] == np.sum(soft == 0) and counts[7] == np.sum(soft == 1)
    assert counts[8] == np.sum(soft == 2)


def product_grid(m1, g1, m2, g2):
    n1, n2 = len(m1), len(m2)
    m = np.zeros((2, 1, n1 * n2)); gold = np.zeros((2, n1 * n2), np.uint8)
    for i in range(n1):
        for j in range(n2):
            t = i * n2 + j
            m[0, 0, t], gold[0, t] = m1[i], g1[i]
            m[1, 0, t], gold[1, t] = m2[j], g2[j]
    return m, gold


def test_product_of_recalls_identity():
    """on a product-grid dataset TP = TP1·TP2 and |P_g| = G1·G2, so the global
    recall is the product of the per-op recalls; |P_o| = A1·A2 and with F1 first (single
    stage) F2's stage sees A1·n2 tuples."""
    rng = np.random.default_rng(3)
    n1, n2 = 23, 17
    m1, m2 = rng.normal(0, 1, n1), rng.normal(0, 1, n2)
    g1, g2 = (rng.random(n1) < 0.6).astype(np.uint8), (rng.random(n2) < 0.5).astype(np.uint8)
    m, gold = product_grid(m1, g1, m2, g2)
    plan = [(0, 0, 0.0, 0.0, 1), (1, 0, 0.0, 0.0, 1)]
    c = oracle.run_plans([plan], m, np.zeros(m.shape, np.int32), [1, 1], gold)[0]
    A1, A2 = int(np.sum(m1 > 0)), int(np.sum(m2 > 0))
    TP1, TP2 = int(np.sum((m1 > 0) & (g1 == 1))), int(np.sum((m2 > 0) & (g2 == 1)))
    G1, G2 = int(g1.sum()), int(g2.sum())
    assert c[0] == TP1 * TP2 and c[4] == G1 * G2 and c[3] == A1 * A2
    assert c[5 + 4] == A1 * n2
    assert math.isclose(c[0] / c[4], (TP1 / G1) * (TP2 / G2), rel_tol=1e-12)


@pytest.mark.parametrize("k1,k2,n,expect_tp,meets", [
    (19, 19, 20, 361, True),     # symmetric split √0.9 ≈ 0.95: 0.9025 ≥ 0.9
    (47, 47, 50, 2209, False),   # 0.94 each: 0.8836 < 0.9
    (20, 18, 20, 360, True),     # budget shift: easy filter 1.0, other 0.9 ⇒ 0.9
])
def test_symmetric_split_and_budget_shift(k1, k2, n, expect_tp, meets):
    m1 = np.array([1.0] * k1 + [-1.0] * (n - k1)); m2 = np.array([1.0] * k2 + [-1.0] * (n - k2))
    g = np.ones(n, np.uint8)
    m, gold = product_grid(m1, g, m2, g)
    c = oracle.run_plans([[(0, 0, 0.0, 0.0, 1), (1, 0, 0.0, 0.0, 1)]], m,
                         np.zeros(m.shape, np.int32), [1, 1], gold)[0]
    assert c[0] == expect_tp and c[4] == n * n
    assert (c[0] / c[4] >= 0.9) == meets
    assert abs(math.sqrt(0.9) - 0.948683) < 1e-6


def test_map_fever_coughing_example():
    """o1 extracts 'fever' (wrong), o2 'coughing' (gold) ⇒ choosing o2 gives
    TP 1, FP 0, FN 0; choosing o1 gives TP 0, FP 1, FN 1 (map output-tuple semantics)."""
    FEVER, COUGH = 0, 1
    m = np.array([[[2.0], [3.0]]])                  # [op][variant][tuple]
    cls = np.array([[[FEVER], [COUGH]]], np.int32)
    gold = np.array([[COUGH]], np.uint8)
    c_o2 = oracle.run_plans([[(0, 1, 0.0, 0.0, 1)]], m, cls, [2], gold)[0]
    c_o1 = oracle.run_plans([[(0, 0, 0.0, 0.0, 1)]], m, cls, [2], gold)[0]
    assert c_o2[:3].tolist() == [1, 0, 0]
    assert c_o1[:3].tolist() == [0, 1, 1]


def test_map_cascade_resolves_or_passes_on():
    """Q13: a non-final map stage resolves iff m > θ⁺ (else unsure); maps never reject."""
    m = np.array([[[0.5, 3.0, 1.0], [2.0, 2.0, 2.0]]])
    cls = np.array([[[2, 1, 0], [1, 1, 1]]], np.int32)
    gold = np.array([[1, 1, 1]], np.uint8)
    plan = [(0, 0, 1.0, 1.0, 0), (0, 1, 1.0, 1.0, 1)]
    c = oracle.run_plans([plan], m, cls, [3], gold)[0]
    assert c[5:9].tolist() == [3, 1, 0, 2] and c[9:13].tolist() == [2, 2, 0, 0]
    assert c[:5].tolist() == [3, 0, 0, 3, 3]


def test_invalid_plans_rejected():
    m = np.zeros((1, 1, 3))
    with pytest.raises(ValueError):
        oracle.run_plans([[(0, 0, 1.0, -1.0, 0)]], m, np.zeros(m.shape, np.int32), [1])
    with pytest.raises(ValueError):
        oracle.run_plans([[(0, 5, 0.0, 0.0, 1)]], m, np.zeros(m.shape, np.int32), [1])


def test_unlabelled_counts_contract():
    """gold = None (execution on unlabelled data, ko.h / SURVEY §8(b)): TP/FP/FN/|P_g| stay 0;
    |P_o| and the per-stage counts are those of the labelled evaluation."""
    rng = np.random.default_rng(3)
    m = rng.normal(0, 1, size=(2, 2, 500))
    c = np.zeros((2, 2, 500), np.int32)
    gold = (rng.random((2, 500)) < 0.5).astype(np.uint8)
    plan = [[(0, 0, -0.3, 0.3, 0), (0, 1, 0.0, 0.0, 1), (1, 1, 0.0, 0.0, 1)]]
    lab = oracle.run_plans(plan, m, c, [1, 1], gold)[0]
    unl = oracle.run_plans(plan, m, c, [1, 1], None)[0]
    assert unl[0] == unl[1] == unl[2] == unl[4] == 0
    assert unl[3] == lab[3] and np.array_equal(unl[5:], lab[5:])
    assert lab[1] == lab[3] - lab[0]
