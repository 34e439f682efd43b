"""Randomised end-to-end parity: random geometry, ragged lengths, random operators (filters and
maps, fp32 or bf16 readouts), random variants and random valid plans, in grid mode and routed
mode, against the oracle (margins ≤ 2e-3; counts exact under the ambiguity-band merge rule)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from kogen.device import tensors_to_device  # noqa: E402
from tests import parity  # noqa: E402
from tests.helpers import Geom, build_pool, random_problem  # noqa: E402


@pytest.fixture(scope="module")
def ko():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2602_04430_b200 as ko
    return ko


def random_plan(rng, n_ops, n_var, classes, m_or):
    """A valid plan: every op gets 1-3 stages in cost order, the last one final; ops interleaved
    at random.  Thresholds are placed around the oracle margins' quantiles."""
    per_op = []
    budget = 8                                      # KO_MAX_STAGES
    for o in range(n_ops):
        k = int(rng.integers(1, min(4, budget - (n_ops - 1 - o)) + 1)) if budget > 1 else 1
        k = min(k, 3)
        budget -= k
        vs = sorted(rng.choice(n_var, size=k, replace=True).tolist())
        stages = []
        for i, v in enumerate(vs):
            mv = m_or[o, v]
            fin = i == k - 1
            if classes[o] > 1:
                th = float(np.quantile(mv, rng.uniform(0.2, 0.8)))
                stages.append((o, v, th, th, int(fin)))
            elif fin:
                th = float(np.quantile(mv, rng.uniform(0.3, 0.7)))
                stages.append((o, v, th, th, 1))
            else:
                lo, hi = sorted(np.quantile(mv, rng.uniform(0.1, 0.9, size=2)).tolist())
                stages.append((o, v, lo, hi, 0))
        per_op.append(stages)
    plan = []
    while any(per_op):
        o = int(rng.choice([i for i, st in enumerate(per_op) if st]))
        plan.append(per_op[o].pop(0))
    return plan


@pytest.mark.parametrize("seed", range(40))
def test_random_problem_grid_and_routed(ko, seed):
    rng = np.random.default_rng(1000 + seed)
    D = int(rng.choice([64, 128]))
    G = int(rng.choice([1, 2, 4]))
    n_q = int(rng.choice([1, 2])) if G <= 2 else 1
    n_ops = int(rng.integers(1, 4))
    while n_ops * G * n_q > 16:
        n_ops -= 1
    geom = Geom(int(rng.integers(1, 4)), int(rng.integers(1, 3)), G, D, n_q)
    classes = tuple(int(rng.choice([1, 1, 3, 4])) for _ in range(n_ops))
    lengths = rng.integers(1, 200, size=int(rng.integers(3, 40))).tolist()
    K, V, ops_h = random_problem(rng, geom, lengths, n_ops=n_ops, classes=classes)
    pool, indptr, ids, sl = build_pool(K, V, lengths, poison=True, seed=seed)
    n_var = int(rng.integers(1, 5))
    variants = [(int(rng.integers(1, 1001)), int(rng.integers(1, geom.n_layers + 1)))
                for _ in range(n_var)]
    m_or, c_or = oracle.score(geom, pool, indptr, ids, sl, ops_h, variants)
    kv, ops = tensors_to_device(pool, indptr, ids, sl, geom, ops_h)
    if rng.random() < 0.5:
        for op in ops:
            op.w = op.w.to(torch.bfloat16)
    gold = np.stack([(rng.random(len(lengths)) < 0.5) if classes[o] <= 1
                     else rng.integers(0, classes[o], len(lengths))
                     for o in range(n_ops)]).astype(np.uint8)
    gold_d = torch.from_numpy(gold).cuda()
    plans = [random_plan(rng, n_ops, n_var, classes, m_or) for _ in range(3)]
    # grid mode: every margin, 3 plans
    m, c, counts = ko.score_batch(kv, ops, variants, plans=plans, gold=gold_d)
    torch.cuda.synchronize()
    mg, cg = m.cpu().numpy(), c.cpu().numpy()
    parity.assert_margins(mg, m_or)
    parity.assert_classes(cg, c_or, m_or, classes)
    parity.assert_counts(counts.cpu().numpy(), m_or, c_or, mg, cg, plans, list(classes), gold)
    # routed mode, each plan
    for plan in plans:
        m2, c2, cnt2 = ko.score_batch(kv, ops, variants, plans=[plan], gold=gold_d)
        torch.cuda.synchronize()
        m2n, c2n = m2.cpu().numpy(), c2.cpu().numpy()
        parity.assert_margins(m2n, m_or, mask=np.isfinite(m2n))
        parity.assert_counts(cnt2.cpu().numpy(), m_or, c_or, m2n, c2n, [plan], list(classes), gold)


@pytest.mark.parametrize("seed", range(16))
def test_random_routed_with_external_stages(ko, seed):
    """Routed plans mixing external stages (caller-supplied margins, e.g. an embedding filter) at
    random positions — including first, where position 0 is a walk-only launch — with KV stages:
    reached margins and counts equal the oracle's."""
    rng = np.random.default_rng(5000 + seed)
    geom = Geom(2, 2, 4, 64, 1)
    n_ops = int(rng.integers(1, 4))
    classes = tuple([1] * n_ops)
    lengths = rng.integers(1, 120, size=30).tolist()
    K, V, ops_h = random_problem(rng, geom, lengths, n_ops=n_ops, classes=classes)
    pool, indptr, ids, sl = build_pool(K, V, lengths, poison=True, seed=seed)
    variants = [(int(rng.integers(100, 600)), 1), (1000, 2), (0, 0)]   # last: external
    ev = len(variants) - 1
    m_or, c_or = oracle.score(geom, pool, indptr, ids, sl, ops_h, variants[:ev])
    n = len(lengths)
    ext = rng.normal(0, 1, size=(n_ops, n)).astype(np.float32)
    m_all = np.concatenate([m_or, ext[:, None, :].astype(np.float64)], axis=1)
    c_all = np.concatenate([c_or, np.zeros((n_ops, 1, n), np.int32)], axis=1)
    plan = []
    per_op = []
    for o in range(n_ops):
        st = []
        if rng.random() < 0.7:                                   # external stage first
            lo, hi = sorted(rng.normal(0, 0.7, size=2).tolist())
            st.append((o, ev, lo, hi, 0))
        if rng.random() < 0.6:
            q = np.quantile(m_or[o, 0], [0.3, 0.7])
            st.append((o, 0, float(q[0]), float(q[1]), 0))
        th = float(np.quantile(m_or[o, 1], 0.5))
        st.append((o, 1, th, th, 1))
        per_op.append(st)
    while any(per_op):
        o = int(rng.choice([i for i, st in enumerate(per_op) if st]))
        plan.append(per_op[o].pop(0))
    gold = np.stack([(m_or[o, 1] > 0) for o in range(n_ops)]).astype(np.uint8)
    kv, ops = tensors_to_device(pool, indptr, ids, sl, geom, ops_h)
    margins = torch.full((n_ops, len(variants), n), float("nan"), device="cuda")
    margins[:, ev, :] = torch.from_numpy(ext).cuda()
    m, c, counts = ko.score_batch(kv, ops, variants, margins=margins, plans=[plan],
                                  gold=torch.from_numpy(gold).cuda())
    torch.cuda.synchronize()
    mg, cg = m.cpu().numpy(), c.cpu().numpy()
    assert np.array_equal(mg[:, ev], ext)                        # external margins untouched
    kvm = np.isfinite(mg[:, :ev])
    parity.assert_margins(mg[:, :ev], m_or, mask=kvm)
    parity.assert_counts(counts.cpu().numpy(), m_all, c_all, mg, cg, [plan], list(classes), gold)
