"""GPU decision parity at the threshold boundaries (Q5/Q6/Q13; P:456, P:471-472 strict '>' and
'<'), per tuple, against the oracle — the GPU mirror of tests/test_oracle_routing.py's boundary
table.  Margins are hand-built fp32 values AT θ⁺, θ⁻, θ_f and one ulp either side
(nextafter toward ±∞), map confidence gaps at θ⁺ and argmax ties (gap 0).  Both sides decide the
same fp32 numbers (the oracle widens them exactly), so every decision, state, worklist and count
must agree bit for bit — there is no ambiguity band here.

Routes: ko_reduce_stats (grid), ko_route stage −1 and stage by stage, the grid kernel's in-kernel
plan evaluation and a routed ko_score_batch, the last two through an EXTERNAL variant whose
caller-supplied margins sit on the boundaries (Eqs. accept-i / reject-i / unsure-i)."""
import itertools

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from kogen import workloads  # noqa: E402
from kogen.device import device_workload  # noqa: E402
from tests import parity  # noqa: E402

F32 = np.float32
LO, HI, FIN, CM = F32(-0.7), F32(1.3), F32(0.1), F32(0.45)


def around(x):
    """x and its fp32 neighbours: nextafter(x, -inf), x, nextafter(x, +inf)."""
    x = F32(x)
    return [np.nextafter(x, F32(-np.inf)), x, np.nextafter(x, F32(np.inf))]


FILTER_VALS = around(HI) + around(LO)                 # non-final filter stage
FINAL_VALS = around(FIN)                              # final filter stage: tie rejects
MAP_VALS = around(CM) + [F32(0.0)]                    # non-final map stage; gap 0 = argmax tie


@pytest.fixture(scope="module")
def ko():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2602_04430_b200 as ko
    return ko


def _problem():
    """3 ops (filter, 4-class map, filter) × 2 variants; every combination of boundary values
    over the six stages of PLAN (6·3·4·3·6·3 = 7776 tuples)."""
    combos = list(itertools.product(FILTER_VALS, FINAL_VALS, MAP_VALS, [F32(0.0), F32(2.0)],
                                    FILTER_VALS, FINAL_VALS))
    n = len(combos)
    m = np.zeros((3, 2, n), np.float32)
    for t, (a, b, c, dm, e, f) in enumerate(combos):
        m[0, 0, t], m[0, 1, t], m[1, 0, t], m[1, 1, t], m[2, 0, t], m[2, 1, t] = a, b, c, dm, e, f
    rng = np.random.default_rng(11)
    cls = rng.integers(0, 4, size=(3, 2, n)).astype(np.int32)
    cls[[0, 2]] = 0
    cls[1, :, m[1, 0] == 0] = 0                        # argmax tie → lowest class index (Q13)
    gold = np.stack([rng.random(n) < 0.6, rng.integers(0, 4, n), rng.random(n) < 0.6]).astype(np.uint8)
    return m, cls, gold


PLAN = [(0, 0, float(LO), float(HI), 0), (0, 1, float(FIN), float(FIN), 1),
        (1, 0, float(CM), float(CM), 0), (1, 1, 0.0, 0.0, 1),
        (2, 0, float(LO), float(HI), 0), (2, 1, float(FIN), float(FIN), 1)]
PLAN_INTERLEAVED = [PLAN[4], PLAN[0], PLAN[2], PLAN[1], PLAN[3], PLAN[5]]
N_CLASSES = [1, 4, 1]


def expected_state(stages, plan, cls, n):
    """tuple_state the ko.h layout implies for the oracle's per-tuple stage outcomes: bit 0
    alive, bits 1+2o status of op o (1 accepted/resolved, 2 rejected), bits 16+4o the resolved
    class of map op o."""
    st = np.ones(n, np.uint32)
    for s, (o, v, lo, hi, fin) in enumerate(plan):
        code = stages[s]
        acc = (code == oracle.STAGE_ACCEPT) | (code == oracle.STAGE_RESOLVED)
        rej = code == oracle.STAGE_REJECT
        st[acc] |= np.uint32(1 << (1 + 2 * o))
        st[rej] |= np.uint32(2 << (1 + 2 * o))
        st[rej] &= ~np.uint32(1)
        res = code == oracle.STAGE_RESOLVED
        st[res] |= (cls[o, v, res].astype(np.uint32) & 15) << np.uint32(16 + 4 * o)
    return st


DEFINED_BITS = np.uint32(0xFFFF01FF)                  # bits 9..15 are reserved (ko.h)


@pytest.mark.parametrize("plan", [PLAN, PLAN_INTERLEAVED], ids=["ordered", "interleaved"])
def test_route_boundaries_per_tuple(ko, plan):
    m, cls, gold = _problem()
    n = m.shape[2]
    counts_or, alive_or, stages_or = oracle.run_plans([plan], m.astype(np.float64), cls, N_CLASSES,
                                                      gold, want_alive=True, want_stages=True)
    # the boundary values really exercise every outcome (a test of the test)
    for s, (o, v, lo, hi, fin) in enumerate(plan):
        seen = set(np.unique(stages_or[0, s]).tolist()) - {oracle.STAGE_NOT_REACHED}
        assert len(seen) >= (1 if (fin and N_CLASSES[o] > 1) else 2), (s, seen)
    mt, ct, gt = (torch.from_numpy(x).cuda() for x in (m, cls, gold))
    # ko_reduce_stats
    red = ko.reduce_stats([plan, plan], mt, ct, N_CLASSES, gold=gt)
    assert np.array_equal(red.cpu().numpy()[0], counts_or[0])
    assert np.array_equal(red.cpu().numpy()[1], counts_or[0])
    # ko_route, whole plan: state, worklist (= P_o) and counts, per tuple
    st = torch.ones(n, dtype=torch.int32, device="cuda")
    wl = torch.empty(n, dtype=torch.int32, device="cuda")
    wlen = torch.zeros(1, dtype=torch.int64, device="cuda")
    c = ko.route(plan, mt, ct, N_CLASSES, -1, st, wl, wlen, gold=gt)
    assert np.array_equal(c.cpu().numpy()[0], counts_or[0])
    want = expected_state(stages_or[0], plan, cls, n)
    got = st.cpu().numpy().astype(np.uint32)
    bad = np.nonzero((got & DEFINED_BITS) != want)[0]
    assert len(bad) == 0, f"tuple_state differs at {bad[:8]}: {got[bad[:4]]} vs {want[bad[:4]]}"
    assert set(wl[:int(wlen.item())].cpu().tolist()) == set(np.nonzero(alive_or[0])[0].tolist())
    # ko_route stage by stage: the worklist after stage s is exactly who reaches stage s + 1
    st2 = torch.ones(n, dtype=torch.int32, device="cuda")
    c2 = torch.zeros((1, 37), dtype=torch.int64, device="cuda")
    for s in range(len(plan)):
        ko.route(plan, mt, ct, N_CLASSES, s, st2, wl, wlen, counts=c2)
        if s + 1 < len(plan):
            got_wl = set(wl[:int(wlen.item())].cpu().tolist())
            assert got_wl == set(np.nonzero(stages_or[0, s + 1])[0].tolist()), f"stage {s + 1}"
    assert np.array_equal(c2.cpu().numpy()[0, 5:], counts_or[0, 5:])
    assert torch.equal(st, st2)


def test_score_batch_external_boundaries(ko):
    """The scoring kernel's own plan evaluation (grid mode) and the routed executor (walk kernel)
    on boundary margins supplied through an external variant (the embedding-stage hook)."""
    wl = workloads.get("C1")
    n = wl.n_tuples
    d = device_workload(wl, n=n, placement="affine")
    variants = [(1000, 1), (0, 0)]                    # KV gold variant + external stage variant
    vals = np.array(FILTER_VALS + [F32(5.0), F32(-5.0)], np.float32)
    ext = np.resize(vals, n)                          # every boundary value, cycled over tuples
    plan = [(0, 1, float(LO), float(HI), 0), (0, 0, 0.0, 0.0, 1)]
    m_or, c_or = oracle.score_workload(wl, np.arange(n), variants=[(1000, 1)])
    m_full = np.zeros((1, 2, n))
    m_full[0, 0] = m_or[0, 0]
    m_full[0, 1] = ext
    c_full = np.zeros((1, 2, n), np.int32)
    gold = (m_or[0, 0] > 0).astype(np.uint8)[None]    # P_g: the gold variant's decision
    cnt_or, alive_or, stages_or = oracle.run_plans([plan], m_full, c_full, [1], gold,
                                                   want_alive=True, want_stages=True)
    gt = torch.from_numpy(gold).cuda()
    # grid mode: in-kernel eval_plan over two plans
    mg = torch.empty((1, 2, n), dtype=torch.float32, device="cuda")
    mg[0, 1] = torch.from_numpy(ext).cuda()
    _, _, cnt = ko.score_batch(d["kv"], d["ops"], variants, margins=mg, plans=[plan, plan],
                               gold=gt)
    torch.cuda.synchronize()
    assert torch.equal(mg[0, 1].cpu(), torch.from_numpy(ext))      # external margins untouched
    parity.assert_margins(mg.cpu().numpy()[:, :1], m_or)
    for row in cnt.cpu().numpy():
        parity.assert_counts(row[None], m_full, c_full, mg.cpu().numpy(),
                             np.zeros((1, 2, n), np.int32), [plan], [1], gold)
    # routed mode: the external stage decides who is streamed at all
    mr = torch.empty((1, 2, n), dtype=torch.float32, device="cuda")
    mr[0, 1] = torch.from_numpy(ext).cuda()
    _, _, cnt_r = ko.score_batch(d["kv"], d["ops"], variants, margins=mr, plans=[plan], gold=gt)
    torch.cuda.synchronize()
    reached_gpu = np.isfinite(mr.cpu().numpy()[0, 0])
    assert np.array_equal(reached_gpu, stages_or[0, 1] != 0)      # exact: the ext decision is
    parity.assert_counts(cnt_r.cpu().numpy(), m_full, c_full, mr.cpu().numpy(),
                         np.zeros((1, 2, n), np.int32), [plan], [1], gold)
    assert (stages_or[0, 0] == oracle.STAGE_UNSURE).sum() >= n // 4
