"""GPU parity: the CUDA path (through the C ABI) against the oracle on the same seeded inputs.
Tolerances: margins 2e-3 absolute; decisions and counts bit-exact outside the 1e-2 ambiguity band
(tests/parity.py)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import kogen  # noqa: E402
import oracle  # noqa: E402
from kogen import workloads  # noqa: E402
from kogen.device import device_workload, tensors_to_device  # noqa: E402
from tests import parity  # noqa: E402
from tests.helpers import Geom, build_pool, random_problem  # noqa: E402


@pytest.fixture(scope="module")
def ko():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2602_04430_b200 as ko
    return ko


def run_oracle_on_host(pool, indptr, ids, sl, geom, ops, variants):
    return oracle.score(geom, pool, indptr, ids, sl, ops, variants)


CASES = [
    # (name, geom, lengths, classes, variants)
    ("d64_g1", Geom(1, 1, 1, 64, 1), [128] * 5 + [1, 7, 16, 17, 100], (1,),
     [(1000, 1), (500, 1), (137, 1)]),
    ("d128_g4_2ops", Geom(2, 2, 4, 128, 1), [1, 15, 16, 33, 64, 200, 257], (1, 1),
     [(1000, 2), (500, 2), (200, 1), (1, 1)]),
    ("d128_map4", Geom(2, 2, 4, 128, 1), [5, 31, 48, 130], (4,), [(1000, 2), (300, 1)]),
    ("d64_rows12_maps", Geom(2, 1, 4, 64, 1), [3, 40, 77], (1, 3, 1), [(1000, 2), (600, 2), (250, 1)]),
    ("d128_nq2_rows16", Geom(1, 2, 4, 128, 2), [9, 63, 64, 65], (1, 2), [(1000, 1), (777, 1)]),
    ("d64_c8", Geom(1, 1, 2, 64, 1), [20, 50], (8,), [(1000, 1)]),
    ("d128_map3_g2", Geom(2, 2, 2, 128, 2), [7, 40, 100], (3,), [(1000, 2), (500, 1)]),
]


@pytest.mark.parametrize("w_bf16", [False, True], ids=["w_fp32", "w_bf16"])
@pytest.mark.parametrize("name,geom,lengths,classes,variants", CASES, ids=[c[0] for c in CASES])
def test_score_parity_random(ko, name, geom, lengths, classes, variants, w_bf16):
    """fp32 readouts (bf16 hi + lo tiles) and bf16 readouts (two classes per tile for maps)."""
    rng = np.random.default_rng(abs(hash(name)) % 2**32)
    K, V, ops_h = random_problem(rng, geom, lengths, n_ops=len(classes), classes=classes)
    pool, indptr, ids, sl = build_pool(K, V, lengths, poison=True)
    m_or, c_or = run_oracle_on_host(pool, indptr, ids, sl, geom, ops_h, variants)
    kv, ops = tensors_to_device(pool, indptr, ids, sl, geom, ops_h)
    if w_bf16:                                       # the random readouts are exact in bf16
        for op in ops:
            wb = op.w.to(torch.bfloat16)
            assert torch.equal(wb.float(), op.w)
            op.w = wb
    m, c, _ = ko.score_batch(kv, ops, variants)
    torch.cuda.synchronize()
    err = parity.assert_margins(m.cpu().numpy(), m_or)
    parity.assert_classes(c.cpu().numpy(), c_or, m_or, classes)
    assert err < 1e-3


def test_c1_grid_parity_and_counts(ko):
    wl = workloads.get("C1")
    d = device_workload(wl)
    m, c, counts = ko.score_batch(d["kv"], d["ops"], wl.variants, plans=wl.plans, gold=d["gold"])
    torch.cuda.synchronize()
    m_or, c_or = oracle.score_workload(wl, np.arange(wl.n_tuples))
    mg, cg = m.cpu().numpy(), c.cpu().numpy()
    parity.assert_margins(mg, m_or)
    gold = d["gold"].cpu().numpy()
    parity.assert_counts(counts.cpu().numpy(), m_or, c_or, mg, cg, wl.plans, wl.spec.op_classes,
                         gold)


def test_generator_twin_bitwise(ko):
    """Device fill ≡ host fill (the fixture both sides consume)."""
    for name, tids in (("C5", [0, 1, 777, 4095]), ("C3", [0, 5, 99])):
        wl = workloads.get(name)
        n = max(tids) + 1
        d = device_workload(wl, n=n, placement="affine")
        pool_d = d["kv"].pool.view(torch.int16).cpu().numpy().view(np.uint16)
        for t in tids:
            hp, hi, hid, hsl = kogen.host_pool(wl.spec, [t], placement="contiguous")
            L = int(hsl[0])
            for pi in range(int(hi[1])):
                dp = pool_d[d["page_ids"][d["indptr"][t] + pi]]
                hpg = hp[pi]
                valid = min(16, L - 16 * pi)
                assert np.array_equal(dp[:, :, :, :valid], hpg[:, :, :, :valid]), (name, t, pi)
                if valid < 16:                   # device poisons the unused tail slots
                    assert np.all(dp[:, :, :, valid:] == 0x7FC0)


def test_determinism_order_and_placement(ko):
    wl = workloads.get("C5")
    n = 300
    d = device_workload(wl, n=n)
    m1, _, c1 = ko.score_batch(d["kv"], d["ops"], wl.variants, plans=wl.plans, gold=d["gold"])
    m2, _, c2 = ko.score_batch(d["kv"], d["ops"], wl.variants, plans=wl.plans, gold=d["gold"])
    perm = torch.randperm(n, generator=torch.Generator().manual_seed(0)).to(torch.int32).cuda()
    m3, _, c3 = ko.score_batch(d["kv"], d["ops"], wl.variants, tuple_idx=perm, plans=wl.plans,
                               gold=d["gold"])
    d2 = device_workload(wl, n=n, placement="contiguous")
    m4, _, _ = ko.score_batch(d2["kv"], d2["ops"], wl.variants)
    torch.cuda.synchronize()
    assert torch.equal(m1, m2) and torch.equal(c1, c2)
    assert torch.equal(m1, m3) and torch.equal(c1, c3)
    assert torch.equal(m1, m4)


def test_sharded_counts_add_up(ko):
    """Σ of k shard passes (tuple subsets) = 1-shard counts, bit-exact (multi-GPU contract)."""
    wl = workloads.get("C5")
    n = 500
    d = device_workload(wl, n=n)
    _, _, full = ko.score_batch(d["kv"], d["ops"], wl.variants, plans=wl.plans, gold=d["gold"])
    acc = torch.zeros_like(full)
    idx = torch.arange(n, dtype=torch.int32, device="cuda")
    for shard in torch.tensor_split(idx, 3):
        ko.score_batch(d["kv"], d["ops"], wl.variants, tuple_idx=shard.contiguous(),
                       plans=wl.plans, gold=d["gold"], counts=acc)
    torch.cuda.synchronize()
    assert torch.equal(full, acc)


def test_reduce_and_route_exact_on_given_margins(ko):
    """ko_reduce_stats / ko_route on fixed margins equal the oracle's plan evaluation exactly."""
    rng = np.random.default_rng(0)
    n = 3000
    m = rng.normal(0, 2, size=(3, 2, n)).astype(np.float32)
    cls = rng.integers(0, 4, size=(3, 2, n)).astype(np.int32)
    n_classes = [1, 4, 1]
    gold = np.stack([rng.random(n) < 0.5, rng.integers(0, 4, n), rng.random(n) < 0.4]).astype(np.uint8)
    plans = [[(0, 0, -1.0, 1.0, 0), (0, 1, 0.0, 0.0, 1), (1, 0, 1.5, 1.5, 0), (1, 1, 0.0, 0.0, 1),
              (2, 0, -0.5, 0.5, 0), (2, 1, 0.25, 0.25, 1)],
             [(2, 1, 0.0, 0.0, 1), (0, 0, -2.0, 0.5, 0), (0, 1, 0.0, 0.0, 1)],
             [(1, 1, 0.0, 0.0, 1)]]
    mt, ct, gt = (torch.from_numpy(x).cuda() for x in (m, cls, gold))
    counts = ko.reduce_stats(plans, mt, ct, n_classes, gold=gt)
    expect = oracle.run_plans(plans, m.astype(np.float64), cls, n_classes, gold)
    assert np.array_equal(counts.cpu().numpy(), expect)
    # whole plan via ko_route(stage = -1) and stage by stage via ko_route(stage = s)
    for pl, ex in zip(plans, expect):
        st = torch.ones(n, dtype=torch.int32, device="cuda")
        wl_ = torch.empty(n, dtype=torch.int32, device="cuda")
        wlen = torch.zeros(1, dtype=torch.int64, device="cuda")
        c = ko.route(pl, mt, ct, n_classes, -1, st, wl_, wlen, gold=gt)
        assert np.array_equal(c.cpu().numpy()[0], ex)
        assert int(wlen.item()) == ex[3]
        st2 = torch.ones(n, dtype=torch.int32, device="cuda")
        c2 = torch.zeros((1, 37), dtype=torch.int64, device="cuda")
        for s in range(len(pl)):
            ko.route(pl, mt, ct, n_classes, s, st2, wl_, wlen, counts=c2)
            if s + 1 < len(pl):   # the worklist is exactly the set reaching stage s+1
                got = set(wl_[:int(wlen.item())].cpu().tolist())
                o_next = pl[s + 1][0]
                sv = st2.cpu().numpy().astype(np.uint32)
                want = set(np.nonzero((sv & 1) & (((sv >> (1 + 2 * o_next)) & 3) == 0))[0].tolist())
                assert got == want
        assert torch.equal(st, st2)
        assert np.array_equal(c2.cpu().numpy()[0, 5:], ex[5:])


def test_routed_mode_parity(ko):
    """Routed execution (n_plans == 1) of a filter → map → filter cascade plan."""
    wl = workloads.get("C4")
    n = 2000
    d = device_workload(wl, n=n)
    plan = wl.plans[0]
    m, c, counts = ko.score_batch(d["kv"], d["ops"], wl.variants, plans=[plan], gold=d["gold"])
    torch.cuda.synchronize()
    m_or, c_or = oracle.score_workload(wl, np.arange(n))
    mg, cg = m.cpu().numpy(), c.cpu().numpy()
    reached = np.isfinite(mg)
    parity.assert_margins(mg, m_or, mask=reached)
    gold = d["gold"].cpu().numpy()
    parity.assert_counts(counts.cpu().numpy(), m_or, c_or, mg, cg, [plan], wl.spec.op_classes, gold)
    # grid mode on the same plan gives the same counts (execution strategy does not matter)
    mg2, cg2, cnt2 = ko.score_batch(d["kv"], d["ops"], wl.variants, plans=[plan, plan], gold=d["gold"])
    torch.cuda.synchronize()
    assert np.array_equal(cnt2.cpu().numpy()[0], counts.cpu().numpy()[0])


def test_empty_and_single_token(ko):
    geom = Geom(1, 1, 1, 64, 1)
    rng = np.random.default_rng(1)
    K, V, ops_h = random_problem(rng, geom, [1, 1, 2])
    pool, indptr, ids, sl = build_pool(K, V, [1, 1, 2], poison=True)
    kv, ops = tensors_to_device(pool, indptr, ids, sl, geom, ops_h)
    m_or, _ = oracle.score(geom, pool, indptr, ids, sl, ops_h, [(1000, 1), (1, 1)])
    m, _, _ = ko.score_batch(kv, ops, [(1000, 1), (1, 1)])
    torch.cuda.synchronize()
    parity.assert_margins(m.cpu().numpy(), m_or, tol=1e-4)
    empty = torch.empty(0, dtype=torch.int32, device="cuda")
    m2 = torch.full_like(m, 7.0)
    ko.score_batch(kv, ops, [(1000, 1), (1, 1)], tuple_idx=empty, margins=m2)
    torch.cuda.synchronize()
    assert torch.all(m2 == 7.0)


def test_error_paths(ko):
    wl = workloads.get("C1")
    d = device_workload(wl, n=4)
    with pytest.raises(ko.KoError, match="keep_permille"):
        ko.score_batch(d["kv"], d["ops"], [(0, 1)])
    with pytest.raises(ko.KoError, match="layer_cut"):
        ko.score_batch(d["kv"], d["ops"], [(1000, 2)])
    with pytest.raises(ko.KoError, match="no final"):
        ko.score_batch(d["kv"], d["ops"], wl.variants, plans=[[(0, 1, -1, 1, 0)], [(0, 0, 0, 0, 1)]])
    ws = torch.empty(64, dtype=torch.uint8, device="cuda")
    with pytest.raises(ko.KoError, match="workspace"):
        ko.score_batch(d["kv"], d["ops"], wl.variants, workspace=ws)


def test_routed_rounds_c2_plan(ko):
    """Routed execution by rounds of nested extents on a 2-filter, 3-variant cascade plan."""
    wl = workloads.get("C2")
    n = 600
    d = device_workload(wl, n=n)
    plan = wl.plans[5]
    m, c, counts = ko.score_batch(d["kv"], d["ops"], wl.variants, plans=[plan], gold=d["gold"])
    _, _, grid = ko.score_batch(d["kv"], d["ops"], wl.variants, plans=[plan, plan], gold=d["gold"])
    torch.cuda.synchronize()
    m_or, c_or = oracle.score_workload(wl, np.arange(n))
    mg, cg = m.cpu().numpy(), c.cpu().numpy()
    reached = np.isfinite(mg)
    assert reached[0, 0].all()                       # every tuple meets the first stage
    assert not reached.all()                         # ... and the cascade skips work
    parity.assert_margins(mg, m_or, mask=reached)
    parity.assert_counts(counts.cpu().numpy(), m_or, c_or, mg, cg, [plan], wl.spec.op_classes,
                         d["gold"].cpu().numpy())
    assert np.array_equal(grid.cpu().numpy()[0], counts.cpu().numpy()[0])


def test_routed_fallback_many_rows(ko):
    """Plans whose ops need > 16 rows per kv-head run one launch per stage (fallback path)."""
    geom = Geom(2, 1, 4, 64, 2)                      # 8 rows per op, 3 ops = 24 rows
    rng = np.random.default_rng(11)
    lengths = [5, 40, 64, 90, 17, 33]
    K, V, ops_h = random_problem(rng, geom, lengths, n_ops=3, classes=(1, 3, 1))
    pool, indptr, ids, sl = build_pool(K, V, lengths, poison=True)
    variants = [(400, 1), (1000, 2)]
    plan = [(0, 0, -0.05, 0.05, 0), (0, 1, 0.0, 0.0, 1), (1, 0, 0.1, 0.1, 0), (1, 1, 0.0, 0.0, 1),
            (2, 1, 0.0, 0.0, 1)]
    m_or, c_or = oracle.score(geom, pool, indptr, ids, sl, ops_h, variants)
    gold = np.stack([(m_or[0, 1] > 0), c_or[1, 1], (m_or[2, 1] > 0)]).astype(np.uint8)
    kv, ops = tensors_to_device(pool, indptr, ids, sl, geom, ops_h)
    m, c, counts = ko.score_batch(kv, ops, variants, plans=[plan],
                                  gold=torch.from_numpy(gold).cuda())
    torch.cuda.synchronize()
    mg, cg = m.cpu().numpy(), c.cpu().numpy()
    parity.assert_margins(mg, m_or, mask=np.isfinite(mg))
    parity.assert_counts(counts.cpu().numpy(), m_or, c_or, mg, cg, [plan], [1, 3, 1], gold)


@pytest.mark.parametrize("variants,plan", [
    # rank 0 = (1000, 1) covers layer 0 entirely; (500, 2)'s layer-0 snapshot is taken in round 0
    # and its layer-1 one in round 1 (partials persist across the rounds of the call)
    ([(1000, 1), (500, 2)], [(0, 0, 0.25, 0.75, 0), (0, 1, 0.5, 0.5, 1)]),
    # three nested ranks, a map and a filter fused into one read, resumed twice
    ([(200, 1), (500, 2), (1000, 2)], [(0, 0, 0.3, 0.7, 0), (1, 0, 0.6, 0.6, 0),
                                       (0, 1, 0.3, 0.7, 0), (1, 1, 0.5, 0.5, 1),
                                       (0, 2, 0.5, 0.5, 1)]),
    # the cheap stage is the later variant in plan order: ranks follow extents, not the plan
    ([(1000, 2), (300, 1)], [(0, 1, 0.25, 0.75, 0), (0, 0, 0.5, 0.5, 1)]),
], ids=["cross_round_partials", "three_ranks_fused_map", "ranks_by_extent"])
def test_routed_resumable_extents(ko, variants, plan):
    """Routed mode streams, per (tuple, layer), only the tokens past what earlier rounds read and
    resumes their saved softmax state: every reached margin equals the oracle's."""
    geom = Geom(2, 2, 4, 128, 1)
    rng = np.random.default_rng(21)
    lengths = [1, 2, 15, 16, 17, 31, 48, 64, 100, 127, 128, 129, 200, 300]
    n_ops = 1 + max(o for (o, *_r) in plan)
    classes = (1, 4)[:n_ops]
    K, V, ops_h = random_problem(rng, geom, lengths, n_ops=n_ops, classes=classes)
    pool, indptr, ids, sl = build_pool(K, V, lengths, poison=True, seed=3)
    m_or, c_or = oracle.score(geom, pool, indptr, ids, sl, ops_h, variants)
    # thresholds at oracle-margin quantiles so every stage sends tuples onward
    plan = [(o, v, float(np.quantile(m_or[o, v], qlo)), float(np.quantile(m_or[o, v], qhi)), f)
            for (o, v, qlo, qhi, f) in plan]
    gold = np.stack([(m_or[o, -1] > 0) if classes[o] <= 1 else c_or[o, -1]
                     for o in range(n_ops)]).astype(np.uint8)
    kv, ops = tensors_to_device(pool, indptr, ids, sl, geom, ops_h)
    m, c, counts = ko.score_batch(kv, ops, variants, plans=[plan], gold=torch.from_numpy(gold).cuda())
    torch.cuda.synchronize()
    mg, cg = m.cpu().numpy(), c.cpu().numpy()
    reached = np.isfinite(mg)
    assert reached.sum() > len(lengths)               # later rounds were reached
    parity.assert_margins(mg, m_or, mask=reached)
    parity.assert_counts(counts.cpu().numpy(), m_or, c_or, mg, cg, [plan], list(classes), gold)


def test_routed_subset_and_launch_count(ko):
    """Routed mode on a tuple subset (tuple_idx): only subset tuples are scored (the rest stay
    NaN) and the counts equal the oracle's on the subset; ko_last_launch_count reports the
    library's launches (prep once per group, score + walk per launched position, final counts)."""
    wl = workloads.get("C4")
    n = 3000
    d = device_workload(wl, n=n)
    plan = wl.plans[0]
    sub = np.arange(7, n, 5, dtype=np.int32)
    m, c, counts = ko.score_batch(d["kv"], d["ops"], wl.variants, plans=[plan], gold=d["gold"],
                                  tuple_idx=torch.from_numpy(sub).cuda())
    torch.cuda.synchronize()
    launches = ko.last_launch_count()
    mg, cg = m.cpu().numpy(), c.cpu().numpy()
    outside = np.setdiff1d(np.arange(n), sub)
    assert np.isnan(mg[:, :, outside]).all()
    m_or, c_or = oracle.score_workload(wl, np.arange(n))
    gold = d["gold"].cpu().numpy()
    parity.assert_margins(mg[:, :, sub], m_or[:, :, sub], mask=np.isfinite(mg[:, :, sub]))
    parity.assert_counts(counts.cpu().numpy(), m_or[:, :, sub], c_or[:, :, sub], mg[:, :, sub],
                         cg[:, :, sub], [plan], wl.spec.op_classes, gold[:, sub])
    # C4's plan: one fused group; positions 0 and 1 launched (2 and 4 are covered by 0; 3 and 5
    # would only repeat position 1's (group, rank 1), so no walk can queue a tuple to them)
    assert launches == 1 + 2 * 2 + 1
    # caller-owned margins: the tuples outside tuple_idx are not touched (chunked routed calls keep
    # every chunk's results), the subset's unreached entries read NaN
    mine = torch.full_like(m, 7.0)
    ko.score_batch(d["kv"], d["ops"], wl.variants, plans=[plan], gold=d["gold"], margins=mine,
                   tuple_idx=torch.from_numpy(sub).cuda())
    torch.cuda.synchronize()
    mm = mine.cpu().numpy()
    assert (mm[:, :, outside] == 7.0).all()
    assert np.array_equal(np.isnan(mm[:, :, sub]), np.isnan(mg[:, :, sub]))
    assert np.array_equal(mm[:, :, sub][np.isfinite(mm[:, :, sub])], mg[:, :, sub][np.isfinite(mg[:, :, sub])])


def test_routed_wide_map_alone(ko):
    """A 4-class fp32-readout map on 16 rows per kv-head (G = 4, n_q = 4): 8 W·V entries per row
    need 8 table tiles, so the operator runs alone in its group; routed margins and counts still
    match the oracle."""
    geom = Geom(1, 1, 4, 64, 4)
    rng = np.random.default_rng(8)
    lengths = [3, 16, 40, 77, 128]
    K, V, ops_h = random_problem(rng, geom, lengths, n_ops=1, classes=(4,))
    pool, indptr, ids, sl = build_pool(K, V, lengths, poison=True)
    variants = [(300, 1), (1000, 1)]
    m_or, c_or = oracle.score(geom, pool, indptr, ids, sl, ops_h, variants)
    th = float(np.quantile(m_or[0, 0], 0.5))
    plan = [(0, 0, th, th, 0), (0, 1, 0.0, 0.0, 1)]
    gold = c_or[0, 1][None].astype(np.uint8)
    kv, ops = tensors_to_device(pool, indptr, ids, sl, geom, ops_h)
    m, c, counts = ko.score_batch(kv, ops, variants, plans=[plan], gold=torch.from_numpy(gold).cuda())
    torch.cuda.synchronize()
    mg, cg = m.cpu().numpy(), c.cpu().numpy()
    parity.assert_margins(mg, m_or, mask=np.isfinite(mg))
    parity.assert_counts(counts.cpu().numpy(), m_or, c_or, mg, cg, [plan], [4], gold)


@pytest.mark.parametrize("cfg", ["C4", "C5"])
def test_cuda_graph_capture_replay(ko, cfg):
    """The whole pass (routed C4 / grid C5) is asynchronous on the caller's stream with no host
    synchronisation, so it can be captured once in a CUDA graph and replayed: replays give the
    eager call's margins and counts bit for bit."""
    wl = workloads.get(cfg)
    n = 2000
    d = device_workload(wl, n=n)
    nv, no = len(wl.variants), wl.spec.n_ops
    m = torch.empty((no, nv, n), dtype=torch.float32, device="cuda")
    c = torch.empty((no, nv, n), dtype=torch.int32, device="cuda")
    counts = torch.zeros((len(wl.plans), ko.COUNTS_PER_PLAN), dtype=torch.int64, device="cuda")
    ws = ko.alloc_workspace(d["kv"], d["ops"], nv, n)

    def step():
        counts.zero_()
        ko.score_batch(d["kv"], d["ops"], wl.variants, margins=m, classes=c, plans=wl.plans,
                       gold=d["gold"], counts=counts, workspace=ws)

    step()
    torch.cuda.synchronize()
    m0, c0, k0 = m.clone(), c.clone(), counts.clone()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            step()
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(2):
        m.fill_(7.0)
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(torch.nan_to_num(m, nan=-9.0), torch.nan_to_num(m0, nan=-9.0))
    assert torch.equal(c[torch.isfinite(m0)], c0[torch.isfinite(m0)])
    assert torch.equal(counts, k0)


def test_routed_without_labels(ko):
    """Execution on unlabelled data (gold = NULL, §8(b)): TP/FP/FN/|P_g| stay 0, |P_o| and every
    per-stage count equal the labelled run's (labels never steer routing, Q14)."""
    wl = workloads.get("C4")
    n = 1500
    d = device_workload(wl, n=n)
    plan = wl.plans[0]
    _, _, k_gold = ko.score_batch(d["kv"], d["ops"], wl.variants, plans=[plan], gold=d["gold"])
    m, _, k_none = ko.score_batch(d["kv"], d["ops"], wl.variants, plans=[plan], gold=None)
    torch.cuda.synchronize()
    kg, kn = k_gold.cpu().numpy()[0], k_none.cpu().numpy()[0]
    assert kn[0] == kn[1] == kn[2] == kn[4] == 0
    assert kn[3] == kg[3] and np.array_equal(kn[5:], kg[5:])
    assert np.isfinite(m.cpu().numpy()).any()


def test_routed_resume_long_sequences(ko):
    """Routed resume on C3's long variable-length caches (256–4096 tokens, up to 256 pages per
    kv-head): round 1 restarts past page 32 (a later page-id chunk) from the saved state; reached
    margins and counts match the oracle."""
    wl = workloads.get("C3")
    n = 160
    d = device_workload(wl, n=n)
    m_or, c_or = oracle.score_workload(wl, np.arange(n))
    # C3's variants: (1000,1) (500,1) (200,1) (1000,2) (500,2) (200,2); cascade 200‰/1 → 500‰/2 → gold
    v_small, v_mid, v_gold = 2, 4, 3
    q = lambda v, a: float(np.quantile(m_or[0, v], a))
    plan = [(0, v_small, q(v_small, 0.3), q(v_small, 0.7), 0), (0, v_mid, q(v_mid, 0.4), q(v_mid, 0.6), 0),
            (0, v_gold, 0.0, 0.0, 1)]
    m, c, counts = ko.score_batch(d["kv"], d["ops"], wl.variants, plans=[plan], gold=d["gold"])
    torch.cuda.synchronize()
    mg, cg = m.cpu().numpy(), c.cpu().numpy()
    reached = np.isfinite(mg)
    assert reached[0, v_gold].any() and not reached[0, v_gold].all()
    parity.assert_margins(mg, m_or, mask=reached)
    parity.assert_counts(counts.cpu().numpy(), m_or, c_or, mg, cg, [plan], wl.spec.op_classes,
                         d["gold"].cpu().numpy())
