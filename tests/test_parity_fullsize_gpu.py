"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (one resident
batch of wl.bench_n tuples per GPU, the bench's page placement), against the ORACLE on every tuple
it scores — SURVEY §8(d) "Oracle timing": full inputs for C2 and C5; for C3 and C4 a deterministic
every-k-th subset of >= 20 k tuples, which the GPU also reruns as its own pass via tuple_idx.

Asserted (north star):
  * margins within 2e-3 of the oracle on every (op, variant, tuple) the GPU computed;
  * counts exactly equal to oracle.run_plans on the merged margins (Q19 (iii)), with gold = the
    paper's P_g (the oracle's gold-variant decision);
  * per tuple, for every plan: P_o membership (ko_route on the GPU's margins) equal to the oracle's
    outside the ±1e-2 band (Eqs. accept-i / reject-i / unsure-i); routed mode: also the
    reached set (finite margins) equal to the oracle's reached set outside the band;
  * a tuple's margins are bitwise the same in the full pass and in the subset pass.
The oracle reads the generator's pages copied from the device (tests/fullsize.py, checked bitwise
against the host twin)."""
import gc
import time
import traceback

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from kogen import workloads  # noqa: E402
from kogen.device import device_workload  # noqa: E402
from tests import fullsize, parity  # noqa: E402

# config: (resident batches of bench_n tuples, every k-th tuple scored by the oracle)
CASES = {"C2": (1, 1), "C5": (1, 1), "C3": (4, 2), "C4": (1, 6)}


@pytest.fixture(scope="module")
def ko():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2602_04430_b200 as ko
    return ko


def _free():
    gc.collect()
    torch.cuda.empty_cache()


def _check_plans(ko, plans, n_classes, m_or, c_or, mg_t, cg_t, gold, routed):
    """Per-tuple decisions of every plan against the oracle, outside the band."""
    n_clear_min = None
    _, alive_or, stages_or = oracle.run_plans(plans, m_or, c_or, n_classes, gold, want_alive=True,
                                              want_stages=True)
    mg = mg_t.cpu().numpy()
    for g, pl in enumerate(plans):
        clear = parity.clear_tuples(m_or, pl, n_classes)
        alive, _ = parity.gpu_alive(ko, pl, mg_t, cg_t, n_classes)
        bad = np.nonzero(clear & (alive != alive_or[g].astype(bool)))[0]
        assert len(bad) == 0, f"plan {g}: P_o membership differs on clear tuples {bad[:10]}"
        if routed:
            r_or = parity.oracle_reached(stages_or[g], pl, m_or.shape)
            r_gpu = np.isfinite(mg)
            diff = (r_or != r_gpu).any(axis=(0, 1)) & clear
            assert not diff.any(), f"reached set differs on clear tuples {np.nonzero(diff)[0][:10]}"
        n_clear_min = int(clear.sum()) if n_clear_min is None else min(n_clear_min, int(clear.sum()))
    return n_clear_min


@pytest.mark.parametrize("name", ["C2", "C5", "C4", "C3"])
def test_full_size_vs_oracle(ko, name):
    wl = workloads.get(name)
    n_batches, k = CASES[name]
    n = wl.bench_n
    routed = len(wl.plans) == 1
    ncls = wl.spec.op_classes
    stats = {"worst": 0.0, "n_or": 0, "n_band": 0, "t_or": 0.0}
    _free()
    for b in range(n_batches):
        try:
            n_clear = _one_batch(ko, wl, b, n, k, routed, ncls, stats)
        except BaseException as e:      # drop the failed batch's 100+ GB of locals for the next case
            traceback.clear_frames(e.__traceback__)
            raise
        finally:
            _free()
    worst, n_or, n_band_tot, t_or = stats["worst"], stats["n_or"], stats["n_band"], stats["t_or"]
    print(f"{name}: {n_or} tuples vs oracle ({t_or:.0f} s), max|dm| = {worst:.2e}, "
          f"band entries = {n_band_tot}, min clear tuples per plan = {n_clear}")


def _one_batch(ko, wl, b, n, k, routed, ncls, stats):
    t0 = b * n
    d = device_workload(wl, t0=t0, n=n, placement=wl.placement)
    kv, ops = d["kv"], d["ops"]
    sub = np.arange(0, n, k, dtype=np.int64)
    if sub[-1] != n - 1:
        sub = np.append(sub, n - 1)                   # and the batch's last tuple
    tic = time.perf_counter()
    m_or, c_or = fullsize.oracle_scores(wl, d, t0, sub)
    stats["t_or"] += time.perf_counter() - tic
    stats["n_or"] += len(sub)
    gold_sub = parity.gold_from_oracle(m_or, c_or, wl.gold_variant, ncls)
    gold = d["gold"].clone()                          # latent labels off the oracle subset
    gold[:, torch.from_numpy(sub).cuda()] = torch.from_numpy(gold_sub).cuda()
    # (1) the bench launch: every tuple of the resident batch
    m_full, c_full, cnt_full = ko.score_batch(kv, ops, wl.variants, plans=wl.plans, gold=gold)
    torch.cuda.synchronize()
    mf = m_full.cpu().numpy()[:, :, sub]
    if not routed:
        assert np.isfinite(m_full.cpu().numpy()).all()
    mask = np.isfinite(mf) if routed else None
    stats["worst"] = max(stats["worst"], parity.assert_margins(mf, m_or, mask=mask))
    parity.assert_classes(np.where(np.isfinite(mf), c_full.cpu().numpy()[:, :, sub], c_or),
                          c_or, m_or, ncls)
    if k == 1:
        stats["n_band"] += parity.assert_counts(cnt_full.cpu().numpy(), m_or, c_or, mf,
                                           c_full.cpu().numpy(), wl.plans, ncls, gold_sub)
        mg_t, cg_t = m_full, c_full
    else:
        # (2) the subset as its own pass (tuple_idx): exact counts on exactly those tuples
        idx = torch.from_numpy(sub.astype(np.int32)).cuda()
        m_s, c_s, cnt_s = ko.score_batch(kv, ops, wl.variants, tuple_idx=idx, plans=wl.plans,
                                         gold=gold)
        torch.cuda.synchronize()
        ms = np.ascontiguousarray(m_s.cpu().numpy()[:, :, sub])
        cs = np.ascontiguousarray(c_s.cpu().numpy()[:, :, sub])
        fin = np.isfinite(ms)
        assert np.array_equal(np.isfinite(mf), fin)
        assert np.array_equal(ms[fin], mf[fin]), "full-pass and subset-pass margins differ"
        stats["n_band"] += parity.assert_counts(cnt_s.cpu().numpy(), m_or, c_or, ms, cs, wl.plans,
                                           ncls, gold_sub)
        mg_t = torch.from_numpy(ms).cuda()
        cg_t = torch.from_numpy(cs).cuda()
        del m_s, c_s
    n_clear = _check_plans(ko, wl.plans, ncls, m_or, c_or, mg_t, cg_t, gold_sub, routed)
    del d, kv, ops, m_full, c_full, mg_t, cg_t, gold
    return n_clear
