"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (one resident
batch of wl.bench_n tuples per GPU): margins of a random sample of tuples against the oracle
(computed one by one), and the count property that holds at any size — the GPU counts equal the
oracle's plan evaluation (oracle.run_plans) applied to the GPU's own margins, exactly."""
import gc

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from kogen import workloads  # noqa: E402
from kogen.device import device_workload  # noqa: E402
from tests import parity  # noqa: E402

N_SAMPLE = 48


@pytest.fixture(scope="module")
def ko():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2602_04430_b200 as ko
    return ko


@pytest.mark.parametrize("name", ["C2", "C5", "C3", "C4"])
def test_full_size(ko, name):
    wl = workloads.get(name)
    n = wl.bench_n
    free, _ = torch.cuda.mem_get_info()
    d = device_workload(wl, n=n, placement="contiguous")
    plans = wl.plans
    m, c, counts = ko.score_batch(d["kv"], d["ops"], wl.variants, plans=plans, gold=d["gold"])
    torch.cuda.synchronize()
    mg, cg = m.cpu().numpy(), c.cpu().numpy()
    gold = d["gold"].cpu().numpy()
    routed = len(plans) == 1
    if not routed:
        assert np.isfinite(mg).all()
    # counts == oracle plan evaluation of the GPU's own margins (exact at any size)
    expect = oracle.run_plans(plans, mg.astype(np.float64), cg, wl.spec.op_classes, gold)
    assert np.array_equal(counts.cpu().numpy(), expect)
    # sampled margins vs the oracle, one tuple at a time
    rng = np.random.default_rng(7)
    sample = np.sort(rng.choice(n, size=N_SAMPLE, replace=False))
    sample[0] = n - 1                                  # include the last tuple
    m_or, c_or = oracle.score_workload(wl, sample)
    sub = mg[:, :, sample]
    mask = np.isfinite(sub) if routed else None
    if routed:
        assert mask.any()
    err = parity.assert_margins(sub, m_or, mask=mask)
    parity.assert_classes(np.where(np.isfinite(sub), cg[:, :, sample], c_or), c_or, m_or,
                          wl.spec.op_classes)
    print(f"{name}: n={n} max|dm| over {N_SAMPLE} sampled tuples = {err:.2e}")
    del d, m, c, counts
    gc.collect()
    torch.cuda.empty_cache()
