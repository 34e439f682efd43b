"""Routed mode must never read workspace state it did not write in the same call.  The saved
softmax states of position 0 are written only for tuples whose position-0 walk may resume them
(deferred save); a tuple resumed without its state would read whatever the
workspace held.  Run C4's cascade with a workspace poisoned with NaN bytes (not the caching
allocator's block from an identical earlier call) and require oracle parity, finite reached
margins, and bitwise the margins / counts of a zero-filled workspace."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from kogen import workloads  # noqa: E402
from kogen.device import device_workload  # noqa: E402
from tests import parity  # noqa: E402


@pytest.fixture(scope="module")
def ko():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2602_04430_b200 as ko
    return ko


def test_routed_c4_with_poisoned_workspace(ko):
    wl = workloads.get("C4")
    n = 4000
    d = device_workload(wl, n=n)
    plan = wl.plans[0]
    size = ko.workspace_size(d["kv"], d["ops"], len(wl.variants), n)
    res = []
    for fill in (0xFF, 0x00):                      # 0xFFFFFFFF = NaN as fp32
        ws = torch.full((size,), fill, dtype=torch.uint8, device="cuda")
        m, c, counts = ko.score_batch(d["kv"], d["ops"], wl.variants, plans=[plan],
                                      gold=d["gold"], workspace=ws)
        torch.cuda.synchronize()
        res.append((m.cpu().numpy(), c.cpu().numpy(), counts.cpu().numpy()))
    (m0, c0, k0), (m1, c1, k1) = res
    assert np.array_equal(m0.view(np.uint32), m1.view(np.uint32))
    reached = np.isfinite(m0)                      # classes of unreached entries: unspecified
    assert np.array_equal(c0[reached], c1[reached]) and np.array_equal(k0, k1)
    m_or, c_or = oracle.score_workload(wl, np.arange(n))
    # every variant of the plan is reached by some tuple, the large ones only via resumed state
    for o, v, *_ in plan:
        assert reached[o, v].any()
    parity.assert_margins(m0, m_or, mask=reached)
    parity.assert_counts(k0, m_or, c_or, m0, c0, [plan], wl.spec.op_classes,
                         d["gold"].cpu().numpy())
