"""GPU parity of ko_soft_stats (NEXT-1) against the oracle (oracle/soft.py, torch fp64 +
autograd): values and Jacobian to ~1e-9 relative on the same margins."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import loss, soft  # noqa: E402


@pytest.fixture(scope="module")
def ko():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2602_04430_b200 as ko
    return ko


@pytest.mark.parametrize("tau", [1.0, 0.1, 0.01])
def test_soft_stats_parity(ko, tau):
    rng = np.random.default_rng(int(tau * 1000))
    n = 5000
    m = rng.normal(0, 2, size=(3, 3, n)).astype(np.float32)
    gold = (rng.random((3, n)) < 0.5).astype(np.uint8)
    plan = [(0, 0, -1.0, 0.7, 0), (2, 0, -0.3, 0.2, 0), (0, 1, -0.5, 0.5, 0), (0, 2, 0.0, 0.0, 1),
            (2, 2, 0.1, 0.1, 1), (1, 1, -0.2, 0.4, 0), (1, 2, -0.25, -0.25, 1)]
    pick = [0.3, -0.2, 0.1, 0.0, 0.0, 0.05, 0.0]
    cost = [1.0, 1.5, 3.0, 10.0, 10.0, 2.0, 10.0]
    exp = soft.soft_stats(plan, pick, tau, m.astype(np.float64), gold, cost)
    out = ko.soft_stats(plan, pick, cost, tau, torch.from_numpy(m).cuda(), [1, 1, 1],
                        gold=torch.from_numpy(gold).cuda())
    assert ko.last_launch_count() == 2        # per-tuple values with CTA sums, in-order final sum
    got = out.cpu().numpy()
    S = len(plan)
    assert np.allclose(got[:4], exp["values"], rtol=1e-10, atol=1e-9)
    jac = got[4:].reshape(4, 3 * S)
    scale = np.abs(exp["jacobian"]).max()
    assert np.allclose(jac, exp["jacobian"], rtol=1e-8, atol=1e-10 * max(scale, 1.0))
    out2 = ko.soft_stats(plan, pick, cost, tau, torch.from_numpy(m).cuda(), [1, 1, 1],
                         gold=torch.from_numpy(gold).cuda())
    assert torch.equal(out, out2)                      # fixed-order sums: bitwise reproducible


@pytest.mark.parametrize("tau", [1.0, 0.05])
def test_soft_stats_map_plan_parity(ko, tau):
    """Filter → 4-class map → filter cascades (C4's shape) relaxed with the map's output-tuple
    selection, against the oracle: values and the Jacobian."""
    rng = np.random.default_rng(int(tau * 100) + 3)
    n = 6000
    m = rng.normal(0, 2, size=(3, 2, n)).astype(np.float32)
    m[1] = np.abs(m[1])
    cls = rng.integers(0, 4, size=(3, 2, n)).astype(np.int32)
    cls[[0, 2]] = 0
    gold = np.stack([rng.random(n) < 0.5, rng.integers(0, 4, n), rng.random(n) < 0.5]).astype(np.uint8)
    plan = [(0, 0, -1.0, 0.7, 0), (0, 1, 0.0, 0.0, 1), (1, 0, 0.5, 0.5, 0), (1, 1, 0.0, 0.0, 1),
            (2, 0, -0.4, 0.4, 0), (2, 1, 0.1, 0.1, 1)]
    pick = [0.3, 0.0, -0.2, 0.0, 0.1, 0.0]
    cost = [1.0, 10.0, 2.0, 12.0, 1.5, 9.0]
    exp = soft.soft_stats(plan, pick, tau, m.astype(np.float64), gold, cost, cls, [1, 4, 1])
    out = ko.soft_stats(plan, pick, cost, tau, torch.from_numpy(m).cuda(), [1, 4, 1],
                        gold=torch.from_numpy(gold).cuda(), classes=torch.from_numpy(cls).cuda())
    got = out.cpu().numpy()
    assert np.allclose(got[:4], exp["values"], rtol=1e-10, atol=1e-9)
    jac = got[4:].reshape(4, 3 * len(plan))
    assert np.allclose(jac, exp["jacobian"], rtol=1e-8,
                       atol=1e-10 * max(np.abs(exp["jacobian"]).max(), 1.0))
    with pytest.raises(ko.KoError, match="classes"):
        ko.soft_stats(plan, pick, cost, tau, torch.from_numpy(m).cuda(), [1, 4, 1])


@pytest.mark.parametrize("tr,tpr", [(0.05, 0.05), (0.99, 0.99)])
def test_loss_gradient_through_gpu_jacobian(ko, tr, tpr):
    """NEXT-2 chain: ko_soft_stats' GPU Jacobian → ko_plan_loss → dL/d(s, θ⁻, θ⁺), against the
    oracle's relaxation + loss (oracle/loss.py)."""
    rng = np.random.default_rng(17)
    n = 20000
    m = rng.normal(0, 2, size=(2, 2, n)).astype(np.float32)
    gold = (rng.random((2, n)) < 0.4).astype(np.uint8)
    plan = [(0, 0, -0.8, 0.6, 0), (0, 1, 0.0, 0.0, 1), (1, 0, -0.4, 0.9, 0), (1, 1, 0.1, 0.1, 1)]
    pick, cost = [0.2, 0.0, -0.1, 0.0], [0.25, 1.0, 0.3, 1.0]
    vals_or, grad_or, _ = loss.soft_loss(plan, pick, 0.3, m.astype(np.float64), gold, cost, tr,
                                         tpr, 0.95, 10.0)
    out = ko.soft_stats(plan, pick, cost, 0.3, torch.from_numpy(m).cuda(), [1, 1],
                        gold=torch.from_numpy(gold).cuda()).cpu().numpy()
    v, g = ko.plan_loss(out[:4], cost, n, tr, tpr, 0.95, 10.0, jacobian=out[4:].reshape(4, -1))
    assert abs(v["loss"] - vals_or["loss"]) <= 1e-9 * max(1.0, vals_or["loss"])
    assert np.allclose(g, grad_or, rtol=1e-6, atol=1e-9 * np.abs(grad_or).max())


def _random_soft_problem(rng, n):
    """A random plan over a random subset of the 4 operator ids (exercising the kernel's compact
    operator slots), 1-2 stages per operator (the last one final), interleaved, maps mixed in."""
    n_ops, n_var = 4, 2
    used = sorted(rng.choice(n_ops, size=int(rng.integers(1, n_ops + 1)), replace=False).tolist())
    n_classes = [int(rng.choice([1, 1, 3])) for _ in range(n_ops)]
    seqs = []
    for o in used:
        k = int(rng.integers(1, 3))
        st = []
        for j in range(k):
            final = j == k - 1
            v = int(rng.integers(0, n_var))
            if final:
                th = float(rng.normal(0, 0.5)) if n_classes[o] == 1 else 0.0
                st.append((o, v, th, th, 1))
            else:
                lo, hi = sorted(rng.normal(0, 1, size=2).tolist())
                st.append((o, v, lo if n_classes[o] == 1 else hi, hi, 0))
        seqs.append(st)
    plan = []
    while any(seqs):
        i = int(rng.choice([j for j, s in enumerate(seqs) if s]))
        plan.append(seqs[i].pop(0))
    m = rng.normal(0, 2, size=(n_ops, n_var, n)).astype(np.float32)
    cls = np.zeros((n_ops, n_var, n), np.int32)
    gold = np.zeros((n_ops, n), np.uint8)
    for o in range(n_ops):
        if n_classes[o] > 1:
            m[o] = np.abs(m[o])
            cls[o] = rng.integers(0, n_classes[o], size=(n_var, n))
            gold[o] = rng.integers(0, n_classes[o], size=n)
        else:
            gold[o] = rng.random(n) < 0.5
    pick = rng.normal(0, 0.3, size=len(plan)).tolist()
    cost = rng.uniform(0.5, 10, size=len(plan)).tolist()
    return plan, pick, cost, m, cls, gold, n_classes


@pytest.mark.parametrize("seed,n", [(1, 1), (2, 77), (3, 5000), (4, 5000), (5, 9999), (6, 5000),
                                    (7, 160_000)])
def test_soft_stats_random_plans(ko, seed, n):
    """Random plans (1-4 operators with arbitrary ids, up to 8 stages, maps, tiny and multi-pass
    tuple counts: 160 k > one grid of the tuple kernel) against the oracle, bitwise repeatable."""
    rng = np.random.default_rng(seed)
    plan, pick, cost, m, cls, gold, ncl = _random_soft_problem(rng, n)
    tau = float(rng.choice([1.0, 0.2, 0.05]))
    exp = soft.soft_stats(plan, pick, tau, m.astype(np.float64), gold, cost, cls, ncl)
    args = (plan, pick, cost, tau, torch.from_numpy(m).cuda(), ncl)
    kw = dict(gold=torch.from_numpy(gold).cuda(), classes=torch.from_numpy(cls).cuda())
    out = ko.soft_stats(*args, **kw)
    got = out.cpu().numpy()
    assert np.allclose(got[:4], exp["values"], rtol=1e-10, atol=1e-9), (plan, got[:4], exp["values"])
    jac = got[4:].reshape(4, 3 * len(plan))
    assert np.allclose(jac, exp["jacobian"], rtol=1e-8,
                       atol=1e-10 * max(np.abs(exp["jacobian"]).max(), 1.0)), plan
    assert torch.equal(out, ko.soft_stats(*args, **kw))
