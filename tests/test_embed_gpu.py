"""Embedding-similarity stage on the GPU (NEXT-3): ko_embed_scores vs the oracle, and cascades
whose cheap first stage is the embedding filter (external variant) in grid and routed mode."""
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


def _dev_bits(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda().view(torch.bfloat16)


@pytest.mark.parametrize("dim", [64, 256, 520])
def test_embed_scores_parity(ko, dim):
    wl = workloads.get("C5")
    n = 3001
    item, op = wl.spec.embeddings(0, n, dim)
    exp = oracle.embed_scores(item, op)
    m = torch.full((2, 2, n), 7.0, device="cuda")
    ko.embed_scores(_dev_bits(item), _dev_bits(op), [0, 1], m, variant=1)
    torch.cuda.synchronize()
    got = m.cpu().numpy()
    assert np.abs(got[:, 1, :] - exp).max() < 1e-5
    assert np.all(got[:, 0, :] == 7.0)                  # other variants untouched
    idx = torch.tensor([5, 3000, 17], dtype=torch.int32, device="cuda")
    m2 = torch.zeros((2, 2, n), device="cuda")
    ko.embed_scores(_dev_bits(item), _dev_bits(op), [1, 0], m2, variant=0, tuple_idx=idx)
    torch.cuda.synchronize()
    g2 = m2.cpu().numpy()
    assert np.abs(g2[1, 0, [5, 3000, 17]] - exp[0, [5, 3000, 17]]).max() < 1e-5
    assert np.count_nonzero(g2) == 6


@pytest.mark.parametrize("dim", [64, 128, 192, 256, 512])
def test_embed_scores_gathered(ko, dim):
    """tuple_idx path (per-lane 16-byte copies into padded rows): many full 16-row blocks plus a
    ragged tail, unsorted and repeated indices; entries outside the subset stay untouched."""
    wl = workloads.get("C5")
    n = 4099
    item, op = wl.spec.embeddings(3, n, dim)
    exp = oracle.embed_scores(item, op)
    rng = np.random.default_rng(dim)
    sub = rng.choice(n, size=2477, replace=False).astype(np.int32)
    sub = np.concatenate([sub, sub[:5]])              # repeats write the same value twice
    m = torch.full((2, 1, n), -9.0, device="cuda")
    ko.embed_scores(_dev_bits(item), _dev_bits(op), [0, 1], m, variant=0,
                    tuple_idx=torch.from_numpy(sub).cuda())
    torch.cuda.synchronize()
    got = m.cpu().numpy()[:, 0, :]
    assert np.abs(got[:, sub] - exp[:, sub]).max() < 1e-5
    rest = np.setdiff1d(np.arange(n), sub)
    assert np.all(got[:, rest] == -9.0)


def test_embedding_first_stage_cascade(ko):
    """C5-shaped cascade: [embedding stage (external) → KV gold] per filter, routed and grid."""
    wl = workloads.get("C5")
    n = 1500
    d = device_workload(wl, n=n)
    item, op = wl.spec.embeddings(0, n, 256)
    emb = oracle.embed_scores(item, op)                           # [2][n] fp64
    variants = list(wl.variants) + [(0, 0)]                        # variant 3 = external
    ev = len(variants) - 1
    c0 = [float(np.quantile(emb[o], 0.5)) for o in range(2)]
    plan = [(0, ev, c0[0] - 0.05, c0[0] + 0.05, 0), (0, 0, 0.0, 0.0, 1),
            (1, ev, c0[1] - 0.05, c0[1] + 0.05, 0), (1, 0, 0.0, 0.0, 1)]
    margins = torch.empty((2, len(variants), n), device="cuda")
    ko.embed_scores(_dev_bits(item), _dev_bits(op), [0, 1], margins, variant=ev)
    m, c, counts = ko.score_batch(d["kv"], d["ops"], variants, margins=margins, plans=[plan],
                                  gold=d["gold"])
    torch.cuda.synchronize()
    # the embedding stage at position 0 streams no KV: a walk-only launch decides every tuple from
    # the caller's margins and queues the survivors; then F1's gold position (prep, score, walk —
    # its fused read also completes F2's gold margin, so F2's position never receives a tuple and
    # is not launched) and the final counts
    assert ko.last_launch_count() == 1 + 3 + 1
    mg, cg = m.cpu().numpy(), c.cpu().numpy()
    m_or, c_or = oracle.score_workload(wl, np.arange(n))
    m_all = np.concatenate([m_or, emb[:, None, :]], axis=1)
    c_all = np.concatenate([c_or, np.zeros((2, 1, n), np.int32)], axis=1)
    gold = d["gold"].cpu().numpy()
    assert np.abs(mg[:, ev] - emb).max() < 1e-5                   # external margins untouched
    reached = np.isfinite(mg)
    parity.assert_margins(mg, m_all, mask=reached)
    parity.assert_counts(counts.cpu().numpy(), m_all, c_all, mg, cg, [plan], [1, 1], gold)
    # the cascade saves work: the gold variant is read only for tuples the embedding left unsure
    assert 0 < reached[0, 0].sum() < n
    # grid mode over the same variants (external margins supplied) gives the same counts
    margins2 = torch.empty((2, len(variants), n), device="cuda")
    ko.embed_scores(_dev_bits(item), _dev_bits(op), [0, 1], margins2, variant=ev)
    _, _, grid = ko.score_batch(d["kv"], d["ops"], variants, margins=margins2, plans=[plan, plan],
                                gold=d["gold"])
    torch.cuda.synchronize()
    assert np.array_equal(grid.cpu().numpy()[0], counts.cpu().numpy()[0])
