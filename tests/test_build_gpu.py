"""GPU parity of the importance-ordered cache builder (NEXT-4) against the oracle: bit-exact
bytes of every valid slot (integer/byte work), on ragged lengths incl. 1 and 4096 tokens."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import kogen  # noqa: E402
import oracle  # noqa: E402
from kogen import workloads  # noqa: E402
from kogen.device import tensors_to_device  # noqa: E402
from tests.helpers import Geom, build_pool, random_problem  # noqa: E402


@pytest.fixture(scope="module")
def ko():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2602_04430_b200 as ko
    return ko


def _valid_slots_equal(a, b, indptr, ids, sl):
    for t, L in enumerate(sl):
        for i in range(L):
            p = ids[indptr[t] + i // 16]
            if not np.array_equal(a[p, :, :, :, i % 16], b[p, :, :, :, i % 16]):
                return False
    return True


@pytest.mark.parametrize("D", [64, 128])
def test_build_matches_oracle(ko, D):
    rng = np.random.default_rng(D)
    geom = Geom(2, 2, 1, D, 1)
    lengths = [1, 15, 16, 17, 300, 1024, 1025, 2049, 4096]   # both launches, their boundary
    K, V, _ = random_problem(rng, geom, lengths)
    pool, indptr, ids, sl = build_pool(K, V, lengths, placement="shuffle", seed=1, poison=True)
    mu = rng.normal(0, 1, size=(2, 2, D)).astype(np.float32)
    s2 = rng.uniform(0, 2, size=(2, 2, D)).astype(np.float32)
    dst_ids = np.random.default_rng(2).permutation(len(ids)).astype(np.int32)
    exp = oracle.build_order(geom, pool, indptr, ids, sl, mu, s2, dst_ids)
    kv, _ = tensors_to_device(pool, indptr, ids, sl, geom,
                              [dict(n_classes=1, q=np.zeros((2, 2, 1, D), np.uint16),
                                    w=np.zeros((1, 2, 2, 1, D), np.float32),
                                    b=np.zeros(1, np.float32))])
    dst = torch.zeros_like(kv.pool)
    ko.build_importance_order(kv, torch.from_numpy(mu).cuda(), torch.from_numpy(s2).cuda(), dst,
                              torch.from_numpy(dst_ids).cuda())
    assert ko.last_launch_count() == 2                    # short- and long-tuple kernels
    torch.cuda.synchronize()
    got = dst.view(torch.int16).cpu().numpy().view(np.uint16)
    assert _valid_slots_equal(got, exp, indptr, dst_ids, sl)


def test_build_on_generated_workload(ko):
    """Builder on a generator store (natural order = the generator's ramp order) vs oracle."""
    wl = workloads.get("C5")
    tids = np.arange(40)
    pool, indptr, ids, sl = kogen.host_pool(wl.spec, tids)
    rng = np.random.default_rng(5)
    mu = rng.normal(0, 0.5, size=(2, 8, 128)).astype(np.float32)
    s2 = rng.uniform(0, 1, size=(2, 8, 128)).astype(np.float32)
    exp = oracle.build_order(wl.spec, pool, indptr, ids, sl, mu, s2, ids)
    kv, _ = tensors_to_device(pool, indptr, ids, sl, wl.spec, oracle.workload_ops(wl))
    dst = torch.zeros_like(kv.pool)
    ko.build_importance_order(kv, torch.from_numpy(mu).cuda(), torch.from_numpy(s2).cuda(), dst,
                              kv.page_ids)
    torch.cuda.synchronize()
    got = dst.view(torch.int16).cpu().numpy().view(np.uint16)
    assert _valid_slots_equal(got, exp, indptr, ids, sl)


def test_build_ties_keep_source_order(ko):
    """mu = sigma2 = 0: every score ties, so (ties: lower source index first, ko.h) the built
    store is the source order — exercises every tie-break branch of the register and shared
    memory sort phases; plus duplicated rows mixed with distinct ones, vs the oracle."""
    rng = np.random.default_rng(11)
    geom = Geom(1, 2, 1, 64, 1)
    lengths = [5, 64, 65, 700, 1500]
    K, V, _ = random_problem(rng, geom, lengths)
    for t in range(len(lengths)):                  # duplicate rows: equal scores, distinct tokens
        K[t][..., 1::3, :] = K[t][..., :1, :]
    pool, indptr, ids, sl = build_pool(K, V, lengths, placement="shuffle", seed=4, poison=True)
    kv, _ = tensors_to_device(pool, indptr, ids, sl, geom,
                              [dict(n_classes=1, q=np.zeros((1, 2, 1, 64), np.uint16),
                                    w=np.zeros((1, 1, 2, 1, 64), np.float32),
                                    b=np.zeros(1, np.float32))])
    for mu_scale in (0.0, 1.0):
        mu = (mu_scale * rng.normal(0, 1, size=(1, 2, 64))).astype(np.float32)
        s2 = (mu_scale * rng.uniform(0, 1, size=(1, 2, 64))).astype(np.float32)
        exp = oracle.build_order(geom, pool, indptr, ids, sl, mu, s2, ids)
        if mu_scale == 0.0:
            assert _valid_slots_equal(exp, pool, indptr, ids, sl)   # identity order
        dst = torch.zeros_like(kv.pool)
        ko.build_importance_order(kv, torch.from_numpy(mu).cuda(), torch.from_numpy(s2).cuda(),
                                  dst, kv.page_ids)
        torch.cuda.synchronize()
        got = dst.view(torch.int16).cpu().numpy().view(np.uint16)
        assert _valid_slots_equal(got, exp, indptr, ids, sl)


def test_build_rank_path_every_segment_count(ko):
    """The short-tuple kernel ranks by merging sorted 64-token segments (1 … 16 segments): every
    segment count and the lengths around each 64-token boundary and each page boundary, with
    duplicated rows (equal scores across segments) mixed in, vs the oracle."""
    rng = np.random.default_rng(23)
    geom = Geom(1, 2, 1, 128, 1)
    lengths = [2, 31, 63, 64, 65, 127, 128, 129, 191, 255, 256, 257, 383, 511, 512, 513, 639,
               767, 768, 895, 1000, 1023, 1024]
    K, V, _ = random_problem(rng, geom, lengths)
    for t in range(len(lengths)):                  # ties that straddle segments
        K[t][..., 7::5, :] = K[t][..., :1, :]
    pool, indptr, ids, sl = build_pool(K, V, lengths, placement="shuffle", seed=9, poison=True)
    mu = rng.normal(0, 1, size=(1, 2, 128)).astype(np.float32)
    s2 = rng.uniform(0, 1, size=(1, 2, 128)).astype(np.float32)
    dst_ids = np.random.default_rng(3).permutation(len(ids)).astype(np.int32)
    exp = oracle.build_order(geom, pool, indptr, ids, sl, mu, s2, dst_ids)
    kv, _ = tensors_to_device(pool, indptr, ids, sl, geom,
                              [dict(n_classes=1, q=np.zeros((1, 2, 1, 128), np.uint16),
                                    w=np.zeros((1, 1, 2, 1, 128), np.float32),
                                    b=np.zeros(1, np.float32))])
    dst = torch.zeros_like(kv.pool)
    ko.build_importance_order(kv, torch.from_numpy(mu).cuda(), torch.from_numpy(s2).cuda(), dst,
                              torch.from_numpy(dst_ids).cuda())
    torch.cuda.synchronize()
    got = dst.view(torch.int16).cpu().numpy().view(np.uint16)
    assert _valid_slots_equal(got, exp, indptr, dst_ids, sl)
