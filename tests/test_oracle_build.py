"""Pins of the importance-ordered cache builder oracle (NEXT-4, ko_oracle.cpp
oracle_build_order; Expected-Attention reading Q25)."""
import numpy as np

import oracle
from tests.helpers import Geom, bf16_bits, bf16_value, build_pool, grid_values, random_problem


def _rows(pool, indptr, ids, t, L, l, which, h):
    return np.stack([pool[ids[indptr[t] + i // 16], l, which, h, i % 16] for i in range(L)])


def _setup(seed=0, lengths=(37, 16, 1, 130), geom=Geom(2, 3, 1, 64, 1)):
    rng = np.random.default_rng(seed)
    K, V, _ = random_problem(rng, geom, list(lengths))
    pool, indptr, ids, sl = build_pool(K, V, list(lengths), placement="shuffle", seed=seed)
    return rng, geom, K, V, pool, indptr, ids, sl


def test_mean_direction_only_orders_by_projection():
    """σ² = 0, μ = e_0 ⇒ tokens in descending K[:, 0], ties by original index."""
    rng, geom, K, V, pool, indptr, ids, sl = _setup(1)
    mu = np.zeros((2, 3, 64), np.float32); mu[..., 0] = 1.0
    s2 = np.zeros_like(mu)
    dst_ids = rng.permutation(len(ids)).astype(np.int32)
    dst = oracle.build_order(geom, pool, indptr, ids, sl, mu, s2, dst_ids)
    for t, L in enumerate(sl):
        for l in range(2):
            for h in range(3):
                k0 = K[t][l, h, :L, 0].astype(np.float64)
                order = sorted(range(L), key=lambda i: (-k0[i], i))
                got_k = _rows(dst, indptr, dst_ids, t, L, l, 0, h)
                got_v = _rows(dst, indptr, dst_ids, t, L, l, 1, h)
                assert np.array_equal(got_k, bf16_bits(K[t][l, h, order]))
                assert np.array_equal(got_v, bf16_bits(V[t][l, h, order]))


def test_permutation_monotone_and_idempotent():
    rng, geom, K, V, pool, indptr, ids, sl = _setup(2)
    mu = (rng.integers(-8, 9, size=(2, 3, 64)) / 8).astype(np.float32)
    s2 = (rng.integers(0, 5, size=(2, 3, 64)) / 4).astype(np.float32)
    dst = oracle.build_order(geom, pool, indptr, ids, sl, mu, s2, ids)
    for t, L in enumerate(sl):
        for l in range(2):
            for h in range(3):
                src = _rows(pool, indptr, ids, t, L, l, 0, h)
                out = _rows(dst, indptr, ids, t, L, l, 0, h)
                # a permutation of the rows (K and V move together: same multiset of pairs)
                pairs_in = sorted(map(tuple, np.concatenate([src, _rows(pool, indptr, ids, t, L, l, 1, h)], 1)))
                pairs_out = sorted(map(tuple, np.concatenate([out, _rows(dst, indptr, ids, t, L, l, 1, h)], 1)))
                assert pairs_in == pairs_out
                # values on the 1/32 grid and μ, σ² on 1/8, 1/4 grids: exact scores, so the
                # expected-attention score is non-increasing along the stored order
                k = bf16_value(out)
                sc = (k @ mu[l, h].astype(np.float64)) / 8.0 + (k * k) @ s2[l, h].astype(np.float64) / 128.0
                assert np.all(np.diff(sc) <= 0)
    again = oracle.build_order(geom, dst, indptr, ids, sl, mu, s2, ids)
    assert np.array_equal(again, dst)                     # a built store is a fixed point


def test_keep_prefix_is_the_top_tokens():
    """Q2: after building, variant keep‰ attends exactly the n_kept tokens of highest expected
    attention — scoring the built store with keep k equals scoring the natural store restricted
    to those tokens (single kv-head, where the top set is one set of tokens)."""
    rng = np.random.default_rng(3)
    geom = Geom(1, 1, 2, 64, 1)
    L = 90
    K, V, ops = random_problem(rng, geom, [L])
    pool, indptr, ids, sl = build_pool(K, V, [L])
    mu = (rng.integers(-8, 9, size=(1, 1, 64)) / 8).astype(np.float32)
    s2 = (rng.integers(0, 5, size=(1, 1, 64)) / 4).astype(np.float32)
    built = oracle.build_order(geom, pool, indptr, ids, sl, mu, s2, ids)
    kf = K[0][0, 0].astype(np.float64)
    sc = kf @ mu[0, 0] / 8.0 + (kf * kf) @ s2[0, 0] / 128.0
    top_order = sorted(range(L), key=lambda i: (-sc[i], i))
    for keep in (500, 250, 999):
        n = max(1, L * keep // 1000)
        m_built, _ = oracle.score(geom, built, indptr, ids, sl, ops, [(keep, 1)])
        sel = sorted(top_order[:n])
        p2, i2, d2, s2_ = build_pool([K[0][:, :, sel]], [V[0][:, :, sel]], [n])
        m_ref, _ = oracle.score(geom, p2, i2, d2, s2_, ops, [(1000, 1)])
        assert abs(m_built[0, 0, 0] - m_ref[0, 0, 0]) < 1e-12
