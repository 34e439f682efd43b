"""Pins of the oracle's scoring (SURVEY §8(c) steps 1–4) to things other than itself:
a library routine (torch fp64 scaled_dot_product_attention with enable_gqa), closed forms,
and invariants.  CPU only."""
import numpy as np
import pytest
import torch

import oracle
from tests.helpers import Geom, bf16_bits, bf16_value, build_pool, grid_values, random_problem


def sdpa_reference(geom, K, V, ops, variants, lengths):
    """z via torch fp64 SDPA (library routine; GQA by the library's own enable_gqa mapping)
    and a numpy readout.  Returns margins/classes/z like oracle.score."""
    n = len(lengths)
    n_ops, n_var = len(ops), len(variants)
    cmax = max(o["n_classes"] for o in ops)
    z = np.zeros((n_ops, n_var, n, cmax))
    for t in range(n):
        for o, op in enumerate(ops):
            q = torch.tensor(bf16_value(op["q"]))          # [Lyr][Hq][n_q][D]
            for v, (keep, cut) in enumerate(variants):
                nk = max(1, (int(lengths[t]) * keep) // 1000)
                zz = op["b"].astype(np.float64).copy()
                for l in range(cut):
                    k = torch.tensor(K[t][l, :, :nk, :], dtype=torch.float64)   # [Hkv][n][D]
                    vv = torch.tensor(V[t][l, :, :nk, :], dtype=torch.float64)
                    O = torch.nn.functional.scaled_dot_product_attention(
                        q[l][None], k[None], vv[None], enable_gqa=True)[0]     # [Hq][n_q][D]
                    w = op["w"][:, l].astype(np.float64)                       # [C][Hq][n_q][D]
                    zz += np.einsum("cjrd,jrd->c", w, O.numpy())
                z[o, v, t, :len(zz)] = zz
    return z


def _margins_from_z(z, ops):
    m = np.zeros(z.shape[:3]); cls = np.zeros(z.shape[:3], np.int32)
    for o, op in enumerate(ops):
        C = op["n_classes"]
        zz = z[o, :, :, :C]
        if C == 1:
            m[o] = zz[..., 0]
        else:
            a = np.argmax(zz, axis=-1)     # numpy argmax returns the lowest index on ties
            srt = np.sort(zz, axis=-1)
            m[o] = srt[..., -1] - srt[..., -2]
            cls[o] = a
    return m, cls


@pytest.mark.parametrize("G,n_q,D", [(1, 1, 64), (2, 2, 64), (4, 1, 128)])
def test_oracle_matches_torch_sdpa(G, n_q, D):
    rng = np.random.default_rng(10 + G + D)
    geom = Geom(n_layers=2, n_kv_heads=2, gqa=G, head_dim=D, n_q=n_q)
    lengths = [1, 13, 16, 37]            # single token, partial page, exact page, ragged tail
    K, V, ops = random_problem(rng, geom, lengths, n_ops=2, classes=(1, 3))
    variants = [(1000, 2), (500, 1), (250, 2), (1, 1)]
    pool, indptr, ids, sl = build_pool(K, V, lengths, poison=True)
    m, cls, z = oracle.score(geom, pool, indptr, ids, sl, ops, variants, n_threads=2, want_z=True)
    zr = sdpa_reference(geom, K, V, ops, variants, lengths)
    for o, op in enumerate(ops):
        C = op["n_classes"]
        np.testing.assert_allclose(z[o, :, :, :C], zr[o, :, :, :C], rtol=0, atol=1e-12)
    mr, cr = _margins_from_z(zr, ops)
    np.testing.assert_allclose(m, mr, rtol=0, atol=1e-12)
    assert np.array_equal(cls[1], cr[1])


def test_single_token_closed_form():
    """L_t = 1 ⇒ softmax is 1 on the only token: O = V_0 and z = b + Σ W·V_0 (exact)."""
    rng = np.random.default_rng(1)
    geom = Geom(2, 2, 2, 64, 1)
    K, V, ops = random_problem(rng, geom, [1], n_ops=1)
    pool, indptr, ids, sl = build_pool(K, V, [1])
    m, _ = oracle.score(geom, pool, indptr, ids, sl, ops, [(1000, 2)])
    w = ops[0]["w"].astype(np.float64)[0]          # [Lyr][Hq][1][D]
    expect = float(ops[0]["b"][0])
    for l in range(2):
        for j in range(4):
            expect += float(np.dot(w[l, j, 0], V[0][l, j // 2, 0].astype(np.float64)))
    assert abs(m[0, 0, 0] - expect) < 1e-13


def test_zero_query_is_mean_of_values():
    """Q = 0 ⇒ all scores equal ⇒ O = mean of the kept V rows (closed form)."""
    rng = np.random.default_rng(2)
    geom = Geom(1, 1, 1, 64, 1)
    L = 45
    K, V, ops = random_problem(rng, geom, [L])
    ops[0]["q"] = np.zeros_like(ops[0]["q"])
    pool, indptr, ids, sl = build_pool(K, V, [L])
    for keep in (1000, 300):
        n = max(1, L * keep // 1000)
        m, _ = oracle.score(geom, pool, indptr, ids, sl, ops, [(keep, 1)])
        O = V[0][0, 0, :n].astype(np.float64).mean(axis=0)
        expect = float(ops[0]["b"][0]) + float(np.dot(ops[0]["w"][0, 0, 0, 0].astype(np.float64), O))
        assert abs(m[0, 0, 0] - expect) < 1e-12


def test_dominant_key_selects_its_value():
    """One key with a score gap ≥ 60 over all others ⇒ O = V_{i*} to ~e^-60."""
    geom = Geom(1, 1, 1, 64, 1)
    L = 20
    K = [np.zeros((1, 1, L, 64), np.float32)]
    rng = np.random.default_rng(3)
    V = [grid_values(rng, (1, 1, L, 64))]
    istar = 13
    K[0][0, 0, istar, :] = 2.0                      # q·k = 64·2·(127/32)/8 ≈ 63.5 after scaling
    q = np.full((1, 1, 1, 64), 127 / 32, np.float32)
    w = (rng.integers(-50, 51, size=(1, 1, 1, 1, 64)) / 256).astype(np.float32)
    ops = [dict(n_classes=1, q=bf16_bits(q), w=w, b=np.zeros(1, np.float32))]
    pool, indptr, ids, sl = build_pool(K, V, [L])
    m, _ = oracle.score(geom, pool, indptr, ids, sl, ops, [(1000, 1)])
    expect = float(np.dot(w[0, 0, 0, 0].astype(np.float64), V[0][0, 0, istar].astype(np.float64)))
    # other keys weigh ≤ 19·e^-63.5 ≈ 5e-27 relative: below fp64 resolution of O
    assert abs(m[0, 0, 0] - expect) < 1e-14


def test_keep_is_a_prefix_and_full_keep_is_full_attention():
    """Variant keep‰ ≡ full attention over the truncated store of n_kept tokens (Q2, Q3)."""
    rng = np.random.default_rng(4)
    geom = Geom(2, 2, 2, 64, 1)
    L = 50
    K, V, ops = random_problem(rng, geom, [L])
    pool, indptr, ids, sl = build_pool(K, V, [L])
    for keep in (999, 500, 333, 10, 1):
        n = max(1, L * keep // 1000)
        m, _ = oracle.score(geom, pool, indptr, ids, sl, ops, [(keep, 2)])
        p2, i2, d2, s2 = build_pool([K[0][:, :, :n]], [V[0][:, :, :n]], [n])
        mf, _ = oracle.score(geom, p2, i2, d2, s2, ops, [(1000, 2)])
        assert m[0, 0, 0] == mf[0, 0, 0]


def test_layer_additivity():
    """z(cut=2) − z(cut=1) is exactly the layer-1 term: equals z with layer-0 readout zeroed."""
    rng = np.random.default_rng(5)
    geom = Geom(2, 2, 2, 64, 2)
    K, V, ops = random_problem(rng, geom, [40, 23])
    pool, indptr, ids, sl = build_pool(K, V, [40, 23])
    m, _ = oracle.score(geom, pool, indptr, ids, sl, ops, [(1000, 2), (1000, 1)])
    ops0 = [dict(ops[0])]
    ops0[0]["w"] = ops[0]["w"].copy(); ops0[0]["w"][:, 0] = 0
    ops0[0]["b"] = np.zeros(1, np.float32)
    m1, _ = oracle.score(geom, pool, indptr, ids, sl, ops0, [(1000, 2)])
    np.testing.assert_allclose(m[0, 0] - m[0, 1], m1[0, 0], rtol=0, atol=1e-12)


def test_token_permutation_and_page_placement():
    """Attention is permutation-invariant over the kept keys; physical placement is irrelevant."""
    rng = np.random.default_rng(6)
    geom = Geom(1, 2, 2, 64, 1)
    L = 48
    K, V, ops = random_problem(rng, geom, [L])
    pool, indptr, ids, sl = build_pool(K, V, [L], placement="shuffle", seed=1)
    m, _ = oracle.score(geom, pool, indptr, ids, sl, ops, [(1000, 1)])
    perm = rng.permutation(L)
    p2, i2, d2, s2 = build_pool([K[0][:, :, perm]], [V[0][:, :, perm]], [L], placement="reverse")
    mp, _ = oracle.score(geom, p2, i2, d2, s2, ops, [(1000, 1)])
    assert abs(m[0, 0, 0] - mp[0, 0, 0]) < 1e-12
    p3, i3, d3, s3 = build_pool(K, V, [L], placement="reverse")
    m3, _ = oracle.score(geom, p3, i3, d3, s3, ops, [(1000, 1)])
    assert m3[0, 0, 0] == m[0, 0, 0]


def test_gqa_group_equals_mha_on_repeated_kv():
    """G > 1 ≡ MHA over repeat_kv-expanded K/V (Q18)."""
    rng = np.random.default_rng(7)
    g4 = Geom(1, 2, 4, 64, 1)
    K, V, ops = random_problem(rng, g4, [30])
    pool, indptr, ids, sl = build_pool(K, V, [30])
    m, _ = oracle.score(g4, pool, indptr, ids, sl, ops, [(1000, 1)])
    g1 = Geom(1, 8, 1, 64, 1)
    Kx = [np.repeat(K[0], 4, axis=1)]
    Vx = [np.repeat(V[0], 4, axis=1)]
    p2, i2, d2, s2 = build_pool(Kx, Vx, [30])
    m1, _ = oracle.score(g1, p2, i2, d2, s2, ops, [(1000, 1)])
    assert abs(m[0, 0, 0] - m1[0, 0, 0]) < 1e-12


def test_map_margin_argmax_ties_lowest():
    """Map: class = argmax (lowest index on ties), m = top1 − top2; tie ⇒ m = 0 and class 0."""
    geom = Geom(1, 1, 1, 64, 1)
    rng = np.random.default_rng(8)
    K, V, _ = random_problem(rng, geom, [5])
    w = np.zeros((3, 1, 1, 1, 64), np.float32)
    ops = [dict(n_classes=3, q=bf16_bits(np.zeros((1, 1, 1, 64), np.float32)), w=w,
                b=np.array([0.5, 0.5, -1.0], np.float32))]
    pool, indptr, ids, sl = build_pool(K, V, [5])
    m, cls = oracle.score(geom, pool, indptr, ids, sl, ops, [(1000, 1)])
    assert cls[0, 0, 0] == 0 and m[0, 0, 0] == 0.0
    ops[0]["b"] = np.array([0.25, 1.0, 0.75], np.float32)
    m, cls = oracle.score(geom, pool, indptr, ids, sl, ops, [(1000, 1)])
    assert cls[0, 0, 0] == 1 and m[0, 0, 0] == 0.25
