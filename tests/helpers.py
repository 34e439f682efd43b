"""Test-only helpers: build small paged KV stores from logical tensors, bf16 bit conversions."""
from __future__ import annotations

import numpy as np

PAGE = 16


class Geom:
    def __init__(self, n_layers, n_kv_heads, gqa, head_dim, n_q):
        self.n_layers, self.n_kv_heads, self.gqa = n_layers, n_kv_heads, gqa
        self.head_dim, self.n_q = head_dim, n_q

    @property
    def n_q_heads(self):
        return self.n_kv_heads * self.gqa


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """float32 values that are exactly representable in bf16 → uint16 bits (asserts exactness)."""
    f = np.ascontiguousarray(x, np.float32)
    u = f.view(np.uint32)
    assert np.all((u & 0xFFFF) == 0), "value not exactly representable in bf16"
    return (u >> 16).astype(np.uint16)


def bf16_value(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, np.uint32) << 16).view(np.float32).astype(np.float64)


def grid_values(rng, shape, lim=127):
    """random values on the 1/32 grid in [-lim/32, lim/32] (exact in bf16)."""
    return rng.integers(-lim, lim + 1, size=shape).astype(np.float32) / 32.0


def build_pool(K, V, lengths, placement="shuffle", seed=0, poison=False):
    """K, V: lists (per tuple) of float32 arrays [Lyr][Hkv][L_t][D] (bf16-exact).
    Returns pool (uint16 [n_pages][Lyr][2][Hkv][16][D]), indptr, page_ids, seq_len."""
    n = len(lengths)
    Lyr, H, _, D = K[0].shape
    pages = [(int(L) + PAGE - 1) // PAGE for L in lengths]
    indptr = np.zeros(n + 1, np.int64)
    indptr[1:] = np.cumsum(pages)
    nnz = int(indptr[-1])
    ids = np.arange(nnz, dtype=np.int64)
    if placement == "shuffle":
        ids = np.random.default_rng(seed).permutation(nnz)
    elif placement == "reverse":
        ids = ids[::-1].copy()
    fill = 0x7FC0 if poison else 0
    pool = np.full((max(nnz, 1), Lyr, 2, H, PAGE, D), fill, np.uint16)
    for t in range(n):
        L = int(lengths[t])
        kb, vb = bf16_bits(K[t][:, :, :L]), bf16_bits(V[t][:, :, :L])
        for i in range(L):
            p = ids[indptr[t] + i // PAGE]
            pool[p, :, 0, :, i % PAGE, :] = kb[:, :, i, :]
            pool[p, :, 1, :, i % PAGE, :] = vb[:, :, i, :]
    return pool, indptr, ids.astype(np.int32), np.asarray(lengths, np.int32)


def random_problem(rng, geom, lengths, n_ops=1, classes=(1,), w_scale=1 / 64.0):
    """Random bf16-exact K/V per tuple plus operators (Q bf16 bits, W fp32, b fp32)."""
    K = [grid_values(rng, (geom.n_layers, geom.n_kv_heads, L, geom.head_dim)) for L in lengths]
    V = [grid_values(rng, (geom.n_layers, geom.n_kv_heads, L, geom.head_dim)) for L in lengths]
    ops = []
    for o in range(n_ops):
        C = classes[o]
        q = grid_values(rng, (geom.n_layers, geom.n_q_heads, geom.n_q, geom.head_dim), 40)
        w = (rng.integers(-100, 101, size=(C, geom.n_layers, geom.n_q_heads, geom.n_q,
                                          geom.head_dim)) * w_scale / 16).astype(np.float32)
        b = (rng.integers(-64, 65, size=C) / 64.0).astype(np.float32)
        ops.append(dict(n_classes=C, q=bf16_bits(q), w=w, b=b, qf=q))
    return K, V, ops
