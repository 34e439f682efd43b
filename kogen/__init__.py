"""kogen — seeded synthetic workload generator (FIXTURE shared by the oracle and the CUDA path).

Holds none of the method's arithmetic: it only produces inputs (bf16 KV pages, operator queries
Q, readouts W, lengths, latent labels) from the integer-only recipe in ``kogen.h`` (SURVEY.md
§8(d), restated in DESIGN.md §"Input recipe").  The host fill feeds ``oracle/``; the device
fill feeds ``paper_2602_04430_b200``; tests check the two fills are bit-identical.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libkogen.so")
PAGE = 16
MAX_OPS = 4


class KgCfg(ctypes.Structure):
    _fields_ = [
        ("seed", ctypes.c_uint64),
        ("n_layers", ctypes.c_int32),
        ("n_kv_heads", ctypes.c_int32),
        ("gqa", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("n_q", ctypes.c_int32),
        ("n_ops", ctypes.c_int32),
        ("op_classes", ctypes.c_int32 * MAX_OPS),
        ("op_pi_permille", ctypes.c_int32 * MAX_OPS),
        ("len_min", ctypes.c_int32),
        ("len_max", ctypes.c_int32),
        ("n_evid", ctypes.c_int32),
        ("k_ramp", ctypes.c_int32),
        ("k_beta", ctypes.c_int32),
        ("v_gamma", ctypes.c_int32),
        ("w_log2_den", ctypes.c_int32),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"kogen: {_LIB_PATH} missing — run __graft_entry__.build()")
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        L.kg_fill_q.argtypes = [ctypes.POINTER(KgCfg), ctypes.c_int32, P]
        L.kg_fill_w.argtypes = [ctypes.POINTER(KgCfg), ctypes.c_int32, P]
        L.kg_fill_meta.argtypes = [ctypes.POINTER(KgCfg), ctypes.c_int64, ctypes.c_int64, P, P]
        L.kg_fill_evidence.argtypes = [ctypes.POINTER(KgCfg), ctypes.c_int64, ctypes.c_int64, P]
        L.kg_fill_embeddings.argtypes = [ctypes.POINTER(KgCfg), ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_int32, ctypes.c_int32, P, P, ctypes.c_int32]
        L.kg_fill_pool_host.argtypes = [ctypes.POINTER(KgCfg), P, ctypes.c_int64, P, P, P,
                                        ctypes.c_int32, ctypes.c_int32]
        L.kg_fill_pool_host.restype = ctypes.c_int
        L.kg_fill_pool_device.argtypes = [ctypes.POINTER(KgCfg), ctypes.c_int64, ctypes.c_int64,
                                          P, P, P, ctypes.c_int32, P]
        L.kg_fill_pool_device.restype = ctypes.c_int
        L.kg_read_stream.argtypes = [P, ctypes.c_int64, P, P]
        L.kg_read_stream.restype = ctypes.c_int
        L.kg_gather_stream.argtypes = [P, ctypes.c_int32, P, ctypes.c_int64, P, P]
        L.kg_gather_stream.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


@dataclass
class GenSpec:
    """Geometry + recipe parameters of one synthetic workload."""
    seed: int
    n_layers: int
    n_kv_heads: int
    gqa: int
    head_dim: int
    n_q: int
    op_classes: Sequence[int]              # 1 = filter, K = map-classify
    op_pi_permille: Sequence[int] = ()     # filters: P(label = +1)
    len_min: int = 128
    len_max: int = 128
    n_evid: int = 3
    k_ramp: int = 8
    k_beta: int = 16
    v_gamma: int = 10
    w_log2_den: int = 12

    @property
    def n_ops(self) -> int:
        return len(self.op_classes)

    @property
    def n_q_heads(self) -> int:
        return self.n_kv_heads * self.gqa

    def cfg(self) -> KgCfg:
        c = KgCfg()
        c.seed = self.seed
        c.n_layers, c.n_kv_heads, c.gqa = self.n_layers, self.n_kv_heads, self.gqa
        c.head_dim, c.n_q, c.n_ops = self.head_dim, self.n_q, self.n_ops
        pis = list(self.op_pi_permille) + [500] * MAX_OPS
        for o in range(MAX_OPS):
            c.op_classes[o] = self.op_classes[o] if o < self.n_ops else 1
            c.op_pi_permille[o] = pis[o]
        c.len_min, c.len_max = self.len_min, self.len_max
        c.n_evid, c.k_ramp, c.k_beta, c.v_gamma = self.n_evid, self.k_ramp, self.k_beta, self.v_gamma
        c.w_log2_den = self.w_log2_den
        return c

    # ---- small host tensors ---------------------------------------------------------------
    def q(self, o: int) -> np.ndarray:
        """bf16 bits [n_layers][Hq][n_q][head_dim] (uint16)."""
        out = np.empty((self.n_layers, self.n_q_heads, self.n_q, self.head_dim), np.uint16)
        c = self.cfg()
        lib().kg_fill_q(ctypes.byref(c), o, _ptr(out))
        return out

    def w(self, o: int) -> np.ndarray:
        """fp32 [n_classes][n_layers][Hq][n_q][head_dim]."""
        C = self.op_classes[o]
        out = np.empty((C, self.n_layers, self.n_q_heads, self.n_q, self.head_dim), np.float32)
        c = self.cfg()
        lib().kg_fill_w(ctypes.byref(c), o, _ptr(out))
        return out

    def seq_len(self, t0: int, n: int) -> np.ndarray:
        out = np.empty(n, np.int32)
        c = self.cfg()
        lib().kg_fill_meta(ctypes.byref(c), t0, n, _ptr(out), None)
        return out

    def labels(self, t0: int, n: int) -> np.ndarray:
        """latent labels [n_ops][n]: filters ±1, maps class."""
        out = np.empty((self.n_ops, n), np.int32)
        c = self.cfg()
        lib().kg_fill_meta(ctypes.byref(c), t0, n, None, _ptr(out))
        return out

    def evidence(self, t0: int, n: int) -> np.ndarray:
        out = np.empty((n, self.n_ops, self.n_evid), np.int32)
        c = self.cfg()
        lib().kg_fill_evidence(ctypes.byref(c), t0, n, _ptr(out))
        return out

    def embeddings(self, t0: int, n: int, dim: int = 256, gamma: int = 2):
        """(item bf16 bits [n][dim], op bf16 bits [n_ops][dim]) for the embedding stage."""
        item = np.empty((n, dim), np.uint16)
        op = np.empty((self.n_ops, dim), np.uint16)
        c = self.cfg()
        lib().kg_fill_embeddings(ctypes.byref(c), t0, n, dim, gamma, _ptr(item), _ptr(op),
                                 max(1, min(16, os.cpu_count() or 1)))
        return item, op

    def page_elems(self) -> int:
        return self.n_layers * 2 * self.n_kv_heads * PAGE * self.head_dim

    def page_bytes(self) -> int:
        return 2 * self.page_elems()


def page_table(seq_len: np.ndarray, placement: str = "affine", salt: int = 0
               ) -> Tuple[np.ndarray, np.ndarray]:
    """CSR page table for tuples with the given lengths: indptr int64 [n+1] (from 0) and
    physical page ids int32 [nnz].  placement 'contiguous' = identity, 'affine' = the bijection
    p -> (a·p + salt) mod nnz (a odd and coprime to nnz), so pages of a tuple are scattered."""
    pages = (seq_len.astype(np.int64) + PAGE - 1) // PAGE
    indptr = np.zeros(len(seq_len) + 1, np.int64)
    np.cumsum(pages, out=indptr[1:])
    nnz = int(indptr[-1])
    p = np.arange(nnz, dtype=np.int64)
    if placement == "contiguous" or nnz <= 1:
        ids = p
    else:
        a = 7919
        while math.gcd(a, nnz) != 1:
            a += 2
        ids = (a * p + salt) % nnz
    return indptr, ids.astype(np.int32)


def host_pool(spec: GenSpec, tuple_ids: Sequence[int], placement: str = "affine",
              poison: bool = False, n_threads: int = 0):
    """Generate a compact host pool for the given tuples.  Returns (pool uint16
    [n_pages][Lyr][2][Hkv][16][D], indptr, page_ids, seq_len) with a LOCAL CSR (row i = tuple
    tuple_ids[i])."""
    tids = np.ascontiguousarray(np.asarray(tuple_ids, dtype=np.int64))
    sl = np.array([spec.seq_len(int(t), 1)[0] for t in tids], np.int32) if len(tids) < 64 else \
        _seq_len_gather(spec, tids)
    indptr, ids = page_table(sl, placement)
    n_pages = int(indptr[-1])
    pool = np.zeros((max(n_pages, 1), spec.n_layers, 2, spec.n_kv_heads, PAGE, spec.head_dim),
                    np.uint16)
    c = spec.cfg()
    nt = n_threads or max(1, min(16, os.cpu_count() or 1))
    rc = lib().kg_fill_pool_host(ctypes.byref(c), _ptr(tids), len(tids), _ptr(indptr), _ptr(ids),
                                 _ptr(pool), int(poison), nt)
    assert rc == 0
    return pool, indptr, ids, sl


def _seq_len_gather(spec: GenSpec, tids: np.ndarray) -> np.ndarray:
    if spec.len_min == spec.len_max:
        return np.full(len(tids), spec.len_min, np.int32)
    lo, hi = int(tids.min()), int(tids.max())
    if hi - lo < 4 * len(tids) + 1024:
        allv = spec.seq_len(lo, hi - lo + 1)
        return allv[tids - lo]
    return np.array([spec.seq_len(int(t), 1)[0] for t in tids], np.int32)


def fill_device_pool(spec: GenSpec, t_begin: int, n_tuples: int, d_indptr: int, d_page_ids: int,
                     d_pool: int, stream: int = 0, poison: bool = True) -> None:
    """Device twin: fill pages of tuples t_begin.. t_begin+n_tuples-1 (device CSR pointers)."""
    c = spec.cfg()
    rc = lib().kg_fill_pool_device(ctypes.byref(c), t_begin, n_tuples, ctypes.c_void_p(d_indptr),
                                   ctypes.c_void_p(d_page_ids), ctypes.c_void_p(d_pool),
                                   int(poison), ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(f"kg_fill_pool_device failed rc={rc}")


def read_stream(d_buf: int, nbytes: int, d_sink: int, stream: int = 0) -> None:
    """Measurement helper (bench.py): one read-only pass over nbytes of a device buffer."""
    if lib().kg_read_stream(ctypes.c_void_p(d_buf), int(nbytes), ctypes.c_void_p(d_sink),
                            ctypes.c_void_p(stream)) != 0:
        raise RuntimeError("kg_read_stream failed")


def gather_stream(d_base: int, row_bytes: int, d_idx: int, n: int, d_sink: int,
                  stream: int = 0) -> None:
    """Measurement helper (bench.py): one read of rows idx[0..n) of a device buffer (the
    gathered-read ceiling of the embedding stage's tuple_idx path)."""
    if lib().kg_gather_stream(ctypes.c_void_p(d_base), int(row_bytes), ctypes.c_void_p(d_idx),
                              int(n), ctypes.c_void_p(d_sink), ctypes.c_void_p(stream)) != 0:
        raise RuntimeError("kg_gather_stream failed")
