"""oracle — plain fp64 CPU oracle of the KV-cache scoring → routing → count pass (TEST INFRA).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` / ``--impl reference``
legs may import this package.  It shares no code with the CUDA path; the C++ core is
``ko_oracle.cpp`` (see its header for the paper passages each step follows).

parity pinned: see tests/test_oracle_*.py (SDPA library routine, closed forms, invariants,
brute-force routing, paper worked examples, Beta closed forms).
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
MAX_STAGES = 8
COUNTS_PER_PLAN = 5 + 4 * MAX_STAGES


class OrKV(ctypes.Structure):
    _fields_ = [("n_layers", ctypes.c_int32), ("n_kv_heads", ctypes.c_int32),
                ("gqa", ctypes.c_int32), ("head_dim", ctypes.c_int32), ("n_q", ctypes.c_int32),
                ("kv_pool", ctypes.c_void_p), ("n_pages", ctypes.c_int64),
                ("page_indptr", ctypes.c_void_p), ("page_ids", ctypes.c_void_p),
                ("seq_len", ctypes.c_void_p), ("n_tuples", ctypes.c_int64)]


class OrOp(ctypes.Structure):
    _fields_ = [("n_classes", ctypes.c_int32), ("q", ctypes.c_void_p), ("w", ctypes.c_void_p),
                ("b", ctypes.c_void_p)]


class OrVariant(ctypes.Structure):
    _fields_ = [("keep_permille", ctypes.c_int32), ("layer_cut", ctypes.c_int32)]


class OrStage(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("variant", ctypes.c_int32), ("theta_lo", ctypes.c_float),
                ("theta_hi", ctypes.c_float), ("is_final", ctypes.c_int32)]


class OrPlan(ctypes.Structure):
    _fields_ = [("n_stages", ctypes.c_int32), ("stage", OrStage * MAX_STAGES)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"oracle: {_LIB_PATH} missing — run __graft_entry__.build()")
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        L.oracle_score.argtypes = [ctypes.POINTER(OrKV), P, ctypes.c_int32, P, ctypes.c_int32, P,
                                   ctypes.c_int64, P, P, P, ctypes.c_int32, ctypes.c_int32]
        L.oracle_score.restype = ctypes.c_int
        L.oracle_run_plans.argtypes = [P, ctypes.c_int32, P, P, P, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.c_int64, P, P, P, P]
        L.oracle_run_plans.restype = ctypes.c_int
        L.oracle_build_order.argtypes = [ctypes.POINTER(OrKV), P, P, P, P, ctypes.c_int32]
        L.oracle_build_order.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def make_plans(plans: Sequence[Sequence[Tuple]]) -> ctypes.Array:
    arr = (OrPlan * len(plans))()
    for g, pl in enumerate(plans):
        assert 1 <= len(pl) <= MAX_STAGES
        arr[g].n_stages = len(pl)
        for s, (op, var, lo, hi, fin) in enumerate(pl):
            arr[g].stage[s] = OrStage(op, var, lo, hi, fin)
    return arr


def score(geom, pool: np.ndarray, indptr: np.ndarray, page_ids: np.ndarray, seq_len: np.ndarray,
          ops: Sequence[dict], variants: Sequence[Tuple[int, int]],
          tuples: Optional[np.ndarray] = None, n_threads: int = 0, want_z: bool = False):
    """fp64 margins [n_ops][n_variants][n], classes (int32, same), z [.., n, Cmax] (optional).

    geom: object with n_layers, n_kv_heads, gqa, head_dim, n_q.  ops: dicts with n_classes,
    q (uint16 bf16 bits [Lyr][Hq][n_q][D]), w (fp32 [C][Lyr][Hq][n_q][D]), b (fp32 [C])."""
    pool = np.ascontiguousarray(pool, np.uint16)
    indptr = np.ascontiguousarray(indptr, np.int64)
    page_ids = np.ascontiguousarray(page_ids, np.int32)
    seq_len = np.ascontiguousarray(seq_len, np.int32)
    kv = OrKV(geom.n_layers, geom.n_kv_heads, geom.gqa, geom.head_dim, geom.n_q,
              pool.ctypes.data, pool.shape[0], indptr.ctypes.data, page_ids.ctypes.data,
              seq_len.ctypes.data, len(seq_len))
    keep = []
    ops_arr = (OrOp * len(ops))()
    for i, o in enumerate(ops):
        q = np.ascontiguousarray(o["q"], np.uint16)
        w = np.ascontiguousarray(o["w"], np.float32)
        b = np.ascontiguousarray(o["b"], np.float32)
        keep += [q, w, b]
        ops_arr[i] = OrOp(int(o["n_classes"]), q.ctypes.data, w.ctypes.data, b.ctypes.data)
    var_arr = (OrVariant * len(variants))(*[OrVariant(k, c) for k, c in variants])
    if tuples is None:
        n = len(seq_len)
        tarr = None
    else:
        tarr = np.ascontiguousarray(tuples, np.int64)
        n = len(tarr)
    margins = np.empty((len(ops), len(variants), n), np.float64)
    classes = np.empty((len(ops), len(variants), n), np.int32)
    cmax = max(int(o["n_classes"]) for o in ops)
    z = np.empty((len(ops), len(variants), n, cmax), np.float64) if want_z else None
    nt = n_threads or max(1, len(os.sched_getaffinity(0)))
    rc = lib().oracle_score(ctypes.byref(kv), ops_arr, len(ops), var_arr, len(variants),
                            _p(tarr), n, _p(margins), _p(classes), _p(z), cmax, nt)
    assert rc == 0
    if want_z:
        return margins, classes, z
    return margins, classes


STAGE_NOT_REACHED, STAGE_ACCEPT, STAGE_REJECT, STAGE_UNSURE, STAGE_RESOLVED = 0, 1, 2, 3, 4


def run_plans(plans: Sequence[Sequence[Tuple]], margins: np.ndarray, classes: np.ndarray,
              n_classes: Sequence[int], gold: Optional[np.ndarray] = None,
              want_alive: bool = False, want_stages: bool = False):
    """Counts int64 [n_plans][37] (TP, FP, FN, n_out, n_gold, per-stage n_in/acc/rej/uns).

    want_alive: also return alive uint8 [n_plans][n] (1 = tuple in P_o).
    want_stages: also return the per-tuple stage outcomes int8 [n_plans][MAX_STAGES][n]
    (STAGE_NOT_REACHED / ACCEPT / REJECT / UNSURE / RESOLVED; Eqs. accept-i / reject-i /
    unsure-i).  Returns counts, then alive, then stages, for the ones requested."""
    margins = np.ascontiguousarray(margins, np.float64)
    classes = np.ascontiguousarray(classes, np.int32)
    n_ops, n_var, n = margins.shape
    nc = np.ascontiguousarray(n_classes, np.int32)
    g = None if gold is None else np.ascontiguousarray(gold, np.uint8)
    counts = np.zeros((len(plans), COUNTS_PER_PLAN), np.int64)
    alive = np.zeros((len(plans), n), np.uint8) if want_alive else None
    stages = np.zeros((len(plans), MAX_STAGES, n), np.int8) if want_stages else None
    parr = make_plans(plans)
    rc = lib().oracle_run_plans(parr, len(plans), _p(margins), _p(classes), _p(nc), n_ops, n_var,
                                n, _p(g), _p(counts), _p(alive), _p(stages))
    if rc != 0:
        raise ValueError("oracle_run_plans: invalid plan")
    out = (counts,) + ((alive,) if want_alive else ()) + ((stages,) if want_stages else ())
    return out if len(out) > 1 else counts


def beta_lower_bound(a: int, b: int, alpha: float) -> float:
    """ℓ_α = I^{-1}(1 − α; 1 + a, 1 + b) (Eqs. recall/precision lower bound; Q7),
    by the library routine scipy.special.betaincinv."""
    from scipy.special import betaincinv
    return float(betaincinv(1.0 + a, 1.0 + b, 1.0 - alpha))


def workload_ops(wl, spec=None) -> List[dict]:
    """Host operator tensors of a kogen workload (Q, W from the generator, b from calibration)."""
    spec = spec or wl.spec
    bias = wl.biases()
    return [dict(n_classes=spec.op_classes[o], q=spec.q(o), w=spec.w(o),
                 b=np.asarray(bias[o], np.float32)) for o in range(spec.n_ops)]


def score_workload(wl, tuple_ids, n_threads: int = 0, variants=None, want_z=False):
    """Generate the host pool for tuple_ids (kogen) and score them with the oracle."""
    import kogen
    pool, indptr, ids, sl = kogen.host_pool(wl.spec, tuple_ids)
    ops = workload_ops(wl)
    return score(wl.spec, pool, indptr, ids, sl, ops, variants or wl.variants,
                 n_threads=n_threads, want_z=want_z)


def embed_scores(item_bits: np.ndarray, op_bits: np.ndarray) -> np.ndarray:
    """Embedding-similarity stage (NEXT-3): cosine similarity of every item
    embedding with every operator embedding, fp64, by definition: ⟨e, q⟩ / (‖e‖ ‖q‖) (0 if a norm
    is 0).  item_bits: bf16 bits [n][dim]; op_bits: bf16 bits [n_e][dim].  Returns [n_e][n]."""
    def f(b):
        return (np.asarray(b, np.uint32) << 16).view(np.float32).astype(np.float64)
    e, q = f(item_bits), f(op_bits)
    out = np.zeros((q.shape[0], e.shape[0]))
    ne = np.sqrt((e * e).sum(axis=1))
    for k in range(q.shape[0]):
        nq = np.sqrt((q[k] * q[k]).sum())
        dot = e @ q[k]
        den = ne * nq
        out[k] = np.where(den > 0, dot / np.where(den > 0, den, 1.0), 0.0)
    return out


def build_order(geom, pool, indptr, page_ids, seq_len, mu, sigma2, dst_page_ids,
                n_threads: int = 0) -> np.ndarray:
    """Offline importance-ordered cache builder (NEXT-4, see ko_oracle.cpp): returns a new pool
    (uint16 bf16 bits, same shape) whose pages dst_page_ids (same CSR indptr) hold each tuple's
    tokens in descending expected-attention score per (layer, kv-head)."""
    pool = np.ascontiguousarray(pool, np.uint16)
    indptr = np.ascontiguousarray(indptr, np.int64)
    page_ids = np.ascontiguousarray(page_ids, np.int32)
    seq_len = np.ascontiguousarray(seq_len, np.int32)
    mu = np.ascontiguousarray(mu, np.float32)
    sigma2 = np.ascontiguousarray(sigma2, np.float32)
    dst_ids = np.ascontiguousarray(dst_page_ids, np.int32)
    kv = OrKV(geom.n_layers, geom.n_kv_heads, geom.gqa, geom.head_dim, geom.n_q,
              pool.ctypes.data, pool.shape[0], indptr.ctypes.data, page_ids.ctypes.data,
              seq_len.ctypes.data, len(seq_len))
    dst = np.zeros_like(pool)
    nt = n_threads or max(1, len(os.sched_getaffinity(0)))
    rc = lib().oracle_build_order(ctypes.byref(kv), _p(mu), _p(sigma2), _p(dst), _p(dst_ids), nt)
    assert rc == 0
    return dst
