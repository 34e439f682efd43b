"""paper_2602_04430_b200 — thin Python binding of libko.so (include/ko.h).

Argument marshalling only: every step of the scoring → routing → count pass runs in the sm_100a
kernels of ``csrc/``.  torch supplies device memory and streams; there is no CPU fallback — if
``lib/libko.so`` is missing, importing this package raises.

Names mirror the C ABI: ``score_batch`` ↔ ``ko_score_batch``, ``route`` ↔ ``ko_route``,
``reduce_stats`` ↔ ``ko_reduce_stats``, ``workspace_size``, ``beta_lower_bound``, ``last_error``.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

_HERE = os.path.dirname(os.path.abspath(__file__))
# KO_LIB: alternative build of the same ABI (A/B measurements of kernel variants)
LIB_PATH = os.environ.get("KO_LIB") or os.path.join(_HERE, "lib", "libko.so")

PAGE_TOKENS = 16
MAX_OPS, MAX_VARIANTS, MAX_STAGES, MAX_PLANS, MAX_CLASSES, MAX_ROWS = 4, 8, 8, 64, 8, 16
COUNTS_PER_PLAN = 5 + 4 * MAX_STAGES
C_TP, C_FP, C_FN, C_OUT, C_GOLD = 0, 1, 2, 3, 4
STATUS = {0: "KO_OK", 1: "KO_EINVAL", 2: "KO_EUNSUPPORTED", 3: "KO_ECUDA", 4: "KO_EWORKSPACE"}


class KoError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class _KV(ctypes.Structure):
    _fields_ = [("n_layers", ctypes.c_int32), ("n_kv_heads", ctypes.c_int32),
                ("gqa_group", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("n_q", ctypes.c_int32), ("kv_pool", ctypes.c_void_p), ("n_pages", ctypes.c_int64),
                ("page_indptr", ctypes.c_void_p), ("page_ids", ctypes.c_void_p),
                ("seq_len", ctypes.c_void_p), ("n_tuples", ctypes.c_int64)]


class _Op(ctypes.Structure):
    _fields_ = [("n_classes", ctypes.c_int32), ("q", ctypes.c_void_p), ("w", ctypes.c_void_p),
                ("b", ctypes.c_void_p), ("w_is_bf16", ctypes.c_int32)]


class _Variant(ctypes.Structure):
    _fields_ = [("keep_permille", ctypes.c_int32), ("layer_cut", ctypes.c_int32)]


class _Stage(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("variant", ctypes.c_int32),
                ("theta_lo", ctypes.c_float), ("theta_hi", ctypes.c_float),
                ("is_final", ctypes.c_int32)]


class _Plan(ctypes.Structure):
    _fields_ = [("n_stages", ctypes.c_int32), ("stage", _Stage * MAX_STAGES)]


class _LossParams(ctypes.Structure):
    _fields_ = [("target_recall", ctypes.c_double), ("target_precision", ctypes.c_double),
                ("alpha", ctypes.c_double), ("beta", ctypes.c_double)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python __graft_entry__.py` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    L.ko_score_batch.argtypes = [ctypes.POINTER(_KV), P, I32, P, I32, P, I64, P, P, P, I32, P, P,
                                 P, ctypes.c_size_t, P]
    L.ko_score_batch.restype = ctypes.c_int
    L.ko_route.argtypes = [P, P, P, P, I32, I32, I64, I32, P, P, P, P, P, P]
    L.ko_route.restype = ctypes.c_int
    L.ko_reduce_stats.argtypes = [P, I32, P, P, P, I32, I32, I64, P, P, P]
    L.ko_reduce_stats.restype = ctypes.c_int
    L.ko_workspace_size.argtypes = [ctypes.POINTER(_KV), P, I32, I32, I64]
    L.ko_workspace_size.restype = ctypes.c_size_t
    L.ko_beta_lower_bound.argtypes = [I64, I64, ctypes.c_double]
    L.ko_beta_lower_bound.restype = ctypes.c_double
    L.ko_build_importance_order.argtypes = [ctypes.POINTER(_KV), P, P, P, P, P]
    L.ko_build_importance_order.restype = ctypes.c_int
    L.ko_embed_scores.argtypes = [P, I32, I64, P, I32, P, I32, I32, I32, P, I64, P, P]
    L.ko_embed_scores.restype = ctypes.c_int
    L.ko_soft_stats.argtypes = [P, P, P, ctypes.c_double, P, P, P, I32, I32, I64, P, P, P,
                                ctypes.c_size_t, P]
    L.ko_soft_stats.restype = ctypes.c_int
    L.ko_soft_workspace_size.argtypes = [I32, I64]
    L.ko_soft_workspace_size.restype = ctypes.c_size_t
    L.ko_beta_lower_bound_real.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double, P, P]
    L.ko_beta_lower_bound_real.restype = ctypes.c_double
    L.ko_plan_loss.argtypes = [P, P, I32, ctypes.c_double, P, I32, ctypes.POINTER(_LossParams),
                               P, P]
    L.ko_plan_loss.restype = ctypes.c_int
    L.ko_set_trace_events.argtypes = [P, P]
    L.ko_set_trace_events.restype = None
    L.ko_last_error.restype = ctypes.c_char_p
    L.ko_version.restype = ctypes.c_char_p
    L.ko_last_launch_count.restype = ctypes.c_int32
    return L


_lib = _load()
EXPORTS = ("ko_score_batch", "ko_route", "ko_reduce_stats", "ko_workspace_size",
           "ko_embed_scores", "ko_build_importance_order", "ko_soft_stats", "ko_soft_workspace_size",
           "ko_beta_lower_bound", "ko_beta_lower_bound_real", "ko_plan_loss",
           "ko_set_trace_events", "ko_last_error", "ko_version", "ko_last_launch_count")


def lib():
    return _lib


def last_error() -> str:
    return _lib.ko_last_error().decode()


def version() -> str:
    return _lib.ko_version().decode()


def last_launch_count() -> int:
    """Kernels launched by the last compute call on this thread (ko_last_launch_count)."""
    return int(_lib.ko_last_launch_count())


def _check(rc: int):
    if rc != 0:
        raise KoError(rc, last_error())


# ---------------------------------------------------------------------------------------------
# descriptors
# ---------------------------------------------------------------------------------------------
@dataclass
class KVCache:
    """Device tensors of one importance-ordered paged KV store (ko_kv_cache)."""
    pool: "torch.Tensor"          # bf16/uint16/int16 [n_pages][n_layers][2][n_kv_heads][16][D]
    page_indptr: "torch.Tensor"   # int64 [n_tuples+1]
    page_ids: "torch.Tensor"      # int32 [nnz]
    seq_len: "torch.Tensor"       # int32 [n_tuples]
    n_layers: int
    n_kv_heads: int
    gqa_group: int
    head_dim: int
    n_q: int = 1

    @property
    def n_tuples(self) -> int:
        return int(self.seq_len.numel())

    def _c(self) -> _KV:
        for name in ("pool", "page_indptr", "page_ids", "seq_len"):
            t = getattr(self, name)
            if not t.is_cuda:
                raise ValueError(f"KVCache.{name} must be a CUDA tensor (no CPU path)")
        return _KV(self.n_layers, self.n_kv_heads, self.gqa_group, self.head_dim, self.n_q,
                   _dp(self.pool), int(self.pool.shape[0]), _dp(self.page_indptr),
                   _dp(self.page_ids), _dp(self.seq_len), self.n_tuples)


@dataclass
class Operator:
    """One logical operator (ko_operator): n_classes 1 = filter, >= 2 = map-classify."""
    n_classes: int
    q: "torch.Tensor"   # bf16 [n_layers][Hq][n_q][D]
    w: "torch.Tensor"   # fp32 or bf16 [n_classes][n_layers][Hq][n_q][D]
    b: "torch.Tensor"   # fp32 [n_classes]


Stage = Tuple[int, int, float, float, int]


def _ops(ops: Sequence[Operator]):
    arr = (_Op * len(ops))()
    for i, o in enumerate(ops):
        for name in ("q", "w", "b"):
            if not getattr(o, name).is_cuda:
                raise ValueError(f"Operator.{name} must be a CUDA tensor")
        import torch
        w_bf16 = 1 if o.w.dtype == torch.bfloat16 else 0
        if not w_bf16 and o.w.dtype != torch.float32:
            raise ValueError("Operator.w must be float32 or bfloat16")
        arr[i] = _Op(int(o.n_classes), _dp(o.q), _dp(o.w), _dp(o.b), w_bf16)
    return arr


def _variants(vs: Sequence[Tuple[int, int]]):
    return (_Variant * len(vs))(*[_Variant(int(k), int(c)) for k, c in vs])


def make_plans(plans: Sequence[Sequence[Stage]]):
    arr = (_Plan * max(1, len(plans)))()
    for g, pl in enumerate(plans):
        if not 1 <= len(pl) <= MAX_STAGES:
            raise ValueError(f"plan {g}: {len(pl)} stages")
        arr[g].n_stages = len(pl)
        for s, (op, var, lo, hi, fin) in enumerate(pl):
            arr[g].stage[s] = _Stage(int(op), int(var), float(lo), float(hi), int(fin))
    return arr


def _dp(t) -> int:
    """Device pointer of a dense CUDA tensor.  The C ABI takes plain pointers to row-major arrays,
    so a strided view would be read with the wrong layout: refuse it (and host tensors)."""
    if not t.is_cuda:
        raise ValueError("tensor arguments must be CUDA tensors (there is no CPU path)")
    if not t.is_contiguous():
        raise ValueError(f"tensor of shape {tuple(t.shape)} is not contiguous: pass .contiguous()")
    return t.data_ptr()


def _ptr(t) -> Optional[int]:
    return None if t is None else _dp(t)


def _stream(stream) -> Optional[int]:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


# ---------------------------------------------------------------------------------------------
# entry points
# ---------------------------------------------------------------------------------------------
def workspace_size(kv: KVCache, ops: Sequence[Operator], n_variants: int, n_work: int) -> int:
    return int(_lib.ko_workspace_size(ctypes.byref(kv._c()), _ops(ops), len(ops), n_variants,
                                      n_work))


def alloc_workspace(kv: KVCache, ops: Sequence[Operator], n_variants: int, n_work: int):
    import torch
    n = workspace_size(kv, ops, n_variants, n_work)
    if n == 0:
        raise KoError(1, last_error() or "invalid arguments to ko_workspace_size")
    # torch's caching allocator returns ≥ 512-byte aligned blocks
    return torch.empty(n, dtype=torch.uint8, device=kv.pool.device)


def score_batch(kv: KVCache, ops: Sequence[Operator], variants: Sequence[Tuple[int, int]],
                tuple_idx=None, margins=None, classes=None, plans=None, gold=None, counts=None,
                workspace=None, stream=None, want_classes: bool = True):
    """ko_score_batch.  Returns (margins, classes, counts) device tensors (allocated here when not
    given; counts are accumulated into a given tensor)."""
    import torch
    dev = kv.pool.device
    n_ops, n_var, n = len(ops), len(variants), kv.n_tuples
    routed = plans is not None and len(plans) == 1
    if margins is None:  # with a tuple subset, the tuples outside it read NaN (not scored)
        margins = (torch.empty if tuple_idx is None else
                   lambda *a, **k: torch.full(*a, float("nan"), **k))(
            (n_ops, n_var, n), dtype=torch.float32, device=dev)
    if classes is None and want_classes:
        classes = torch.empty((n_ops, n_var, n), dtype=torch.int32, device=dev)
    n_plans = 0 if plans is None else len(plans)
    if counts is None and n_plans:
        counts = torch.zeros((n_plans, COUNTS_PER_PLAN), dtype=torch.int64, device=dev)
    n_work = n if tuple_idx is None else int(tuple_idx.numel())
    if tuple_idx is not None and n_work == 0:
        return margins, classes, counts      # empty selection: nothing to score or count
    if workspace is None:
        workspace = alloc_workspace(kv, ops, n_var, n_work)
    parr = make_plans(plans) if n_plans else None
    rc = _lib.ko_score_batch(ctypes.byref(kv._c()), _ops(ops), n_ops, _variants(variants), n_var,
                             _ptr(tuple_idx), n_work if tuple_idx is not None else 0,
                             _ptr(margins), _ptr(classes), parr, n_plans, _ptr(gold),
                             _ptr(counts), _dp(workspace), workspace.numel(),
                             _stream(stream))
    _check(rc)
    return margins, classes, counts


def route(plan: Sequence[Stage], margins, classes, n_classes: Sequence[int], stage: int,
          tuple_state, worklist=None, worklist_len=None, gold=None, counts=None, stream=None):
    """ko_route.  tuple_state (uint32 as int32 tensor) is updated in place."""
    import torch
    n_ops, n_var, n = margins.shape
    if counts is None:
        counts = torch.zeros((1, COUNTS_PER_PLAN), dtype=torch.int64, device=margins.device)
    nc = (ctypes.c_int32 * n_ops)(*[int(c) for c in n_classes])
    rc = _lib.ko_route(make_plans([plan]), _dp(margins), _ptr(classes), nc, n_ops, n_var, n,
                       stage, _dp(tuple_state), _ptr(worklist), _ptr(worklist_len),
                       _ptr(gold), _dp(counts), _stream(stream))
    _check(rc)
    return counts


def reduce_stats(plans: Sequence[Sequence[Stage]], margins, classes, n_classes: Sequence[int],
                 gold=None, counts=None, stream=None):
    """ko_reduce_stats: per-plan count rows on precomputed margins."""
    import torch
    n_ops, n_var, n = margins.shape
    if counts is None:
        counts = torch.zeros((len(plans), COUNTS_PER_PLAN), dtype=torch.int64,
                             device=margins.device)
    nc = (ctypes.c_int32 * n_ops)(*[int(c) for c in n_classes])
    rc = _lib.ko_reduce_stats(make_plans(plans), len(plans), _dp(margins), _ptr(classes),
                              nc, n_ops, n_var, n, _ptr(gold), _dp(counts), _stream(stream))
    _check(rc)
    return counts


def build_importance_order(src: KVCache, mu, sigma2, dst_pool, dst_page_ids, stream=None):
    """ko_build_importance_order: dst_pool (same geometry, pages dst_page_ids under the same
    CSR) receives every tuple's tokens in descending expected-attention order."""
    rc = _lib.ko_build_importance_order(ctypes.byref(src._c()), _dp(mu), _dp(sigma2),
                                        _dp(dst_pool), _dp(dst_page_ids),
                                        _stream(stream))
    _check(rc)
    return dst_pool


EXTERNAL = (0, 0)  # variant whose margins the caller supplies (e.g. embed_scores)


def embed_scores(item_emb, op_emb, op_ids: Sequence[int], margins, variant: int,
                 tuple_idx=None, stream=None):
    """ko_embed_scores: margins[op_ids[e]][variant][t] = cos(item_emb[t], op_emb[e])."""
    n_ops, n_var, n = margins.shape
    ids = (ctypes.c_int32 * len(op_ids))(*[int(x) for x in op_ids])
    n_idx = 0 if tuple_idx is None else int(tuple_idx.numel())
    rc = _lib.ko_embed_scores(_dp(item_emb), int(item_emb.shape[1]), int(item_emb.shape[0]),
                              _dp(op_emb), int(op_emb.shape[0]), ids, n_ops, int(variant),
                              n_var, _ptr(tuple_idx), n_idx, _dp(margins), _stream(stream))
    _check(rc)
    return margins


def soft_stats(plan: Sequence[Stage], pick_scores: Sequence[float], stage_cost: Sequence[float],
               tau: float, margins, n_classes: Sequence[int], gold=None, out=None,
               workspace=None, stream=None, classes=None):
    """ko_soft_stats: relaxed TP/FP/FN/cost and their Jacobian w.r.t. (s_i, θ⁻_i, θ⁺_i).
    Returns a device fp64 tensor [4 + 12·S] (see include/ko.h for the layout)."""
    import torch
    n_ops, n_var, n = margins.shape
    S = len(plan)
    if out is None:
        out = torch.empty(4 + 12 * S, dtype=torch.float64, device=margins.device)
    if workspace is None:
        workspace = torch.empty(int(_lib.ko_soft_workspace_size(S, n)), dtype=torch.uint8,
                                device=margins.device)
    pk = (ctypes.c_double * S)(*[float(x) for x in pick_scores])
    cs = (ctypes.c_double * S)(*[float(x) for x in stage_cost])
    nc = (ctypes.c_int32 * n_ops)(*[int(c) for c in n_classes])
    rc = _lib.ko_soft_stats(make_plans([plan]), pk, cs, float(tau), _dp(margins), _ptr(classes), nc, n_ops,
                            n_var, n, _ptr(gold), _dp(out), _dp(workspace),
                            workspace.numel(), _stream(stream))
    _check(rc)
    return out


def set_trace_events(ev_begin=None, ev_end=None) -> None:
    """ko_set_trace_events: torch.cuda.Event pair recorded around the hot kernel of later
    score_batch calls on this thread (None, None disables)."""
    import torch
    def handle(ev):
        if ev is None:
            return None
        if ev.cuda_event == 0:          # torch creates the CUDA event lazily on first record
            ev.record(torch.cuda.current_stream())
        return ev.cuda_event
    _lib.ko_set_trace_events(handle(ev_begin), handle(ev_end))


def beta_lower_bound(a: int, b: int, alpha: float) -> float:
    """ℓ_α = I^{-1}(1 − α; 1 + a, 1 + b) (Eqs. recall/precision lower bound)."""
    return float(_lib.ko_beta_lower_bound(int(a), int(b), float(alpha)))


def abi_ok() -> bool:
    """True when every symbol include/ko.h declares is exported by the loaded library."""
    return all(hasattr(_lib, s) for s in EXPORTS)


def beta_lower_bound_real(a: float, b: float, alpha: float):
    """ko_beta_lower_bound_real: (ℓ, dℓ/da, dℓ/db) for real-valued counts."""
    da, db = ctypes.c_double(), ctypes.c_double()
    v = float(_lib.ko_beta_lower_bound_real(float(a), float(b), float(alpha), ctypes.byref(da),
                                            ctypes.byref(db)))
    return v, da.value, db.value


LOSS_FIELDS = ("loss", "l_cost", "l_recall", "l_precision", "recall_lb", "precision_lb", "recall",
               "precision", "target_met_recall", "target_met_precision")


def plan_loss(stats: Sequence[float], stage_cost: Sequence[float], n_tuples: float,
              target_recall: float = 0.0, target_precision: float = 0.0, alpha: float = 0.95,
              beta: float = 10.0, jacobian=None):
    """ko_plan_loss (host).  stats = (TP, FP, FN, cost); jacobian: None or a [4][n_params] array
    (e.g. ko_soft_stats' out[4:].reshape(4, -1)).  Returns (dict of LOSS_FIELDS, grad list)."""
    import numpy as np
    st = (ctypes.c_double * 4)(*[float(x) for x in stats[:4]])
    sc = (ctypes.c_double * len(stage_cost))(*[float(x) for x in stage_cost])
    n_par, jac, grad = 0, None, None
    if jacobian is not None:
        J = np.ascontiguousarray(np.asarray(jacobian, np.float64).reshape(4, -1))
        n_par = J.shape[1]
        jac = (ctypes.c_double * J.size)(*J.ravel().tolist())
        grad = (ctypes.c_double * max(n_par, 1))()
    out = (ctypes.c_double * 10)()
    lp = _LossParams(float(target_recall), float(target_precision), float(alpha), float(beta))
    _check(_lib.ko_plan_loss(st, jac, n_par, float(n_tuples), sc, len(stage_cost),
                             ctypes.byref(lp), out, grad))
    return dict(zip(LOSS_FIELDS, list(out))), (list(grad)[:n_par] if grad is not None else None)
