"""Device-side fixture: generate a workload's paged KV store, operators and labels on a GPU with
the device twin of the generator, wrapped in the product's descriptor types."""
from __future__ import annotations

from typing import Optional

import numpy as np

from . import PAGE, fill_device_pool, page_table
from .workloads import Workload, gold_from_labels


def device_workload(wl: Workload, t0: int = 0, n: Optional[int] = None, device: str = "cuda",
                    placement: str = "affine", poison: bool = True, w_dtype: str = "bf16"):
    """Returns dict(kv, ops, gold, seq_len, indptr, page_ids) for tuples t0 .. t0+n-1.

    kv.pool is generated on the device (bit-identical to kogen.host_pool); gold is the latent
    label of each tuple (filters y == +1, maps the class) — the labelled sample."""
    import torch
    import paper_2602_04430_b200 as ko

    spec = wl.spec
    n = wl.n_tuples if n is None else n
    seq_len = spec.seq_len(t0, n)
    indptr, ids = page_table(seq_len, placement)
    n_pages = max(int(indptr[-1]), 1)
    pool = torch.empty((n_pages, spec.n_layers, 2, spec.n_kv_heads, PAGE, spec.head_dim),
                       dtype=torch.bfloat16, device=device)
    d_indptr = torch.from_numpy(indptr).to(device)
    d_ids = torch.from_numpy(ids).to(device)
    stream = torch.cuda.current_stream().cuda_stream
    fill_device_pool(spec, t0, n, d_indptr.data_ptr(), d_ids.data_ptr(), pool.data_ptr(),
                     stream=stream, poison=poison)
    kv = ko.KVCache(pool=pool, page_indptr=d_indptr, page_ids=d_ids,
                    seq_len=torch.from_numpy(seq_len).to(device), n_layers=spec.n_layers,
                    n_kv_heads=spec.n_kv_heads, gqa_group=spec.gqa, head_dim=spec.head_dim,
                    n_q=spec.n_q)
    ops = host_ops_to_device(wl, device, w_dtype)
    gold = torch.from_numpy(gold_from_labels(spec.labels(t0, n), spec.op_classes)).to(device)
    return dict(kv=kv, ops=ops, gold=gold, seq_len=seq_len, indptr=indptr, page_ids=ids)


def host_ops_to_device(wl: Workload, device: str = "cuda", w_dtype: str = "bf16"):
    """Operators on the device.  The generator's readout is exactly representable in bf16
    (|int| ≤ 138 over a power of two), so w_dtype="bf16" passes the same values."""
    import torch
    import paper_2602_04430_b200 as ko
    bias = wl.biases()
    ops = []
    for o in range(wl.spec.n_ops):
        q = torch.from_numpy(wl.spec.q(o).view(np.int16)).to(device).view(torch.bfloat16)
        w32 = torch.from_numpy(wl.spec.w(o))
        if w_dtype == "bf16":
            wb = w32.to(torch.bfloat16)
            assert torch.equal(wb.float(), w32), "readout not exact in bf16"
            w = wb.to(device)
        else:
            w = w32.to(device)
        b = torch.tensor(bias[o], dtype=torch.float32, device=device)
        ops.append(ko.Operator(wl.spec.op_classes[o], q, w, b))
    return ops


def tensors_to_device(pool, indptr, page_ids, seq_len, geom, ops_host, device="cuda"):
    """Upload a host-built store (e.g. tests/helpers.build_pool) and oracle-style op dicts."""
    import torch
    import paper_2602_04430_b200 as ko
    kv = ko.KVCache(pool=torch.from_numpy(np.ascontiguousarray(pool).view(np.int16)).to(device)
                    .view(torch.bfloat16),
                    page_indptr=torch.from_numpy(np.ascontiguousarray(indptr, np.int64)).to(device),
                    page_ids=torch.from_numpy(np.ascontiguousarray(page_ids, np.int32)).to(device),
                    seq_len=torch.from_numpy(np.ascontiguousarray(seq_len, np.int32)).to(device),
                    n_layers=geom.n_layers, n_kv_heads=geom.n_kv_heads, gqa_group=geom.gqa,
                    head_dim=geom.head_dim, n_q=geom.n_q)
    ops = []
    for o in ops_host:
        q = torch.from_numpy(np.ascontiguousarray(o["q"]).view(np.int16)).to(device).view(torch.bfloat16)
        ops.append(ko.Operator(int(o["n_classes"]), q,
                               torch.from_numpy(np.ascontiguousarray(o["w"], np.float32)).to(device),
                               torch.from_numpy(np.ascontiguousarray(o["b"], np.float32)).to(device)))
    return kv, ops
