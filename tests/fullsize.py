"""Test infrastructure for full-size parity: oracle scores of the tuples of a DEVICE-generated
workload.

The KV pages the GPU reads were written by kogen's device twin of the generator (a fixture, not the
product path).  They are copied to the host (each tuple's pages in logical order) and handed to the
CPU oracle, because regenerating hundreds of GB with the host twin would take tens of minutes; that
the copies are the generator's output is re-checked bitwise against the host twin
(kogen.host_pool) on a few tuples of every call.  Nothing here touches the product's outputs.
"""
from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

import kogen
import oracle


def _gather(d, local_ids):
    import torch
    indptr, ids, sl = d["indptr"], d["page_ids"], d["seq_len"]
    local_ids = np.asarray(local_ids, np.int64)
    cnt = indptr[local_ids + 1] - indptr[local_ids]
    lind = np.zeros(len(local_ids) + 1, np.int64)
    np.cumsum(cnt, out=lind[1:])
    pos = np.repeat(indptr[local_ids] - lind[:-1], cnt) + np.arange(int(lind[-1]))
    g = torch.from_numpy(ids[pos].astype(np.int64)).to(d["kv"].pool.device)
    host = d["kv"].pool.view(torch.int16).index_select(0, g).cpu().numpy().view(np.uint16)
    return host, lind, np.arange(int(lind[-1]), dtype=np.int32), sl[local_ids].copy()


def _verify(wl, t0, host, lind, sl, rows):
    """Bitwise: the copied pages of tuples `rows` (local) equal the host twin's, on valid slots."""
    spec = wl.spec
    for r in rows:
        ref, rind, rids, rsl = kogen.host_pool(spec, [t0 + int(r[1])], placement="contiguous")
        L = int(sl[r[0]])
        a = host[lind[r[0]]:lind[r[0] + 1]]
        b = ref[rids[rind[0]:rind[1]]]
        assert a.shape == b.shape
        full, rem = divmod(L, 16)
        assert np.array_equal(a[:full], b[:full]), "device pages differ from the host generator"
        if rem:
            assert np.array_equal(a[full, :, :, :, :rem], b[full, :, :, :, :rem])


def oracle_scores(wl, d, t0, local_ids, chunk_bytes=2 << 30, n_threads=0, verify=2):
    """fp64 oracle margins / classes [n_ops][n_var][len(local_ids)] of tuples local_ids (indices
    into the device workload d, whose tuple 0 is generator id t0)."""
    local_ids = np.asarray(local_ids, np.int64)
    ops = oracle.workload_ops(wl)
    n_ops, n_var = wl.spec.n_ops, len(wl.variants)
    m = np.empty((n_ops, n_var, len(local_ids)))
    c = np.empty((n_ops, n_var, len(local_ids)), np.int32)
    pages = (d["indptr"][local_ids + 1] - d["indptr"][local_ids]).astype(np.int64)
    per_chunk = max(1, int(chunk_bytes // wl.spec.page_bytes()))
    bounds = [0]
    acc = 0
    for i, p in enumerate(pages):
        acc += int(p)
        if acc >= per_chunk:
            bounds.append(i + 1)
            acc = 0
    if bounds[-1] != len(local_ids):
        bounds.append(len(local_ids))
    rng = np.random.default_rng(len(local_ids))
    checked = 0

    def run(a, b, host, lind, lids, sl):
        mm, cc = oracle.score(wl.spec, host, lind, lids, sl, ops, wl.variants, n_threads=n_threads)
        m[:, :, a:b] = mm
        c[:, :, a:b] = cc

    with ThreadPoolExecutor(1) as ex:          # copy chunk i+1 while the oracle scores chunk i
        fut = None
        for a, b in zip(bounds[:-1], bounds[1:]):
            host, lind, lids, sl = _gather(d, local_ids[a:b])
            if checked < verify:              # first tuple of chunk 0, a random one of chunk 1
                k = 0 if checked == 0 else int(rng.integers(b - a))
                _verify(wl, t0, host, lind, sl, [(k, local_ids[a + k])])
                checked += 1
            if fut is not None:
                fut.result()
            fut = ex.submit(run, a, b, host, lind, lids, sl)
        if fut is not None:
            fut.result()
    return m, c
