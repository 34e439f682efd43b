"""Parity rules between the CUDA path and the oracle (north star).

* margins: |m_gpu − m_oracle| ≤ MARGIN_TOL = 2e-3 for every computed (op, variant, tuple);
* decisions / counts: bit-exact wherever |m_oracle − θ| > BAND = 1e-2 for every threshold θ the
  entry meets (for maps also the top-1/top-2 gap, which decides the class).  Inside the band either
  decision is correct, so counts are compared as oracle.run_plans(m_merged) == gpu counts, where
  m_merged takes the oracle margin outside the band and the GPU margin inside it (Q19 (iii)).
"""
from __future__ import annotations

import numpy as np

import oracle

MARGIN_TOL = 2e-3
BAND = 1e-2


def thresholds_by_entry(plans, n_ops, n_var):
    th = [[set() for _ in range(n_var)] for _ in range(n_ops)]
    for pl in plans:
        for (o, v, lo, hi, fin) in pl:
            th[o][v].add(float(np.float32(lo)))
            th[o][v].add(float(np.float32(hi)))
    return th


def merged(m_or, c_or, m_gpu, c_gpu, plans, n_classes):
    """Q19 (iii) merge: GPU values inside the ambiguity band, oracle values outside."""
    n_ops, n_var, n = m_or.shape
    th = thresholds_by_entry(plans, n_ops, n_var)
    mm = m_or.astype(np.float64).copy()
    cc = c_or.copy()
    n_band = 0
    for o in range(n_ops):
        for v in range(n_var):
            band = np.zeros(n, bool)
            for t in th[o][v]:
                band |= np.abs(m_or[o, v] - t) <= BAND
            if n_classes[o] > 1:
                band |= m_or[o, v] <= BAND          # top-1/top-2 gap decides the class
            band &= np.isfinite(m_gpu[o, v])        # routed mode: unreached entries are NaN
            mm[o, v, band] = m_gpu[o, v, band]
            cc[o, v, band] = c_gpu[o, v, band]
            n_band += int(band.sum())
    return mm, cc, n_band


def assert_margins(m_gpu, m_or, mask=None, tol=MARGIN_TOL):
    d = np.abs(m_gpu.astype(np.float64) - m_or)
    if mask is not None:
        d = d[mask]
    assert np.all(np.isfinite(d)), "non-finite margin"
    assert d.max(initial=0.0) <= tol, f"max |Δm| = {d.max():.3e} > {tol}"
    return float(d.max(initial=0.0))


def assert_classes(c_gpu, c_or, m_or, n_classes):
    for o, C in enumerate(n_classes):
        if C <= 1:
            continue
        clear = m_or[o] > BAND
        assert np.array_equal(c_gpu[o][clear], c_or[o][clear]), "class mismatch outside band"


def assert_counts(counts_gpu, m_or, c_or, m_gpu, c_gpu, plans, n_classes, gold):
    mm, cc, n_band = merged(m_or, c_or, m_gpu, c_gpu, plans, n_classes)
    expect = oracle.run_plans(plans, mm, cc, n_classes, gold)
    assert np.array_equal(counts_gpu, expect), f"counts differ\n gpu {counts_gpu}\n exp {expect}"
    return n_band


def clear_tuples(m_or, plan, n_classes):
    """bool [n]: tuples whose oracle margin is farther than BAND from every threshold of every
    stage of the plan (and, for a map, whose top-1/top-2 gap exceeds BAND).  For them every
    decision of the plan walk is fixed, so per-tuple results must agree exactly (Q19 (ii))."""
    n = m_or.shape[2]
    ok = np.ones(n, bool)
    for (o, v, lo, hi, fin) in plan:
        m = m_or[o, v]
        for t in (float(np.float32(lo)), float(np.float32(hi))):
            ok &= np.abs(m - t) > BAND
        if n_classes[o] > 1:
            ok &= m > BAND
    return ok


def oracle_reached(stages, plan, shape):
    """bool [n_ops][n_var][n]: entries (op, variant) some stage of the plan reaches for the tuple,
    from the oracle's per-tuple stage outcomes (oracle.run_plans(..., want_stages=True)[g])."""
    reached = np.zeros(shape, bool)
    for s, (o, v, lo, hi, fin) in enumerate(plan):
        reached[o, v] |= stages[s] != oracle.STAGE_NOT_REACHED
    return reached


def gold_from_oracle(m_or, c_or, gold_variant, n_classes):
    """P_g of the paper (P:346 'the gold pipeline uses only the most expensive operator';
    P:763-764 recall/precision against P_g): per op, the final decision (θ_f = 0, Q6) of its gold
    variant on the ORACLE's margins — filters 1 iff m > 0, maps the argmax class."""
    n_ops = m_or.shape[0]
    g = np.empty((n_ops, m_or.shape[2]), np.uint8)
    for o in range(n_ops):
        g[o] = (m_or[o, gold_variant] > 0.0) if n_classes[o] <= 1 else c_or[o, gold_variant]
    return g


def gpu_alive(ko, plan, m_gpu, c_gpu, n_classes, gold=None):
    """P_o membership bool [n] by ko_route (stage −1) on the GPU's margins: the worklist it
    writes is exactly the alive set.  Also returns that call's count row."""
    import torch
    n = m_gpu.shape[2]
    st = torch.ones(n, dtype=torch.int32, device=m_gpu.device)
    wl = torch.empty(n, dtype=torch.int32, device=m_gpu.device)
    wlen = torch.zeros(1, dtype=torch.int64, device=m_gpu.device)
    cnt = ko.route(plan, m_gpu, c_gpu, n_classes, -1, st, wl, wlen, gold=gold)
    alive = np.zeros(n, bool)
    alive[wl[:int(wlen.item())].cpu().numpy()] = True
    sv = st.cpu().numpy().astype(np.uint32)
    assert np.array_equal(alive, (sv & 1).astype(bool)), "worklist != alive bits"
    return alive, cnt.cpu().numpy()[0]
