"""The seeded generator (kogen) — the input fixture shared by the oracle and the CUDA path.
Checks the recipe's properties (DESIGN.md §Input recipe) and determinism."""
import numpy as np

import kogen
from kogen import workloads
from tests.helpers import bf16_value


def test_values_exact_and_bounded():
    wl = workloads.get("C1")
    pool, indptr, ids, sl = kogen.host_pool(wl.spec, np.arange(8))
    v = bf16_value(pool)
    assert np.all(np.abs(v) <= 127 / 32)
    assert np.all(np.round(v * 32) == v * 32)         # on the 1/32 grid
    q = bf16_value(wl.spec.q(0))
    assert np.all(np.round(q * 32) == q * 32) and np.all(np.abs(q) <= 127 / 32)
    w = wl.spec.w(0).astype(np.float64) * (1 << wl.spec.w_log2_den)
    assert np.all(np.round(w) == w) and np.all(np.abs(w) <= 256)   # exact in bf16


def test_determinism_and_seed_separation():
    wl = workloads.get("C5")
    a = kogen.host_pool(wl.spec, [3, 7])[0]
    b = kogen.host_pool(wl.spec, [3, 7])[0]
    assert np.array_equal(a, b)
    wl2 = workloads.get("C5"); wl2.spec.seed = 99
    c = kogen.host_pool(wl2.spec, [3, 7])[0]
    assert not np.array_equal(a, c)


def test_tuple_subset_is_position_independent():
    """A tuple's pages do not depend on which other tuples are generated with it."""
    wl = workloads.get("C5")
    p1, i1, d1, _ = kogen.host_pool(wl.spec, [5], placement="contiguous")
    p2, i2, d2, _ = kogen.host_pool(wl.spec, [1, 5, 9], placement="contiguous")
    assert np.array_equal(p1[d1[i1[0]:i1[1]]], p2[d2[i2[1]:i2[2]]])


def test_noise_distribution_and_labels():
    wl = workloads.get("C5")
    pool, *_ = kogen.host_pool(wl.spec, np.arange(4))
    x = bf16_value(pool).ravel() * 32
    assert abs(x.mean()) < 1.0 and 28 < x.std() < 40
    lab = wl.spec.labels(0, 20000)
    assert abs(np.mean(lab[0] == 1) - 0.3) < 0.02 and abs(np.mean(lab[1] == 1) - 0.5) < 0.02


def test_lengths_log_uniform_octaves():
    wl = workloads.get("C3")
    L = wl.spec.seq_len(0, 20000)
    assert L.min() >= 256 and L.max() < 4096
    octave = np.floor(np.log2(L / 256)).astype(int)
    frac = np.bincount(octave, minlength=4) / len(L)
    assert np.all(np.abs(frac - 0.25) < 0.02)
    assert 1350 < L.mean() < 1520


def test_evidence_skewed_to_important_prefix():
    wl = workloads.get("C5")
    ev = wl.spec.evidence(0, 5000)
    assert ev.min() >= 0 and ev.max() < 256
    assert abs(np.mean(ev >= 128) - 0.375) < 0.02      # P(pos ≥ L/2) = 0.5·0.5 + 0.5·0.25


def test_page_table_bijection():
    sl = np.array([1, 16, 17, 100, 256], np.int32)
    indptr, ids = kogen.page_table(sl)
    assert indptr.tolist() == [0, 1, 2, 4, 11, 27]
    assert sorted(ids.tolist()) == list(range(27))
