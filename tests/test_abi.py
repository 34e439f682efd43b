"""The C-ABI library loads and exports every symbol include/ko.h declares; host-side validation
and the host helper run without a GPU (no compute calls)."""
import ctypes
import math
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "ko.h")).read()
    return sorted(set(re.findall(r"^\s*(?:ko_status|size_t|double|void|int32_t|const char\*)\s+(ko_\w+)\(",
                                 src, re.M)))


def test_library_exports_every_declared_symbol():
    import paper_2602_04430_b200 as ko
    syms = header_symbols()
    assert set(syms) >= {"ko_score_batch", "ko_route", "ko_reduce_stats", "ko_workspace_size",
                         "ko_beta_lower_bound", "ko_last_error"}
    for s in syms:
        assert hasattr(ko.lib(), s), s
    assert ko.abi_ok()
    assert "sm_100a" in ko.version()


def test_struct_layouts_match_header():
    import paper_2602_04430_b200 as ko
    assert ctypes.sizeof(ko._Stage) == 20
    assert ctypes.sizeof(ko._Plan) == 4 + 8 * 20
    assert ctypes.sizeof(ko._KV) == 5 * 4 + 4 + 8 * 6   # 5 ints, pad, pointer/int64 fields
    assert ctypes.sizeof(ko._Op) == 40


def _kv(head_dim=128, layers=2, gqa=4):
    import paper_2602_04430_b200 as ko
    fake = 1 << 20      # never dereferenced: validation fails before any launch
    return ko._KV(layers, 2, gqa, head_dim, 1, fake, 10, fake, fake, fake, 5)


def _ops(n=1, classes=1):
    import paper_2602_04430_b200 as ko
    fake = 1 << 20
    arr = (ko._Op * n)()
    for i in range(n):
        arr[i] = ko._Op(classes, fake, fake, fake, 0)
    return arr


@pytest.mark.parametrize("mutate,needle,code", [
    (lambda a: a.update(kv=_kv(head_dim=96)), "head_dim", 1),
    (lambda a: a.update(variants=[(1001, 1)]), "keep_permille", 1),
    (lambda a: a.update(variants=[(500, 3)]), "layer_cut", 1),
    (lambda a: a.update(ops=_ops(classes=9)), "n_classes", 2),
    (lambda a: a.update(ops=_ops(n=5)), "n_ops", 1),
    (lambda a: a.update(ops=_ops(n=3), kv=_kv(gqa=8)), "rows", 2),
    (lambda a: a.update(kv=_kv(gqa=32)), "gqa_group", 2),
    (lambda a: a.update(plans=[[(0, 0, 1.0, -1.0, 0), (0, 0, 0, 0, 1)]] * 2), "theta_lo", 1),
    (lambda a: a.update(plans=[[(0, 0, -1.0, 1.0, 0)]] * 2), "no final", 1),
    (lambda a: a.update(plans=[[(0, 0, -1.0, 1.0, 1)]] * 2), "final filter", 1),
    (lambda a: a.update(plans=[[(0, 0, 0, 0, 1), (0, 0, -1, 1, 0)]] * 2), "after its final", 1),
    (lambda a: a.update(ws_bytes=16), "workspace", 4),
    # 16 rows of an 8-class fp32-readout map: 16 W·V entries per row exceed the table packing
    (lambda a: a.update(ops=_ops(classes=8), kv=_kv(gqa=16)), "W·V tiles", 2),
])
def test_validation_errors_without_gpu(mutate, needle, code):
    import paper_2602_04430_b200 as ko
    a = dict(kv=_kv(), ops=_ops(), variants=[(1000, 2), (500, 1)], plans=None, ws_bytes=1 << 40)
    mutate(a)
    plans = a["plans"]
    parr = ko.make_plans(plans) if plans else None
    fake = 1 << 20
    rc = ko.lib().ko_score_batch(ctypes.byref(a["kv"]), a["ops"], len(a["ops"]),
                                 ko._variants(a["variants"]), len(a["variants"]), None, 0,
                                 fake, None, parr, len(plans) if plans else 0, None,
                                 fake if plans else None, 1 << 20, a["ws_bytes"], None)
    assert rc == code, ko.last_error()
    assert needle in ko.last_error()


def test_workspace_size_host_only():
    import paper_2602_04430_b200 as ko
    n = ko.lib().ko_workspace_size(ctypes.byref(_kv()), _ops(2), 2, 3, 1000)
    assert n > 1000 * 2 * 2 * 2 * 3 * 4
    assert ko.lib().ko_workspace_size(ctypes.byref(_kv(head_dim=96)), _ops(), 1, 1, 10) == 0


def test_beta_lower_bound_host_helper():
    """The product's host Beta bound vs closed forms and the library routine (via the oracle)."""
    import paper_2602_04430_b200 as ko
    import oracle
    assert abs(ko.beta_lower_bound(0, 0, 0.95) - 0.05) < 1e-12
    assert abs(ko.beta_lower_bound(19, 0, 0.95) - 0.05 ** (1 / 20)) < 1e-12
    assert abs(ko.beta_lower_bound(0, 9, 0.95) - (1 - 0.95 ** 0.1)) < 1e-12
    for a, b in [(19, 1), (90, 10), (900, 100), (9000, 800), (45000, 3000), (3, 77)]:
        assert abs(ko.beta_lower_bound(a, b, 0.95) - oracle.beta_lower_bound(a, b, 0.95)) < 1e-10
    assert math.isnan(ko.beta_lower_bound(-1, 0, 0.95))


def test_binding_refuses_host_tensors():
    """No CPU path: the binding hands the C ABI device pointers only (and dense arrays only)."""
    import torch
    import paper_2602_04430_b200 as ko
    with pytest.raises(ValueError, match="CUDA"):
        ko._dp(torch.zeros(4))


def test_builder_rejects_pools_beyond_its_tma_views():
    """ko_build_importance_order moves every byte through 2-D TMA views of the pools whose row
    coordinate is int32 (ko.h): a pool of >= 2^31 rows is refused with KO_EUNSUPPORTED before any
    device work (checked here without a GPU: the pointers are never dereferenced)."""
    import paper_2602_04430_b200 as ko
    kv = _kv(head_dim=128, layers=2)
    rows_per_page = 2 * 2 * 2 * 16                      # 2·layers·heads·16 rows of head_dim
    kv.n_pages = (1 << 31) // rows_per_page + 1
    fake = 1 << 20
    rc = ko.lib().ko_build_importance_order(ctypes.byref(kv), ctypes.c_void_p(fake),
                                            ctypes.c_void_p(fake), ctypes.c_void_p(fake),
                                            ctypes.c_void_p(fake), None)
    assert rc == 2, ko.last_error()                     # KO_EUNSUPPORTED
    assert "int32" in ko.last_error()
