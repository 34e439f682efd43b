"""Subprocess probe for tests/test_debug_build_gpu.py: one small call through whichever libko the
KO_LIB environment variable selects, with optionally corrupted caller data.
usage: python tests/debug_probe.py {ok|bad_page|bad_len|bad_build} OUT.npy"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_04430_b200 as ko  # noqa: E402
from kogen import workloads  # noqa: E402
from kogen.device import device_workload  # noqa: E402

mode, out = sys.argv[1], sys.argv[2]
wl = workloads.get("C1")
d = device_workload(wl, n=16)
kv = d["kv"]
if mode == "bad_page":
    kv.page_ids[37] = kv.pool.shape[0] + 7          # a page id past the pool
elif mode == "bad_len":
    kv.seq_len[3] = 0                                # seq_len < 1
if mode == "bad_build":
    kv.page_ids[2] = -1
    mu = torch.zeros((1, 1, 64), device="cuda")
    dst = torch.empty_like(kv.pool)
    ko.build_importance_order(kv, mu, torch.ones_like(mu), dst, kv.page_ids)
    torch.cuda.synchronize()
    print("PROBE_DONE", flush=True)
    sys.exit(0)
m, _, _ = ko.score_batch(kv, d["ops"], wl.variants)
torch.cuda.synchronize()
np.save(out, m.cpu().numpy())
print("PROBE_DONE", ko.LIB_PATH, flush=True)
