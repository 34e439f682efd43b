"""Subprocess helper of tests/test_grid_final_gpu.py: one grid-mode ko_score_batch on C5-shaped
(and C3-shaped varlen) tuples with the 64-plan grid; writes margins, classes and counts to an
.npz.  The finaliser placement is chosen by KO_GRID_FIN_KERNEL in the environment (read once per
process by the library)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2602_04430_b200 as ko  # noqa: E402
from kogen import workloads  # noqa: E402
from kogen.device import device_workload  # noqa: E402

out = {}
for cfg, n in (("C5", 3000), ("C3", 400)):
    wl = workloads.get(cfg)
    d = device_workload(wl, n=n)
    m, c, counts = ko.score_batch(d["kv"], d["ops"], wl.variants, plans=wl.plans, gold=d["gold"])
    torch.cuda.synchronize()
    out[cfg + "_m"] = m.cpu().numpy()
    out[cfg + "_c"] = c.cpu().numpy()
    out[cfg + "_counts"] = counts.cpu().numpy()
    out[cfg + "_launches"] = np.array([ko.last_launch_count()])
np.savez(sys.argv[1], **out)
