"""Small end-to-end exercise of every libko kernel (grid pass C1, routed C4 subset with its walk
kernel, reduce, route, soft relaxation, embedding stage on both load paths, cache builder) for
compute-sanitizer memcheck / racecheck / synccheck (tests/test_sanitizer_gpu.py).  Fixture-only:
no oracle."""
import sys, numpy as np, torch
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_04430_b200 as ko
from kogen import workloads
from kogen.device import device_workload
wl = workloads.get("C1"); d = device_workload(wl)
m, c, cnt = ko.score_batch(d["kv"], d["ops"], wl.variants, plans=wl.plans, gold=d["gold"])
wl4 = workloads.get("C4"); d4 = device_workload(wl4, n=64)
m4, c4, cnt4 = ko.score_batch(d4["kv"], d4["ops"], wl4.variants, plans=wl4.plans, gold=d4["gold"])
ko.reduce_stats(wl.plans, m, c, wl.spec.op_classes, gold=d["gold"])
st = torch.ones(64, dtype=torch.int32, device="cuda"); wlist = torch.empty(64, dtype=torch.int32, device="cuda"); wlen = torch.zeros(1, dtype=torch.int64, device="cuda")
ko.route(wl.plans[0], m, c, wl.spec.op_classes, -1, st, wlist, wlen, gold=d["gold"])
ko.soft_stats(wl.plans[0], [0.1, 0.0], [1.0, 2.0], 0.5, m, [1], gold=d["gold"])
item, opv = wl4.spec.embeddings(0, 100, 256)
di = torch.from_numpy(item.view(np.int16)).cuda().view(torch.bfloat16)
dq = torch.from_numpy(opv.view(np.int16)).cuda().view(torch.bfloat16)
me = torch.zeros((3, 1, 100), device="cuda")
ko.embed_scores(di, dq[:2], [0, 2], me, variant=0)                      # tensor-map path
ko.embed_scores(di, dq[:2], [0, 2], me, variant=0,
                tuple_idx=torch.arange(0, 100, 3, dtype=torch.int32, device="cuda"))  # gathers
sp4 = wl4.spec
mu = torch.randn((sp4.n_layers, sp4.n_kv_heads, sp4.head_dim), device="cuda")
s2 = torch.rand((sp4.n_layers, sp4.n_kv_heads, sp4.head_dim), device="cuda")
ko.build_importance_order(d4["kv"], mu, s2, torch.empty_like(d4["kv"].pool), d4["kv"].page_ids)
torch.cuda.synchronize(); print("ok", cnt[0, :5].tolist(), cnt4[0, :5].tolist())
