#!/usr/bin/env python
"""bench.py — device-timed KV-cache scoring → routing → count pass (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ko|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...          (one rank per GPU, NCCL)

A step = one pass of the whole hot path over one batch of synthetic input resident in HBM:
ko_score_batch over every tuple (all ops × all variants in one read of each tuple's KV, margins,
every plan of the config's grid evaluated per tuple, integer counts) plus, at N > 1, the NCCL
all-reduce of the int64 count vector.  Weak scaling: each rank owns a distinct shard of
n_tuples tuples (tuple ids rank·n .. rank·n + n − 1), so value = N·n_tuples·K / max-rank time.

`--impl reference` times the reference arm of this tier: the fp64 CPU oracle (oracle/) as it
stands, on this host's cores, on a bounded sample of the same workload per step.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tuples scored/sec and % of HBM peak at 1/2/4/8 B200 vs CPU oracle"
UNIT = "tuples/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5",
                    help="C5 (default: the largest single-GPU config, 64-plan grid), C2, C3, C4")
    ap.add_argument("--placement", default="",
                    help="page placement override (default: the workload's, 'affine' = scattered)")
    ap.add_argument("--dump-counts", default="",
                    help="rank 0 writes the final int64 count array (.npy) here (tests)")
    ap.add_argument("--n-tuples", type=int, default=0, help="override tuples per rank")
    ap.add_argument("--impl", default="ko", choices=["ko", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="CPU work budget of the oracle sample (cpu_baseline / reference arm)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-gb", type=float, default=24.0,
                    help="pinned host memory per rank for the e2e batch")
    ap.add_argument("--embed-subset", type=float, default=0.0,
                    help="embed mode: score a sorted random subset (this fraction) of the tuples "
                         "through tuple_idx (the gathered path) instead of all of them")
    ap.add_argument("--mode", default="pass", choices=["pass", "soft", "embed", "build", "reduce"],
                    help="pass: the hot path (default); soft / embed / build: NEXT-1/3/4 kernels")
    return ap.parse_args()


# ------------------------------------------------------------------------------------------
# helpers
# ------------------------------------------------------------------------------------------
def n_kept(L, keep):
    return np.maximum(1, (L.astype(np.int64) * keep) // 1000)


def rank_range(wl, n_per, rank, world):
    """(first tuple id, tuple count) of this rank under weak scaling: the dataset is world·n_per
    tuples; fixed lengths → ids r·n_per .. r·n_per + n_per − 1; variable lengths → the contiguous
    range balanced by algorithmic bytes (full-read upper bound per tuple)."""
    if world == 1 or wl.spec.len_min == wl.spec.len_max:
        return rank * n_per, n_per
    from paper_2602_04430_b200.dist import shard_by_cost
    sl_all = wl.spec.seq_len(0, world * n_per).astype(np.int64)
    cost = np.zeros(len(sl_all))
    for l in range(wl.spec.n_layers):
        ks = [k for (k, c) in wl.variants if c > l]
        if ks:
            cost += n_kept(sl_all, max(ks))
    t0, t1 = shard_by_cost(cost, rank, world)
    return t0, t1 - t0


def algorithmic_bytes_routed(wl, seq_len, margins):
    """Routed mode: need(t,l) = largest n_kept over the (op, variant) entries the GPU itself
    reached for tuple t (finite margins, §8(d)) whose layer cut includes l."""
    sp = wl.spec
    reached = np.isfinite(margins)                     # [n_ops][n_var][n]
    need_tokens = 0
    for l in range(sp.n_layers):
        need = np.zeros(len(seq_len), np.int64)
        for v, (k, c) in enumerate(wl.variants):
            if c <= l:
                continue
            hit = reached[:, v, :].any(axis=0)
            need = np.maximum(need, np.where(hit, n_kept(seq_len, k), 0))
        need_tokens += int(need.sum())
    kv = need_tokens * sp.n_kv_heads * 4 * sp.head_dim
    n = len(seq_len)
    pages = int(((seq_len.astype(np.int64) + 15) // 16).sum())
    meta = 4 * pages + 12 * n
    out = 8 * int(reached.sum())
    return kv + meta + sp.n_ops * n + out, kv


def algorithmic_bytes(wl, seq_len, n_plans):
    """Σ_t Σ_l Hkv·4·d·need(t,l) (need = largest prefix any variant with cut > l
    consults; nested prefixes count once) + 4 B per page-table entry + 4 B seq_len + 8 B indptr
    + 1 B per gold byte + 4 B per margin and class written."""
    sp = wl.spec
    need_tokens = 0
    for l in range(sp.n_layers):
        ks = [k for (k, c) in wl.variants if c > l]
        if ks:
            need_tokens += int(n_kept(seq_len, max(ks)).sum())
    kv = need_tokens * sp.n_kv_heads * 4 * sp.head_dim
    n = len(seq_len)
    pages = int(((seq_len.astype(np.int64) + 15) // 16).sum())
    meta = 4 * pages + 12 * n
    gold = sp.n_ops * n
    out = 8 * sp.n_ops * len(wl.variants) * n
    return kv + meta + gold + out, kv


def gold_from_profiling(ko, torch, wl, kv, ops):
    """uint8 [n_ops][n] gold of every tuple: filters 1 iff the gold variant's margin > 0, maps the
    gold variant's argmax class (P_g, computed by the product outside the timed region)."""
    gv = wl.gold_variant
    m, c, _ = ko.score_batch(kv, ops, [wl.variants[gv]])
    g = torch.empty((wl.spec.n_ops, kv.n_tuples), dtype=torch.uint8, device=m.device)
    for o, C in enumerate(wl.spec.op_classes):
        g[o] = (m[o, 0] > 0).to(torch.uint8) if C <= 1 else c[o, 0].to(torch.uint8)
    del m, c
    return g


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        names = [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def read_stream_peak(torch, pool):
    """Read-only HBM stream rate over the workload's own KV pool (> L2), measured live: the
    ceiling of a kernel that only reads (MEASURED_PEAKS' hbm_gbs is a read+write copy)."""
    import kogen
    nbytes = pool.numel() * pool.element_size()
    nbytes = min(nbytes, 32 << 30) // (1 << 20) * (1 << 20)
    if nbytes < (1 << 30):
        return None
    sink = torch.zeros(148 * 8, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        kogen.read_stream(pool.data_ptr(), nbytes, sink.data_ptr(), s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = None
    for _ in range(5):
        e0.record()
        kogen.read_stream(pool.data_ptr(), nbytes, sink.data_ptr(), s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return nbytes / (best / 1000.0) / 1e9


def ncu_traffic(workload_key):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    e = d.get(workload_key)
    return None if e is None else e.get("dram_bytes_per_launch")


def oracle_sample(wl, seconds, rank_offset=0, threads=None, one_thread=True):
    """Time the oracle as it stands on a bounded, deterministic sample of the workload (all host
    cores; plus a 1-thread rate on a quarter of the budget)."""
    import oracle
    import kogen
    all_threads = len(os.sched_getaffinity(0))
    threads = threads or all_threads
    ops = oracle.workload_ops(wl)
    done, t_used, batch, start_t = 0, 0.0, 16, rank_offset
    stride = max(1, wl.n_tuples // 997)
    while t_used < seconds and done < wl.n_tuples:
        tids = (start_t + (np.arange(done, done + batch) * stride)) % (wl.n_tuples * 1000)
        pool, indptr, ids, sl = kogen.host_pool(wl.spec, tids)
        t0 = time.perf_counter()
        m, c = oracle.score(wl.spec, pool, indptr, ids, sl, ops, wl.variants, n_threads=threads)
        gold = np.zeros((wl.spec.n_ops, len(tids)), np.uint8)
        oracle.run_plans(wl.plans, m, c, wl.spec.op_classes, gold)
        t_used += time.perf_counter() - t0
        done += batch
        batch = min(256, batch * 2)
    out = dict(value=done / t_used, unit=UNIT, cores=threads, kind="oracle",
               sample=f"{done} tuples of {wl.name} (every {stride}-th id), all ops x variants "
                      f"scored + {len(wl.plans)} plans, fp64, input generation excluded",
               seconds=round(t_used, 2))
    if one_thread and threads > 1:
        o1 = oracle_sample(wl, seconds / 4, rank_offset, threads=1, one_thread=False)
        out["value_1_thread"] = o1["value"]
        out["sample_1_thread"] = o1["sample"]
    return out


# ------------------------------------------------------------------------------------------
# reference arm: the oracle on the host cores
# ------------------------------------------------------------------------------------------
def run_reference(args, rank, world):
    if rank != 0:
        return
    from kogen import workloads
    wl = workloads.get(args.config)
    per_step = args.cpu_seconds / max(1, args.steps + args.warmup)
    per_step = max(per_step, 0.5)
    vals = []
    cb = None
    for i in range(args.warmup + args.steps):
        cb = oracle_sample(wl, per_step, rank_offset=i * 7919)
        if i >= args.warmup:
            vals.append(cb["value"])
    v = float(np.mean(vals))
    cb["value"] = v
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{wl.name}: {wl.desc}", "mode": wl.mode,
                       "sample": "bounded per-step sample, host cores"},
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# product arm
# ------------------------------------------------------------------------------------------
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.mode != "pass":
        run_next(args)
        return

    import torch
    import paper_2602_04430_b200 as ko
    from kogen import workloads
    from kogen.device import device_workload

    # one rank per GPU; the modulo only matters for the 2-ranks-on-1-GPU test of this path
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dist = None
    if world > 1 or os.environ.get("KO_FORCE_DIST") == "1":  # (forced: exercise NCCL at N = 1)
        import torch.distributed as dist
        backend = os.environ.get("KO_DIST_BACKEND", "nccl")   # gloo: the same path on one GPU
        if backend == "nccl":
            # NCCL logs each communicator's rank / nranks at init (visible in the run's stderr)
            os.environ["NCCL_DEBUG"] = os.environ.get("KO_NCCL_DEBUG", "INFO")
            os.environ["NCCL_DEBUG_SUBSYS"] = os.environ.get("KO_NCCL_DEBUG_SUBSYS", "INIT")
            # NCCL logs to stdout by default: keep stdout for the one JSON line
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        print(f"[bench] rank {dist.get_rank()} of {dist.get_world_size()}: process group "
              f"backend {dist.get_backend()}, cuda:{local}", file=sys.stderr, flush=True)

    wl = workloads.get(args.config)
    n_per = args.n_tuples or wl.bench_n or wl.n_tuples
    # weak scaling: the dataset is world·n_per tuples; rank r owns a contiguous range — r·n_per
    # .. r·n_per + n_per − 1, or for variable lengths the range balanced by algorithmic bytes
    # (full-read upper bound per tuple)
    t0, n = rank_range(wl, n_per, rank, world)
    placement = args.placement or wl.placement
    d = device_workload(wl, t0=t0, n=n, placement=placement)
    kv, ops = d["kv"], d["ops"]
    n_var, n_ops = len(wl.variants), wl.spec.n_ops
    plans = wl.plans
    # labels = the paper's P_g ("the gold pipeline uses only the most expensive operator",
    # P:763-764 precision/recall against P_g): each op's final decision (θ_f = 0) on its gold
    # variant, from one profiling pass before the timed region (the labelled sample's labels)
    gold = gold_from_profiling(ko, torch, wl, kv, ops)
    margins = torch.empty((n_ops, n_var, n), dtype=torch.float32, device="cuda")
    classes = torch.empty((n_ops, n_var, n), dtype=torch.int32, device="cuda")
    counts = torch.zeros((len(plans), ko.COUNTS_PER_PLAN), dtype=torch.int64, device="cuda")
    ws = ko.alloc_workspace(kv, ops, n_var, n)
    stream = torch.cuda.current_stream()

    def step():
        counts.zero_()
        ko.score_batch(kv, ops, wl.variants, margins=margins, classes=classes, plans=plans,
                       gold=gold, counts=counts, workspace=ws)
        if dist is not None:
            dist.all_reduce(counts, op=dist.ReduceOp.SUM)

    # kernel-only events: the library records them around its hot kernel (ko_set_trace_events)
    ev_pairs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in range(args.steps)]

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for i in range(args.steps):
            ko.set_trace_events(ev_pairs[i][0], ev_pairs[i][1])
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    ko.set_trace_events(None, None)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    launches_per_step = ko.last_launch_count()   # the library's kernels in one step's call
    ms_total = e0.elapsed_time(e1)
    kern_ms = float(np.mean([a.elapsed_time(b) for a, b in ev_pairs]))
    t = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    ms_step = ms_total / args.steps
    value = world * n_per * args.steps / (ms_total / 1000.0)   # every rank's tuples

    cnt = counts.cpu().numpy()
    routed = len(plans) == 1
    if routed:
        alg_bytes, kv_bytes = algorithmic_bytes_routed(wl, d["seq_len"], margins.cpu().numpy())
    else:
        alg_bytes, kv_bytes = algorithmic_bytes(wl, d["seq_len"], len(plans))
    peak, peak_src = measured_peak()
    achieved = alg_bytes / (kern_ms / 1000.0) / 1e9
    read_peak = read_stream_peak(torch, kv.pool)
    key = f"{wl.name}:{n}"
    traffic = ncu_traffic(key)

    # e2e: the same pass through the public API from pinned host buffers, H2D inside the region
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, ko, torch, wl, d, ops, gold, plans, margins, classes, counts, ws, world,
                      dist)

    # host derivation (row a12 / NEXT-2): cheapest plan of the grid meeting the recall target
    selection = None
    if rank == 0 and len(plans) > 1:
        # NEXT-2 on the pass's counts: cheapest plan meeting ℓ_α^R ≥ 0.9 (labels = P_g), its
        # loss L (eqn:loss, β = 10) and Target Met = achieved recall / target
        from paper_2602_04430_b200 import plan_select
        best, _ = plan_select.select_plan(plans, cnt, wl.variants, target_recall=0.9,
                                          n_tuples=world * n_per)
        selection = {"target_recall": 0.9, "alpha": 0.95, "beta": 10.0,
                     "labels": "P_g (gold-variant decisions)",
                     "plan": None if best is None else best.index,
                     "cost_vs_gold": None if best is None else best.cost / (world * n_per * wl.spec.n_ops),
                     "recall_lb": None if best is None else best.recall_lb,
                     "recall": None if best is None else best.recall,
                     "precision": None if best is None else best.precision,
                     "target_met_recall": None if best is None else best.loss["target_met_recall"],
                     "loss": None if best is None else best.loss["loss"],
                     "l_cost": None if best is None else best.loss["l_cost"]}

    cb = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = oracle_sample(wl, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"{wl.name}: {wl.desc}", "n_tuples_per_rank": n,
                       "mode": ("routed (plan stages in order, only reached tuples scored)"
                                if routed else
                                "grid (all ops x variants in one read + per-tuple plan grid)"),
                       "n_plans": len(plans), "variants": wl.variants,
                       "kv_bytes_per_rank": kv_bytes, "placement": placement,
                       "gold": "P_g: each op's gold-variant decision (P:346, P:763-764), from a "
                               "profiling pass before the timed region",
                       "l2": "inputs larger than L2 (KV per rank >> 126 MB); no flush",
                       "parallelism": f"dp{world} (tuple shards, NCCL all-reduce of counts)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "ko_score_kernel", "kernel_ms": kern_ms,
                         "algorithmic_bytes_per_launch": alg_bytes, "peak_source": peak_src,
                         "read_stream_gbs": read_peak,
                         "frac_of_read_stream": None if not read_peak else achieved / read_peak},
            "cpu_baseline": cb,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
            "counts_plan0": cnt[0, :5].tolist(),
            "plan_selection": selection,
        }
        print(json.dumps(line), flush=True)
        if args.dump_counts:
            np.save(args.dump_counts, cnt)
    if dist is not None:
        dist.destroy_process_group()


def _time(fn, steps, warmup):
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def run_next(args):
    """Supplementary lines for the NEXT rows (not the driver's default): the soft relaxation of a
    C5 plan on the margins of a real C5 pass (NEXT-1), and the embedding-similarity stage over
    1 M tuples × 256 dims (NEXT-3)."""
    import torch
    import paper_2602_04430_b200 as ko
    from kogen import workloads
    from kogen.device import device_workload
    peak, peak_src = measured_peak()
    if args.mode == "soft":
        wl = workloads.get("C5")
        n = args.n_tuples or wl.bench_n
        d = device_workload(wl, n=n, placement="contiguous")
        m, c, _ = ko.score_batch(d["kv"], d["ops"], wl.variants)
        plan = wl.plans[9]
        S = len(plan)
        pick = [0.3, 0.0, -0.2, 0.0][:S]
        cost = [0.25, 1.0, 0.25, 1.0][:S]
        out = torch.empty(4 + 12 * S, dtype=torch.float64, device="cuda")
        ws = torch.empty(int(ko.lib().ko_soft_workspace_size(S, n)), dtype=torch.uint8, device="cuda")
        # captured in a CUDA graph: one optimizer iteration's device work without the per-call
        # Python marshalling (the optimizer would replay it the same way)
        gs = torch.cuda.CUDAGraph()
        sgs = torch.cuda.Stream()
        sgs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(sgs):
            ko.soft_stats(plan, pick, cost, 0.1, m, wl.spec.op_classes, gold=d["gold"], out=out,
                          workspace=ws)
            with torch.cuda.graph(gs, stream=sgs):
                ko.soft_stats(plan, pick, cost, 0.1, m, wl.spec.op_classes, gold=d["gold"], out=out,
                              workspace=ws)
        torch.cuda.current_stream().wait_stream(sgs)
        ms = _time(gs.replay, args.steps, args.warmup)
        items = (3 * S + 1) * n
        # bytes the pass reads (one margin per stage + the gold bits; nothing per tuple is
        # written): a latency-bound pass, reported next to its launch-floor-free time
        traffic = n * (S * 4 + wl.spec.n_ops)
        line = {"mode": "soft", "metric": "soft-relaxation evaluations (value + Jacobian) / s",
                "value": 1000.0 / ms, "unit": "evals/s", "ms_per_step": ms, "n_tuples": n,
                "n_stages": S, "params": 3 * S, "tuple_params_per_s": items / (ms / 1000.0),
                "input_gbs": traffic / (ms / 1000.0) / 1e9, "peak_gbs": peak,
                "config": {"workload": "C5 margins (50k tuples), plan " + str(plan)}}
    elif args.mode == "reduce":
        # ko_reduce_stats (the plan-grid reduction on a precomputed ProfileMatrix, §8(b)) and
        # ko_route (a whole routed plan on precomputed margins) over C5's 50 k × 6 margins
        wl = workloads.get("C5")
        n = args.n_tuples or wl.bench_n
        d = device_workload(wl, n=n, placement="contiguous")
        m, c, _ = ko.score_batch(d["kv"], d["ops"], wl.variants)
        counts = torch.zeros((len(wl.plans), ko.COUNTS_PER_PLAN), dtype=torch.int64, device="cuda")
        # captured in a CUDA graph: the per-call ctypes marshalling of 64 plans (≈ 0.1 ms of
        # Python) would otherwise dominate the device time of this small kernel
        g = torch.cuda.CUDAGraph()
        sg = torch.cuda.Stream()
        sg.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(sg):
            ko.reduce_stats(wl.plans, m, c, wl.spec.op_classes, gold=d["gold"], counts=counts)
            with torch.cuda.graph(g, stream=sg):
                ko.reduce_stats(wl.plans, m, c, wl.spec.op_classes, gold=d["gold"], counts=counts)
        torch.cuda.current_stream().wait_stream(sg)
        ms_r = _time(g.replay, args.steps, args.warmup)
        st = torch.ones(n, dtype=torch.int32, device="cuda")
        wlist = torch.empty(n, dtype=torch.int32, device="cuda")
        wlen = torch.zeros(1, dtype=torch.int64, device="cuda")

        def route():
            st.fill_(1)
            ko.route(wl.plans[0], m, c, wl.spec.op_classes, -1, st, wlist, wlen, gold=d["gold"])
        g2 = torch.cuda.CUDAGraph()
        sg.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(sg):
            route()
            with torch.cuda.graph(g2, stream=sg):
                route()
        torch.cuda.current_stream().wait_stream(sg)
        ms_t = _time(g2.replay, args.steps, args.warmup)
        line = {"mode": "reduce", "metric": "plan evaluations on precomputed margins / s",
                "unit": "tuple-plans/s", "value": n * len(wl.plans) / (ms_r / 1000.0),
                "ms_per_step": ms_r, "n_tuples": n, "n_plans": len(wl.plans),
                "route_whole_plan_ms": ms_t,
                "config": {"workload": f"C5 margins ({n} tuples x {len(wl.variants)} variants x "
                                       f"{wl.spec.n_ops} ops), {len(wl.plans)}-plan grid"}}
    elif args.mode == "build":
        wl = workloads.get("C2")
        n = args.n_tuples or 2000
        d = device_workload(wl, n=n, placement="contiguous")
        kv = d["kv"]
        g = torch.Generator().manual_seed(0)
        mu = torch.randn((wl.spec.n_layers, wl.spec.n_kv_heads, wl.spec.head_dim), generator=g).cuda()
        s2 = torch.rand((wl.spec.n_layers, wl.spec.n_kv_heads, wl.spec.head_dim), generator=g).cuda()
        dst = torch.empty_like(kv.pool)
        ms = _time(lambda: ko.build_importance_order(kv, mu, s2, dst, kv.page_ids),
                   args.steps, args.warmup)
        kvb = int(d["indptr"][-1]) * wl.spec.page_bytes()
        alg = 2 * kvb                     # the method's bytes: read K,V once + write K,V once
        line = {"mode": "build", "metric": "tuples ordered by expected attention / s",
                "unit": "tuples/s", "value": n / (ms / 1000.0), "ms_per_step": ms,
                "roofline": {"bound": "hbm", "achieved": alg / (ms / 1000.0) / 1e9, "peak": peak,
                             "unit": "GB/s", "frac": alg / (ms / 1000.0) / 1e9 / peak,
                             "peak_source": peak_src},
                "config": {"workload": f"C2 geometry, {n} tuples x 512 tokens, {kvb} B of KV"}}
    else:
        wl = workloads.get("C5")
        n = args.n_tuples or 8_000_000      # 4.1 GB of item embeddings: steady-state rate
        dim = 256
        item, op = wl.spec.embeddings(0, n, dim)
        di = torch.from_numpy(item.view(np.int16)).cuda().view(torch.bfloat16)
        dq = torch.from_numpy(op.view(np.int16)).cuda().view(torch.bfloat16)
        m = torch.empty((2, 1, n), device="cuda")
        idx, n_sc = None, n
        if args.embed_subset > 0:          # reached tuples of a cascade: a sorted worklist
            r = np.random.default_rng(7).random(n) < args.embed_subset
            idx = torch.from_numpy(np.nonzero(r)[0].astype(np.int32)).cuda()
            n_sc = int(idx.numel())
        ms = _time(lambda: ko.embed_scores(di, dq, [0, 1], m, variant=0, tuple_idx=idx),
                   args.steps, args.warmup)
        n = n_sc
        alg = n * dim * 2 + n * 2 * 4 + (n * 4 if idx is not None else 0)
        # the read ceiling of the same rows, measured live: a bulk-copy read-only stream over the
        # item table (contiguous) or over exactly the gathered rows (tuple_idx)
        if idx is None:
            stream_gbs = read_stream_peak(torch, di)
        else:
            import kogen
            sink = torch.zeros(148 * 8, dtype=torch.int32, device="cuda")
            cs = torch.cuda.current_stream().cuda_stream
            run = lambda: kogen.gather_stream(di.data_ptr(), dim * 2, idx.data_ptr(), n_sc,  # noqa: E731
                                              sink.data_ptr(), cs)
            stream_gbs = n_sc * dim * 2 / (_time(run, 5, 2) / 1000.0) / 1e9
        achieved = alg / (ms / 1000.0) / 1e9
        line = {"mode": "embed", "metric": "embedding-similarity scores / s", "unit": "tuples/s",
                "value": n / (ms / 1000.0), "ms_per_step": ms,
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak,
                             "unit": "GB/s", "frac": achieved / peak,
                             "peak_source": peak_src,
                             ("gather_stream_gbs" if idx is not None else "read_stream_gbs"): stream_gbs,
                             "frac_of_read_stream": achieved / stream_gbs if stream_gbs else None},
                "config": {"workload": f"{n} tuples x {dim}-d bf16 item embeddings, 2 operators"
                           + (f", gathered via tuple_idx ({args.embed_subset:g} of {len(item)})"
                              if idx is not None else "")}}
    print(json.dumps(line), flush=True)


def run_e2e(args, ko, torch, wl, d, ops, gold, plans, margins, classes, counts, ws, world, dist):
    """E2E: host (pinned) KV pages → device in tuple chunks on a copy stream, overlapped with
    scoring of the previous chunk on the compute stream; D2H of counts and margins each step."""
    kv = d["kv"]
    indptr = d["indptr"]
    # the e2e batch: the leading tuples of the shard whose pages fit args.e2e_gb of pinned host
    # memory per rank (pinning hundreds of GB per node would dominate the run; the metric is a
    # rate, and the H2D stream is the bound either way)
    page_bytes = kv.pool[0].numel() * kv.pool.element_size()
    n = kv.n_tuples
    cap_pages = int(args.e2e_gb * 1e9 // page_bytes)
    if int(indptr[-1]) > cap_pages:
        n = int(np.searchsorted(indptr, cap_pages, side="right") - 1)
    n_pages = int(indptr[n])
    try:
        host_pool = torch.empty((n_pages,) + tuple(kv.pool.shape[1:]), dtype=kv.pool.dtype,
                                pin_memory=True)
    except RuntimeError as e:  # noqa: BLE001
        return {"value": None, "unit": UNIT, "error": f"pinned host alloc failed: {e}"[:200]}
    # The host holds the batch's pages in logical (tuple-major) order, the natural layout of a
    # store streamed from host memory; the e2e view uses the matching contiguous page table, so a
    # tuple chunk is one contiguous page range (filled outside the timed region).
    ids_dev = kv.page_ids.to(torch.int64)
    step_p = max(1, (4 << 30) // page_bytes)
    for a in range(0, n_pages, step_p):
        b = min(n_pages, a + step_p)
        host_pool[a:b].copy_(kv.pool.index_select(0, ids_dev[a:b]))
    torch.cuda.synchronize()
    kv = ko.KVCache(pool=kv.pool, page_indptr=kv.page_indptr,
                    page_ids=torch.arange(kv.page_ids.numel(), dtype=torch.int32, device="cuda"),
                    seq_len=kv.seq_len, n_layers=kv.n_layers, n_kv_heads=kv.n_kv_heads,
                    gqa_group=kv.gqa_group, head_dim=kv.head_dim, n_q=kv.n_q)
    h_margins = torch.empty(margins.shape, dtype=margins.dtype, pin_memory=True)
    h_counts = torch.empty(counts.shape, dtype=counts.dtype, pin_memory=True)
    n_chunks = 8
    bounds = np.linspace(0, n, n_chunks + 1).astype(np.int64)
    chunk_idx = [torch.arange(int(a), int(b), dtype=torch.int32, device="cuda")
                 for a, b in zip(bounds[:-1], bounds[1:])]
    copy_s = torch.cuda.Stream()
    comp_s = torch.cuda.current_stream()
    # per-chunk "scored" events: the next step's copy into a chunk's pages waits until this
    # step's scoring of that chunk has read them (no write-after-read race on the device pool)
    done_evs = [None] * n_chunks

    def e2e_step():
        counts.zero_()
        evs = []
        for c in range(n_chunks):
            p0, p1 = int(indptr[bounds[c]]), int(indptr[bounds[c + 1]])
            with torch.cuda.stream(copy_s):
                if done_evs[c] is not None:
                    copy_s.wait_event(done_evs[c])
                kv.pool[p0:p1].copy_(host_pool[p0:p1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy_s)
            evs.append(ev)
        for c in range(n_chunks):
            comp_s.wait_event(evs[c])
            ko.score_batch(kv, ops, wl.variants, tuple_idx=chunk_idx[c], margins=margins,
                           classes=classes, plans=plans, gold=gold, counts=counts, workspace=ws)
            done_evs[c] = torch.cuda.Event()
            done_evs[c].record(comp_s)
        if dist is not None:
            dist.all_reduce(counts, op=dist.ReduceOp.SUM)
        h_counts.copy_(counts, non_blocking=True)
        h_margins.copy_(margins, non_blocking=True)

    # the resident pass's margins of the e2e batch, to check the streamed pass reproduces them
    ref_m = margins[:, :, :n].clone()
    e2e_step()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp_s)
    for _ in range(args.e2e_steps):
        e2e_step()
    e1.record(comp_s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    n_all = torch.tensor([n], dtype=torch.int64, device="cuda")   # tuples of every rank's batch
    if dist is not None:
        dist.all_reduce(n_all, op=dist.ReduceOp.SUM)
    n_all = int(n_all.item())
    h2d = n_pages * page_bytes
    d2h = h_counts.numel() * 8 + h_margins.numel() * 4
    # bitwise: margins are order-independent fixed-order sums, so the streamed pass must equal
    # the resident one on the same pages (routed: the same entries unreached, i.e. NaN)
    a_m, r_m = h_margins[:, :, :n], ref_m.cpu()
    same = bool(((a_m == r_m) | (torch.isnan(a_m) & torch.isnan(r_m))).all())
    del host_pool
    return {"value": n_all * args.e2e_steps / (ms / 1000.0), "unit": UNIT,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
            "ms_per_step": ms / args.e2e_steps, "tuples_per_rank": n,
            "margins_equal_resident_pass": same,
            "how": "pinned host KV pages -> device in 8 tuple chunks on a copy stream, "
                   "overlapped with ko_score_batch on each landed chunk; counts+margins D2H"}


if __name__ == "__main__":
    main()
