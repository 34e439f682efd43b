"""Named synthetic workloads C1–C5 = BASELINE.json configs[0..4] (shapes from SURVEY.md §8(d)).

Each preset fixes the generator geometry, the variant ladder, the plan(s) and the per-op readout
bias b_o.  The biases were written by ``oracle/calibrate.py`` (which calls only ``oracle/``):
b_o = −(1 − π_o)-quantile of the oracle's bias-free gold-variant margins over the first tuples,
rounded to 1/256, so that about π_o of the tuples are gold positives (DESIGN.md §Input recipe).
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

from . import GenSpec

_HERE = os.path.dirname(os.path.abspath(__file__))
CALIBRATION = os.path.join(_HERE, "calibration.json")

Stage = Tuple[int, int, float, float, int]   # (op, variant, theta_lo, theta_hi, is_final)


@dataclass
class Workload:
    name: str
    desc: str
    spec: GenSpec
    n_tuples: int
    variants: List[Tuple[int, int]]          # (keep_permille, layer_cut)
    gold_variant: int                          # index of the gold (most expensive) variant
    plans: List[List[Stage]]
    mode: str = "grid"                         # "grid" (profiling + plan grid) or "routed"
    bias: Optional[List[List[float]]] = None   # [op][class]
    bench_n: int = 0                           # tuples per rank per bench step (resident batch)
    placement: str = "affine"                  # bench page placement: scattered pages (page_table)

    def biases(self) -> List[List[float]]:
        if self.bias is not None:
            return self.bias
        cal = load_calibration().get(self.name)
        if cal is None:
            return [[0.0] * c for c in self.spec.op_classes]
        return cal["bias"]


def load_calibration() -> Dict[str, List[List[float]]]:
    if not os.path.exists(CALIBRATION):
        return {}
    with open(CALIBRATION) as f:
        return {k: v for k, v in json.load(f).items() if isinstance(v, dict)}


def center(name: str, op: int, var: int) -> float:
    """Calibrated threshold center of (op, variant) (oracle/calibrate.py), 0 if uncalibrated."""
    cal = load_calibration().get(name)
    return float(cal["centers"][op][var]) if cal else 0.0


def _sym(op: int, var: int, half: float, c: float = 0.0) -> Stage:
    return (op, var, c - half, c + half, 0)


def _final(op: int, var: int, theta: float = 0.0) -> Stage:
    return (op, var, theta, theta, 1)


def c1() -> Workload:
    spec = GenSpec(seed=1, n_layers=1, n_kv_heads=1, gqa=1, head_dim=64, n_q=1,
                   op_classes=[1], op_pi_permille=[300], len_min=128, len_max=128, w_log2_den=6)
    variants = [(1000, 1), (500, 1)]
    plans = [[_sym(0, 1, h, center("C1", 0, 1)), _final(0, 0)] for h in (0.5, 1.0, 2.0)]
    return Workload("C1", "single semantic filter, 64 tuples, 1 KV head, head_dim 64, 1 layer, "
                    "prefix 128, 3 threshold variants", spec, 64, variants, 0, plans, bench_n=64)


def c2() -> Workload:
    spec = GenSpec(seed=2, n_layers=4, n_kv_heads=8, gqa=4, head_dim=128, n_q=1,
                   op_classes=[1, 1], op_pi_permille=[300, 500], len_min=512, len_max=512)
    variants = [(200, 2), (500, 4), (1000, 4)]
    plans = []
    for h1 in (0.5, 1.0, 2.0, 4.0):          # 4 x 4 grid of per-op half-widths (budget split)
        for h2 in (0.5, 1.0, 2.0, 4.0):
            plans.append([_sym(0, 0, h1, center("C2", 0, 0)), _sym(0, 1, h1, center("C2", 0, 1)),
                          _final(0, 2),
                          _sym(1, 0, h2, center("C2", 1, 0)), _sym(1, 1, h2, center("C2", 1, 1)),
                          _final(1, 2)])
    return Workload("C2", "two-filter conjunctive pipeline, 10k tuples, 8 KV heads GQA 4:1, "
                    "head_dim 128, 4 layers, prefix 512, global recall target 0.9",
                    spec, 10_000, variants, 2, plans, bench_n=10_000)


def c3() -> Workload:
    spec = GenSpec(seed=3, n_layers=2, n_kv_heads=8, gqa=4, head_dim=128, n_q=1,
                   op_classes=[1], op_pi_permille=[300], len_min=256, len_max=4096)
    variants = [(k, c) for c in (1, 2) for k in (1000, 500, 200)]
    plans = [[_final(0, v, center("C3", 0, v))] for v in range(len(variants))]
    return Workload("C3", "100k documents, variable prefix 256-4096 in 16-token pages, sweep of "
                    "prefix/layer-cut variants", spec, 100_000, variants, 3, plans,
                    bench_n=10_000)     # 1.13 TB total: resident batches of 10 k docs (~113 GB)


def c4() -> Workload:
    spec = GenSpec(seed=4, n_layers=2, n_kv_heads=8, gqa=4, head_dim=128, n_q=1,
                   op_classes=[1, 4, 1], op_pi_permille=[500, 500, 500], len_min=128, len_max=128)
    variants = [(500, 1), (1000, 2)]
    cm = max(center("C4", 1, 0), 0.0)
    plans = [[_sym(0, 0, 1.0, center("C4", 0, 0)), _final(0, 1), (1, 0, cm, cm, 0), _final(1, 1),
              _sym(2, 0, 1.0, center("C4", 2, 0)), _final(2, 1)]]
    return Workload("C4", "three-operator pipeline filter->map-classify->filter, small->large "
                    "cascades, 1M tuples", spec, 1_000_000, variants, 1, plans, mode="routed",
                    bench_n=125_000)    # 1M sharded over 8 GPUs = 125 k per GPU (~131 GB)


def c5() -> Workload:
    spec = GenSpec(seed=5, n_layers=2, n_kv_heads=8, gqa=4, head_dim=128, n_q=1,
                   op_classes=[1, 1], op_pi_permille=[300, 500], len_min=256, len_max=256)
    variants = [(1000, 2), (500, 2), (200, 1)]
    per_op = [(v, h) for v in (2, 1) for h in (0.25, 0.5, 1.0, 2.0)]
    plans = []
    for v1, h1 in per_op:
        for v2, h2 in per_op:
            plans.append([_sym(0, v1, h1, center("C5", 0, v1)), _final(0, 0),
                          _sym(1, v2, h2, center("C5", 1, v2)), _final(1, 0)])
    return Workload("C5", "per-pipeline recall/cost statistics over a 50k labelled sample for a "
                    "64-point threshold/variant grid", spec, 50_000, variants, 0, plans,
                    bench_n=50_000)


ALL = {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5}


def get(name: str) -> Workload:
    return ALL[name.upper()]()


def gold_from_labels(labels, op_classes) -> "np.ndarray":
    """uint8 [n_ops][n] gold bytes from latent labels (filters: y == +1; maps: the class)."""
    import numpy as np
    out = np.empty(labels.shape, np.uint8)
    for o, c in enumerate(op_classes):
        out[o] = (labels[o] == 1) if c <= 1 else labels[o]
    return out
