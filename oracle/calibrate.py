"""Calibrate the per-op readout bias b_o of each synthetic workload with the ORACLE only.

b_o = −(1 − π_o)-quantile of the oracle's bias-free gold-variant margins over the first
N_CAL tuples, rounded to 1/256 (DESIGN.md §Input recipe), so that about π_o of
the tuples are gold positives.  Maps keep b = 0 for every class.  Per (op, variant) it also
records the threshold CENTER a stage of that variant is placed around (the per-stage thresholds
the paper's optimizer tunes): for filters the (1 − π_o)-quantile of that variant's
biased margins (same positive rate as gold), for maps the median confidence margin; rounded to
1/256.  Writes kogen/calibration.json and prints the ladder diagnostics (AUC of each variant
against the gold decision, agreement of gold with the latent label).

usage: python oracle/calibrate.py [C1 C2 ...]
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import kogen  # noqa: E402
from kogen import workloads  # noqa: E402
import oracle  # noqa: E402

N_CAL = {"C1": 64, "C2": 400, "C3": 300, "C4": 1000, "C5": 1000}


def auc(score, pos):
    pos = pos.astype(bool)
    if pos.all() or (~pos).all():
        return float("nan")
    order = np.argsort(score, kind="stable")
    ranks = np.empty(len(score)); ranks[order] = np.arange(1, len(score) + 1)
    n1 = pos.sum(); n0 = len(pos) - n1
    return float((ranks[pos].sum() - n1 * (n1 + 1) / 2) / (n1 * n0))


def calibrate(name):
    wl = workloads.get(name)
    n = min(N_CAL[name], wl.n_tuples)
    wl.bias = [[0.0] * c for c in wl.spec.op_classes]
    m, cls = oracle.score_workload(wl, np.arange(n))
    labels = wl.spec.labels(0, n)
    bias, centers = [], []
    for o, C in enumerate(wl.spec.op_classes):
        if C > 1:
            bias.append([0.0] * C)
            centers.append([round(float(np.median(m[o, v])) * 256) / 256
                            for v in range(len(wl.variants))])
            acc = [(cls[o, v] == labels[o]).mean() for v in range(len(wl.variants))]
            print(f"{name} op{o} map: class accuracy vs latent per variant {np.round(acc, 3)}")
            continue
        pi = wl.spec.op_pi_permille[o] / 1000.0
        g = m[o, wl.gold_variant]
        q = np.quantile(g, 1.0 - pi)
        b = -round(q * 256.0) / 256.0
        bias.append([b])
        centers.append([round(float(np.quantile(m[o, v] + b, 1.0 - pi)) * 256) / 256
                        for v in range(len(wl.variants))])
        gold = (g + b) > 0
        lat = labels[o] == 1
        aucs = [auc(m[o, v], gold) for v in range(len(wl.variants))]
        print(f"{name} op{o}: b={b:+.4f} std(gold m)={g.std():.3f} pos={gold.mean():.3f} "
              f"gold-vs-latent agree={np.mean(gold == lat):.3f} "
              f"AUC vs gold per variant {np.round(aucs, 3)} (variants {wl.variants})")
    return {"bias": bias, "centers": centers}


def main(names):
    cal = {k: v for k, v in workloads.load_calibration().items() if isinstance(v, dict)}
    for nm in names:
        cal[nm] = calibrate(nm)
    with open(workloads.CALIBRATION, "w") as f:
        json.dump(cal, f, indent=1, sort_keys=True)
    print("wrote", workloads.CALIBRATION)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"])
