"""Summarise an ncu launch-list CSV (``--metrics gpu__time_duration.sum,dram__bytes_read.sum,...
--csv --log-file X``) as a markdown table: per launch kernel, time, DRAM bytes and GB/s, plus each
kernel's share of the listed time.  Used for the summaries under profiles/."""
import csv
import sys
from collections import OrderedDict


def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    d = OrderedDict()
    for r in rows[1:]:
        e = d.setdefault(r[ii], {"kernel": r[ki]})
        e[r[mi]] = float(r[vi].replace(",", ""))
    return list(d.values())


def short(name):
    name = name.replace("(anonymous namespace)::", "").replace("ko::", "").replace("<unnamed>::", "")
    return name.split("(")[0].replace("void ", "")[:60]


def main(path, skip=0, limit=None):
    ls = load(path)[skip:]
    if limit:
        ls = ls[:limit]
    tot = sum(e.get("gpu__time_duration.sum", 0) for e in ls)
    print("| # | kernel | time (µs) | share | DRAM read (GB) | DRAM write (MB) | read GB/s |")
    print("|---|---|---|---|---|---|---|")
    for i, e in enumerate(ls):
        t = e.get("gpu__time_duration.sum", 0)
        rd = e.get("dram__bytes_read.sum", 0)
        wr = e.get("dram__bytes_write.sum", 0)
        print(f"| {i} | `{short(e['kernel'])}` | {t / 1e3:.1f} | {t / tot * 100:.1f} % | "
              f"{rd / 1e9:.3f} | {wr / 1e6:.1f} | {rd / t if t else 0:.0f} |")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0,
         int(sys.argv[3]) if len(sys.argv) > 3 else None)
