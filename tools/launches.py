"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per-kernel
count, total and mean time.  Usage: python tools/launches.py launches.csv [skip_first_n]"""
import csv
import sys
from collections import defaultdict


def load(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    H = rows[h]
    ki, vi, ui = H.index("Kernel Name"), H.index("Metric Value"), H.index("Metric Unit")
    out = []
    for r in rows[h + 1:]:
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1e-3)
        out.append((r[ki].split("(")[0].replace("void ", "")[:70], v * scale))
    return out


if __name__ == "__main__":
    seq = load(sys.argv[1])
    skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    seq = seq[skip:]
    agg = defaultdict(lambda: [0, 0.0])
    for n, t in seq:
        agg[n][0] += 1
        agg[n][1] += t
    tot = sum(t for _, t in seq)
    print(f"{'kernel':72s} {'count':>6s} {'total us':>11s} {'mean us':>9s} {'share':>6s}")
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n:72s} {c:6d} {t:11.1f} {t / c:9.2f} {100 * t / tot:5.1f}%")
    print(f"{'TOTAL':72s} {len(seq):6d} {tot:11.1f}")
