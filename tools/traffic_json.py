"""Fold the tools/traffic_capture.sh CSVs into profiles/ncu_traffic.json: mean
DRAM bytes (read + write) per MTTKRP launch for each <config>_R<R>_<dtype>.
Usage: python tools/traffic_json.py <dir with traffic_*.csv> [out.json]"""
import csv
import glob
import json
import os
import sys
from collections import defaultdict


def per_launch(path):
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    h = rows[0]
    ii, mi, vi = h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
    acc = defaultdict(float)
    for r in rows[1:]:
        if r[mi] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            acc[r[ii]] += float(r[vi].replace(",", ""))
    return sum(acc.values()) / max(len(acc), 1)


def main():
    d = sys.argv[1]
    out = sys.argv[2] if len(sys.argv) > 2 else "profiles/ncu_traffic.json"
    j = {"_about": "ncu DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per MTTKRP "
                   "launch, mean over the launches of one CP-ALS iteration (all modes), from "
                   "profiles/r01/traffic/ (tools/traffic_capture.sh). Keyed <config>_R<R>_<dtype>."}
    for p in sorted(glob.glob(os.path.join(d, "traffic_*.csv"))):
        key = os.path.basename(p)[len("traffic_"):-len(".csv")]
        j[key] = int(per_launch(p))
    json.dump(j, open(out, "w"), indent=1)
    print(json.dumps(j, indent=1))


if __name__ == "__main__":
    main()
