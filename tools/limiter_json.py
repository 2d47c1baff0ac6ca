"""Fold `ncu --set full` raw exports into profiles/ncu_limiter.json: what bounds
each workload's MTTKRP launches (mean over the captured launches).
Usage: python tools/limiter_json.py <key> <raw.csv> <limiter text> [profiles/ncu_limiter.json]"""
import csv
import json
import sys

M = {
    "l1tex_data_pipe_lsu_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "lts_throughput_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_throughput_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1_hit_pct": "l1tex__t_sector_hit_rate.pct",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
}


def main():
    key, path, limiter = sys.argv[1], sys.argv[2], sys.argv[3]
    out = sys.argv[4] if len(sys.argv) > 4 else "profiles/ncu_limiter.json"
    rows = list(csv.reader(open(path)))
    h, data = rows[0], rows[2:]
    col = {n: h.index(n) for n in h}
    f = lambda r, n: float(r[col[n]].replace(",", ""))  # noqa: E731
    e = {"kernel": sorted({r[col["Kernel Name"]].split("(")[0].replace("void ", "") for r in data}),
         "limiter": limiter, "launches": len(data), "source": path}
    for k, n in M.items():
        if n in col:
            e[k] = round(sum(f(r, n) for r in data) / len(data), 2)
    bscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    b = lambda r, n: f(r, n) * bscale.get(rows[1][col[n]], 1)  # noqa: E731
    e["dram_bytes_per_launch"] = int(sum(b(r, "dram__bytes_read.sum") + b(r, "dram__bytes_write.sum")
                                         for r in data) / len(data))
    unit = rows[1][col["gpu__time_duration.sum"]]
    scale = {"ms": 1.0, "us": 1e-3, "usecond": 1e-3, "ns": 1e-6, "nsecond": 1e-6}.get(unit, 1.0)
    e["duration_ms"] = [round(f(r, "gpu__time_duration.sum") * scale, 4) for r in data]
    try:
        j = json.load(open(out))
    except Exception:
        j = {}
    j["_about"] = ("What bounds the MTTKRP launches of each workload: means over the launches of one "
                   "ncu --set full capture (tools/limiter_json.py). Percentages are of the unit's "
                   "sustained peak over the launch.")
    j[key] = e
    json.dump(j, open(out, "w"), indent=1)
    print(json.dumps(e, indent=1))


if __name__ == "__main__":
    main()
