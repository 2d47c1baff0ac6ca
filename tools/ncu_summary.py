"""Key metrics of every profiled launch in an `ncu --page raw --csv` export.
Usage: python tools/ncu_summary.py raw.csv [label]"""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum", "L2 read hit sectors"),
    ("lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum", "L2 read miss sectors"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 % peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1tex % peak"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers"),
    ("smsp__inst_executed_op_global_red.sum", "RED instructions"),
]


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    h, u = rows[0], rows[1]
    label = sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]
    ki = h.index("Kernel Name")
    print(f"### {label}\n")
    print("| metric | " + " | ".join(f"launch {i}" for i in range(len(rows) - 2)) + " |")
    print("|---|" + "---|" * (len(rows) - 2))
    print("| kernel | " + " | ".join(r[ki].split("(")[0].replace("void ", "")[:48] for r in rows[2:]) + " |")
    for key, name in KEYS:
        if key in h:
            i = h.index(key)
            print(f"| {name} ({u[i]}) | " + " | ".join(r[i] for r in rows[2:]) + " |")
    print()


if __name__ == "__main__":
    main()
