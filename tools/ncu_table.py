"""Per-kernel table (duration, DRAM traffic and rate, SM / DRAM throughput %, registers)
from the raw CSVs tools/dbg/evidence.sh writes (one profiled step per workload).

usage: python tools/ncu_table.py DIR > table.md
"""
import csv
import glob
import os
import re
import sys


def main():
    d = sys.argv[1]
    print("# Every kernel of one profiled step per workload (`ncu --set full`, tools/dbg/evidence.sh)\n")
    print("Durations are ncu's serialised, cold-cache replays (a kernel's share of a step, not a bench value).\n")
    for path in sorted(glob.glob(os.path.join(d, "raw_*.csv"))):
        w = os.path.basename(path)[4:-4]
        rows = list(csv.reader(open(path)))
        hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        h, units = rows[hi], rows[hi + 1]
        col = {n: h.index(n) for n in h}
        scale = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}
        tsc = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
        print(f"## {w}\n")
        print("| kernel | µs | DRAM GB | DRAM GB/s | DRAM % | SM % | regs |")
        print("|---|---|---|---|---|---|---|")
        total = 0.0
        for r in rows[hi + 2:]:
            if len(r) < len(h):
                continue
            name = re.sub(r"\(.*", "", r[col["Kernel Name"]]).replace("aiwc::", "").replace("<unnamed>::", "")
            t = float(r[col["gpu__time_duration.sum"]]) * tsc.get(units[col["gpu__time_duration.sum"]], 1.0)
            rd = float(r[col["dram__bytes_read.sum"]]) * scale.get(units[col["dram__bytes_read.sum"]], 1.0)
            wr = float(r[col["dram__bytes_write.sum"]]) * scale.get(units[col["dram__bytes_write.sum"]], 1.0)
            dp = r[col["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]]
            sm = r[col["sm__throughput.avg.pct_of_peak_sustained_elapsed"]]
            reg = r[col["launch__registers_per_thread"]]
            total += t
            print(f"| {name} | {t:.1f} | {rd + wr:.3f} | {(rd + wr) / (t * 1e-6) if t else 0:.0f} | {float(dp):.1f} | "
                  f"{float(sm):.1f} | {reg} |")
        print(f"\nsum of kernel times: {total:.1f} µs\n")


if __name__ == "__main__":
    main()
