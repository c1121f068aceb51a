"""Summarise `ncu --set full` reports (one launch per kernel) into the text form kept
under profiles/: duration, DRAM traffic and throughput, issue / pipe utilisation,
occupancy, registers, shared memory, and the top warp-stall reasons.

usage: python tools/ncu_summary.py REPORT.ncu-rep [...]
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("duration", "gpu__time_duration.sum"),
    ("DRAM read", "dram__bytes_read.sum"),
    ("DRAM write", "dram__bytes_write.sum"),
    ("DRAM throughput % of peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("SM throughput %", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("issue active %", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
    ("warps active % (achieved occupancy)", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("registers/thread", "launch__registers_per_thread"),
    ("static smem/CTA", "launch__shared_mem_per_block_static"),
    ("dynamic smem/CTA", "launch__shared_mem_per_block_dynamic"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
    ("warp instructions", "smsp__inst_executed.sum"),
    ("L2 hit rate %", "lts__t_sector_hit_rate.pct"),
    ("L2 RED/ATOM sectors", "lts__t_sectors_srcunit_tex_op_red.sum"),
]


def main():
    for rep in sys.argv[1:]:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                             check=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        h, units = rows[0], rows[1]
        for r in rows[2:]:
            print(f"## {r[h.index('Kernel Name')].split('(')[0]}  ({rep.split('/')[-1]})")
            for label, m in METRICS:
                if m in h:
                    i = h.index(m)
                    print(f"{label:40s} {r[i]} {units[i]}")
            stalls = []
            for i, name in enumerate(h):
                if name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio"):
                    try:
                        stalls.append((float(r[i]), name[len("smsp__average_warps_issue_stalled_"):-len(
                            "_per_issue_active.ratio")]))
                    except ValueError:
                        pass
            stalls.sort(reverse=True)
            print("top stalls (warps per issue): " + ", ".join(f"{n} {v:.2f}" for v, n in stalls[:6]))
            print()


if __name__ == "__main__":
    main()
