"""Extract the dominant kernel's DRAM traffic from an `ncu --set full` report into
profiles/ncu_traffic_C<cfg>.json (bench.py reports it as roofline.traffic).

usage: python tools/ncu_traffic.py REPORT.ncu-rep CFG [kernel-regex]
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ALG = {1: 1056770, 2: 268500994, 3: 2148007938, 4: 337649666, 5: 2046951426}


def main():
    rep, cfg = sys.argv[1], int(sys.argv[2])
    pat = re.compile(sys.argv[3] if len(sys.argv) > 3 else r"ingest_kernel")
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ki = h.index("Kernel Name")
    rd, wr, dur = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum"), h.index("gpu__time_duration.sum")
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    tscale = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1, "s": 1}
    for r in rows[2:]:
        if not pat.search(r[ki]):
            continue
        rb = float(r[rd]) * scale[units[rd]]
        wb = float(r[wr]) * scale[units[wr]]
        secs = float(r[dur]) * tscale[units[dur]]
        d = {"kernel": r[ki].split("(")[0], "config": f"C{cfg}", "dram_read_bytes": rb, "dram_write_bytes": wb,
             "traffic_bytes": rb + wb, "alg_bytes": 9 * ALG[cfg], "ncu_duration_s": secs,
             "source": os.path.basename(rep)}
        path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                            f"ncu_traffic_C{cfg}.json")
        with open(path, "w") as fp:
            json.dump(d, fp, indent=1)
        print(json.dumps(d))
        return
    sys.exit("kernel not found in report")


if __name__ == "__main__":
    main()
