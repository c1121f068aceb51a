"""Run a handful of golden producer cases (all schedules) once; used under compute-sanitizer."""
import json, os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from test_gpu_sim import _run, GOLD
cases = GOLD["cases"]
pick = [c for c in cases if c["name"].startswith("random")][:12] + [c for c in cases if not c["name"].startswith("random")][:6]
bad = 0
for c in pick:
    for sch in ("auto", "group", "sequential"):
        lines, err = _run(c, sch)
        ok = len(lines) == c["n_events"] and err == c["error"]
        bad += not ok
        print(c["name"], sch, "ok" if ok else f"MISMATCH {len(lines)} {c['n_events']} {err}")
print("mismatches", bad)
