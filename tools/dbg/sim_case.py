import json, sys, os
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from test_gpu_sim import _run, GOLD
names = sys.argv[1:]
for c in GOLD["cases"]:
    if c["name"] in names:
        for sch in ("auto", "group", "sequential"):
            lines, err = _run(c, sch)
            print(c["name"], sch, len(lines), c["n_events"], err, c["error"])
