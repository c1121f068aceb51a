"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck): golden
traces, every synthetic config at a small size, the sparse and region paths, the
device validator, the NDRange producer and the multi-GPU job mode at world 1."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1805_04207_b200 import consume, finalize, synth  # noqa: E402
from paper_1805_04207_b200.metrics import validate_columnar  # noqa: E402
from paper_1805_04207_b200.trace import ColumnarTrace  # noqa: E402

root = os.getcwd()
cases = {c["name"]: c for c in json.load(open(os.path.join(root, "tests/golden/cases.json")))["cases"]}
arr = np.load(os.path.join(root, "tests/golden/traces.npz"))
for name in ("bfs_flags", "wavefront_big", "coin_20k", "hot_address", "barrier_rounds" if "barrier_rounds" in cases else "sweep4"):
    c = cases[name]
    o, n = c["offset"], c["n_events"]
    tr = ColumnarTrace(torch.from_numpy(arr["kind"][o:o + n].copy()).cuda(),
                       torch.from_numpy(arr["payload"][o:o + n].view(np.int64).copy()).cuda(),
                       c["kernel"], c["invocation"], tuple(c["global_size"]), tuple(c["local_size"]),
                       list(c["opcodes"]), [tuple(g) for g in c["extra_groups"]])
    finalize(consume(tr, max_entries=1 << 40))
    validate_columnar(tr)
for cfg, w in ((1, 4096), (2, 8192), (3, 4096), (4, 2048), (5, 2048)):
    finalize(consume(synth.device_trace(cfg, w), max_entries=1 << 40))
sys.argv = ["x", "sparse2"]
from tools.prof_step import far_buffers, scattered  # noqa: E402

small = synth.device_trace(2, 1 << 14)
finalize(consume(scattered(small), max_entries=1 << 40))
finalize(consume(far_buffers(small), max_entries=1 << 40))
print("sanitize workload done")
