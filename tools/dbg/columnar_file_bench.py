"""consume_file on the binary columnar form of a synthetic config (page cache warm):
file -> memory map -> H2D -> engine (in-pass stream check) -> report."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1805_04207_b200 import consume_file, finalize, synth  # noqa: E402
from paper_1805_04207_b200.tracefile import write_columnar  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
path = f"/tmp/aiwc_c{cfg}.aiwcc"
tr = synth.device_trace(cfg)
n = tr.n_events
t0 = time.perf_counter()
write_columnar(tr, path)
print(f"C{cfg}: {tr.n_events} events, {os.path.getsize(path) / 1e9:.2f} GB written in {time.perf_counter() - t0:.1f} s")
del tr
torch.cuda.empty_cache()
for i in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = finalize(consume_file(path, max_entries=1 << 62))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"consume_file + finalize: {dt * 1e3:.1f} ms = {n / dt / 1e9:.2f} G events/s")
os.remove(path)
