"""Host-side cost of one public-API call on a small trace (C1, pinned host columns):
wall time split by cProfile, next to the bare H2D and the device-resident call."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1805_04207_b200 import ColumnarTrace, consume, finalize, synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
tr = synth.device_trace(cfg, None)
n = tr.n_events
hk = torch.empty(n, dtype=torch.uint8, pin_memory=True); hk.copy_(tr.kind)
hp = torch.empty(n, dtype=torch.int64, pin_memory=True); hp.copy_(tr.payload)
ht = ColumnarTrace(hk, hp, tr.kernel_name, 0, tr.global_size, tr.local_size, tr.opcodes, [], tr.addr_stats)


def t(f, k=50):
    f(); torch.cuda.synchronize()
    s = time.perf_counter()
    for _ in range(k):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - s) / k * 1e3


dk = torch.empty_like(tr.kind); dp = torch.empty_like(tr.payload)
print(f"C{cfg}: bare H2D {t(lambda: (dk.copy_(hk, non_blocking=True), dp.copy_(hp, non_blocking=True))):.3f} ms | "
      f"device consume+finalize {t(lambda: finalize(consume(tr, max_entries=1 << 62))):.3f} ms | "
      f"host consume+finalize {t(lambda: finalize(consume(ht, max_entries=1 << 62))):.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    finalize(consume(ht, max_entries=1 << 62))
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
