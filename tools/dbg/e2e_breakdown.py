"""Where the e2e step's time goes beyond the bare H2D copy (C2, pinned host columns)."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1805_04207_b200 import ColumnarTrace, consume, finalize, synth  # noqa: E402

tr = synth.device_trace(2, None)
n = tr.n_events
hk = torch.empty(n, dtype=torch.uint8, pin_memory=True); hk.copy_(tr.kind)
hp = torch.empty(n, dtype=torch.int64, pin_memory=True); hp.copy_(tr.payload)
ht = ColumnarTrace(hk, hp, tr.kernel_name, 0, tr.global_size, tr.local_size, tr.opcodes, [], tr.addr_stats)
dk = torch.empty_like(tr.kind); dp = torch.empty_like(tr.payload)


def t(f, k=5):
    f(); torch.cuda.synchronize()
    s = time.perf_counter()
    for _ in range(k):
        r = f()
    torch.cuda.synchronize()
    return (time.perf_counter() - s) / k * 1e3, r


bare, _ = t(lambda: (dk.copy_(hk, non_blocking=True), dp.copy_(hp, non_blocking=True)))
dev, _ = t(lambda: finalize(consume(tr, max_entries=1 << 62)))
ut = ColumnarTrace(tr.kind, tr.payload, tr.kernel_name, 0, tr.global_size, tr.local_size, tr.opcodes, [], tr.addr_stats)
devu, _ = t(lambda: finalize(consume(ut, max_entries=1 << 62)))
h2d_sync, _ = t(lambda: (hk.to("cuda"), hp.to("cuda")))
cons, acc = t(lambda: consume(ht, max_entries=1 << 62))
fin, _ = t(lambda: finalize(acc))
full, _ = t(lambda: finalize(consume(ht, max_entries=1 << 62)))
print(f"bare H2D {bare:.3f} ms | .to() H2D {h2d_sync:.3f} | device-resident consume+finalize {dev:.3f} "
      f"(untrusted {devu:.3f}) | host consume {cons:.3f} | finalize {fin:.3f} | host consume+finalize {full:.3f} ms")
