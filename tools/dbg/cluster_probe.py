"""C2 with its two buffers 2^44 bytes apart (region compaction) vs the compact original."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_1805_04207_b200 import synth, consume, finalize
from paper_1805_04207_b200.trace import ColumnarTrace
tr = synth.device_trace(2)
k, p = tr.kind, tr.payload.clone()
st = (k == 0x04)
p[st] = p[st] + (1 << 44)   # the store buffer far away
far = ColumnarTrace(k, p, tr.kernel_name, 0, tr.global_size, tr.local_size, tr.opcodes, [], None, validated=True)
for name, t in (("compact C2", tr), ("C2, buffers 2^44 apart", far)):
    for _ in range(2):
        r = finalize(consume(t, max_entries=1 << 40))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        r = finalize(consume(t, max_entries=1 << 40))
    torch.cuda.synchronize()
    print(f"{name}: {(time.perf_counter() - t0) / 3 * 1e3:.2f} ms  footprint {r.total_memory_footprint} gmae {r.gmae} lmae9 {r.lmae[9]}", flush=True)
