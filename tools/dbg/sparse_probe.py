"""Sparse memory path cost: C2 with its addresses scattered over a 2^40-byte span."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_1805_04207_b200 import synth, consume, finalize
from paper_1805_04207_b200.trace import ColumnarTrace
tr = synth.device_trace(2)
k, p = tr.kind, tr.payload.clone()
mem = (k == 0x02) | (k == 0x04)
a = p[mem]
a = ((a * 0x9E3779B1) ^ (a >> 7)) & ((1 << 40) - 1) & ~3
p[mem] = a
sp = ColumnarTrace(k, p, tr.kernel_name, 0, tr.global_size, tr.local_size, tr.opcodes, [], None, validated=True)
for name, t in (("dense C2", tr), ("sparse C2", sp)):
    for _ in range(2):
        r = finalize(consume(t, max_entries=1 << 40))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        r = finalize(consume(t, max_entries=1 << 40))
    torch.cuda.synchronize()
    print(f"{name}: {(time.perf_counter() - t0) / 3 * 1e3:.2f} ms  footprint {r.total_memory_footprint} gmae {r.gmae}", flush=True)
