"""Engine step on a C2 trace without declared totals / address statistics (a user's own columns)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_1805_04207_b200 import synth, consume, finalize
from paper_1805_04207_b200.trace import ColumnarTrace
for cfg in (2, 3):
    tr = synth.device_trace(cfg)
    plain = ColumnarTrace(tr.kind, tr.payload, tr.kernel_name, 0, tr.global_size, tr.local_size, tr.opcodes, [],
                          None, validated=True)
    for name, t in (("declared", tr), ("plain", plain)):
        for _ in range(3):
            finalize(consume(t, max_entries=1 << 40))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        K = 5
        for _ in range(K):
            finalize(consume(t, max_entries=1 << 40))
        torch.cuda.synchronize()
        print(f"C{cfg} {name}: {(time.perf_counter() - t0) / K * 1e3:.3f} ms", flush=True)
    del tr, plain; torch.cuda.empty_cache()
