import time, sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1805_04207_b200 import consume, finalize, synth
for cfg, w in [(2, None), (1, None)]:
    tr = synth.device_trace(cfg, w)
    for _ in range(3):
        finalize(consume(tr, max_entries=1 << 40))
    torch.cuda.synchronize()
    t = time.perf_counter(); K = 20
    for _ in range(K):
        r = finalize(consume(tr, max_entries=1 << 40))
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / K
    # consume only
    t = time.perf_counter()
    for _ in range(K):
        a = consume(tr, max_entries=1 << 40)
    torch.cuda.synchronize()
    dc = (time.perf_counter() - t) / K
    t = time.perf_counter()
    for _ in range(K):
        r = finalize(a)
    df = (time.perf_counter() - t) / K
    print(f"C{cfg} consume+finalize {dt*1e3:.3f} ms  consume {dc*1e3:.3f} ms  finalize {df*1e3:.3f} ms")
