"""Section timings of the multi-GPU shard path on one rank (NCCL, world 1): both address exchanges."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import torch, torch.distributed as dist
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29534", RANK="0", WORLD_SIZE="1")
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
from paper_1805_04207_b200 import synth, dist as D
T = {}
def tick(name, t0):
    torch.cuda.synchronize(); t1 = time.perf_counter(); T[name] = T.get(name, 0) + (t1 - t0) * 1e3; return t1
for cfg in [int(c) for c in (sys.argv[1:] or ["2", "3", "5"])]:
    tr = synth.device_trace(cfg)
    be = D.CudaBackend(0)
    for mode in ("raw", "runs"):
        T.clear()
        K = 3
        for it in range(K + 1):
            if it == 1: T.clear()
            t = time.perf_counter()
            sp = be.shard(tr, 0); t = tick("shard", t)
            stats = D.allreduce_stats(sp.addr_stats, None, be.device); t = tick("stats", t)
            km = D.key_map(stats, 1)
            lo, n_owned = km.owned(0)
            tm = sp.total_reads + sp.total_writes
            if mode == "raw":
                reads, writes, counts = be.partition(sp, km, 1); t = tick("partition", t)
                rr, nr = D.exchange(reads, counts[:1], None, be.device); rw, nw = D.exchange(writes, counts[1:], None, be.device); t = tick("exchange", t)
                mp = be.memory_partial(rr, nr, rw, nw, km, lo, n_owned, tm); t = tick("owner", t)
            else:
                runs, rc = be.partition_runs(sp, km, 1); t = tick("partition", t)
                recv, nwds = D.exchange(runs, [2 * c for c in rc], None, be.device); t = tick("exchange", t)
                mp = be.memory_partial_runs(recv, nwds // 2, km, lo, n_owned, tm); t = tick("owner", t)
        extra = f" runs={sum(rc)}" if mode == "runs" else ""
        print(f"C{cfg} {mode}", {k: round(v / K, 3) for k, v in T.items()}, f"total {sum(T.values())/K:.2f} ms{extra}", flush=True)
    del tr; torch.cuda.empty_cache()
dist.destroy_process_group()
