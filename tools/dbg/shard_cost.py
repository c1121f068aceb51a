"""Per-rank cost of the multi-GPU shard path, measured with world_size 1 (NCCL on one GPU)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, torch.distributed as dist
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533", RANK="0", WORLD_SIZE="1")
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
from paper_1805_04207_b200 import synth, dist as D
for cfg in [2, 3, 5]:
    tr = synth.device_trace(cfg)
    be = D.CudaBackend(0, timing=True)
    for _ in range(2):
        D.sharded_result(be, tr, 0)
    torch.cuda.synchronize()
    K = 5
    t = time.perf_counter()
    for _ in range(K):
        D.sharded_result(be, tr, 0)
    torch.cuda.synchronize()
    print(f"C{cfg} shard path {1e3*(time.perf_counter()-t)/K:.2f} ms  phases {[round(x,3) for x in be.last_phase_ms]}", flush=True)
    del tr
    torch.cuda.empty_cache()
dist.destroy_process_group()
