"""One profiled step per workload, for `ncu --profile-from-start off` captures of
EVERY kernel the step launches (warm-up steps run outside the profiled range).

usage: python tools/prof_step.py WORKLOAD
  C1..C5       consume + finalize of the synthetic config (device-resident, trusted)
  validate2    aiwc_validate of C2 (the device StreamChecker)
  sparse2      C2 with addresses scattered over 2^40 bytes (the sort path)
  regions2     C2 with its two buffers 2^44 bytes apart (region compaction)
  job2         C2 through the multi-GPU job mode at world 1 (NCCL, dense chunk exchange)
  sim          the device NDRange producer on the bundled kmeans kernel
"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1805_04207_b200 import consume, finalize, synth  # noqa: E402
from paper_1805_04207_b200.trace import ColumnarTrace  # noqa: E402


def scattered(tr, bits=40):
    k, p = tr.kind, tr.payload.clone()
    mem = (k == 0x02) | (k == 0x04)
    a = p[mem]
    p[mem] = ((a * 0x9E3779B1) ^ (a >> 7)) & ((1 << bits) - 1) & ~3
    return ColumnarTrace(k, p, tr.kernel_name, 0, tr.global_size, tr.local_size, tr.opcodes, [], None, validated=True)


def far_buffers(tr):
    k, p = tr.kind, tr.payload.clone()
    mem = (k == 0x02) | (k == 0x04)
    a = p[mem]
    p[mem] = torch.where(a >= (1 << 28), a + (1 << 44), a)
    return ColumnarTrace(k, p, tr.kernel_name, 0, tr.global_size, tr.local_size, tr.opcodes, [], None, validated=True)


def main():
    w = sys.argv[1]
    if w.startswith("C"):
        tr = synth.device_trace(int(w[1:]))
        step = lambda: finalize(consume(tr, max_entries=1 << 62))  # noqa: E731
    elif w == "validate2":
        from paper_1805_04207_b200.metrics import validate_columnar

        tr = synth.device_trace(2)
        step = lambda: validate_columnar(tr)  # noqa: E731
    elif w == "sparse2":
        tr = scattered(synth.device_trace(2))
        step = lambda: finalize(consume(tr, max_entries=1 << 62))  # noqa: E731
    elif w == "regions2":
        tr = far_buffers(synth.device_trace(2))
        step = lambda: finalize(consume(tr, max_entries=1 << 62))  # noqa: E731
    elif w == "job2":
        import torch.distributed as dist

        from paper_1805_04207_b200 import dist as D

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29577", RANK="0", WORLD_SIZE="1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
        tr = synth.device_trace(2)
        job = D.NcclJob(0)
        step = lambda: job.result(tr, 0)  # noqa: E731
    elif w == "sim":
        import numpy as np

        from paper_1805_04207_b200 import ir, sim
        from tools.bench_sim import KERNELS

        src, bufs, local = KERNELS["kmeans"]
        n = 1 << 22
        prog = ir.parse_kernel(src)
        cfg = sim.NDRangeConfig((n, 1, 1), (local, 1, 1),
                                {k: torch.from_numpy(np.ascontiguousarray(v, dtype=np.int64)).cuda()
                                 for k, v in bufs(n).items()})
        step = lambda: sim.simulate_trace(prog, cfg)  # noqa: E731
    else:
        raise SystemExit(f"unknown workload {w}")
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    step()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(f"profiled one step of {w}")


if __name__ == "__main__":
    main()
