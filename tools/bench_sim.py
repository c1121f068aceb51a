"""Throughput of the device NDRange producer (simulate_trace) and of
producer + consume + finalize, on large launches of the reference's kernels
and a C2-shaped kmeans kernel.  CUDA-event timing after a warm-up; one JSON
line per kernel.

    python tools/bench_sim.py [--n 16777216]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

KMEANS = """kernel kmeans(a, b)
entry:
  mul r0, gid0, 8
  load r1, buf[a][r0]
  fmul r2, r1, r1
  add r0, r0, 1
  load r1, buf[a][r0]
  fmul r3, r1, r1
  add r0, r0, 1
  load r1, buf[a][r0]
  fmul r4, r1, r1
  add r0, r0, 1
  load r1, buf[a][r0]
  fmul r5, r1, r1
  fadd.x4 r6, r2, r3
  fadd.x4 r6, r6, r4
  store buf[b][gid0], r5
  ret
"""

SWEEP = "kernel sweep4(a)\nentry:\n  load r0, buf[a][gid0]\n  ret\n"
FLAGS = ("kernel flags(flags, out)\nentry:\n  load r0, buf[flags][gid0]\n  br r0, visit, skip\nvisit:\n"
         "  store buf[out][gid0], 1\n  jmp done\nskip:\n  jmp done\ndone:\n  ret\n")
# neighbour reads after a barrier inside each group: a dependence between work-items
# of one group -> group schedule (groups in parallel, each in the reference's order)
STAGES = ("kernel stages(a)\nentry:\n  mov r9, 0\n  sub r7, gid0, lid0\n  jmp body\nbody:\n  add r1, lid0, 1\n"
          "  rem r1, r1, lsz0\n  add r1, r1, r7\n  load r2, buf[a][gid0]\n  load r3, buf[a][r1]\n  add r4, r2, r3\n"
          "  store buf[a][gid0], r4\n  barrier\n  add r9, r9, 1\n  lt r8, r9, 8\n  br r8, body, done\ndone:\n  ret\n")
# a chain across groups (the reference's wavefront pattern) -> whole-launch sequential schedule
CHAIN = ("kernel chain(a)\nentry:\n  add r1, gid0, 1\n  load r2, buf[a][gid0]\n  add r2, r2, 1\n"
         "  store buf[a][r1], r2\n  ret\n")

import numpy as np  # noqa: E402

KERNELS = {
    "sweep4": (SWEEP, lambda n: {"a": np.arange(n)}, 64),
    "flags": (FLAGS, lambda n: {"flags": (np.arange(n) * 2654435761 >> 7) & 1, "out": np.zeros(n, np.int64)}, 64),
    "kmeans": (KMEANS, lambda n: {"a": np.arange(8 * n), "b": np.zeros(n, np.int64)}, 256),
    "stages(group)": (STAGES, lambda n: {"a": np.ones(n, np.int64)}, 256),
    "chain(seq)": (CHAIN, lambda n: {"a": np.ones(n + 1, np.int64)}, 256),
}


def main():
    import torch

    from paper_1805_04207_b200 import consume, finalize, ir, sim

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 22)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    for name, (src, bufs, local) in KERNELS.items():
        n = min(args.n, 1 << 16) if "(seq)" in name else (min(args.n, 1 << 18) if "(group)" in name else args.n)
        prog = ir.parse_kernel(src)
        t0 = time.time()
        cfg = sim.NDRangeConfig((n, 1, 1), (local, 1, 1),
                                {k: torch.from_numpy(np.ascontiguousarray(v, dtype=np.int64)).cuda()
                                 for k, v in bufs(n).items()})
        t_cfg = time.time() - t0
        tr = sim.simulate_trace(prog, cfg)  # warm-up
        torch.cuda.synchronize()
        ev = tr.n_events
        del tr
        times, e2e, plan, emit = [], [], [], []
        bases = sim._prepare(prog, cfg)
        for _ in range(args.reps):
            torch.cuda.synchronize()
            t = time.perf_counter()
            launch = sim._Launch(prog, cfg, bases, sim.DEFAULT_STEP_LIMIT, 0)
            schedule = launch.schedule
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            tr = launch.emit()
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            launch.close()
            plan.append(t1 - t)
            emit.append(t2 - t1)
            times.append(t2 - t)
            t = time.perf_counter()
            finalize(consume(tr, max_entries=1 << 40))
            torch.cuda.synchronize()
            e2e.append(times[-1] + time.perf_counter() - t)
            del tr
        best, beste = min(times), min(e2e)
        print(json.dumps({"kernel": name, "schedule": schedule, "work_items": n, "events": ev, "producer_s": round(best, 5),
                          "plan_s": round(min(plan), 5), "emit_s": round(min(emit), 5),
                          "producer_events_per_s": ev / best, "producer_plus_report_events_per_s": ev / beste,
                          "host_buffer_setup_s": round(t_cfg, 3)}), flush=True)


if __name__ == "__main__":
    main()
