"""Multi-rank path through the CUDA engine: two ranks on one GPU, each running
dist.CudaBackend (shard ingest, device partition of addresses by owner,
owner-range memory partials) over its work-group shard.  The collectives are
gloo, staged through host memory (dist.comm_device), so no rank's kernel
waits on another rank's kernel.  The combined report must equal the
single-GPU report of the whole trace (and, for golden traces, the
reference's own report)."""

import os
import socket

import numpy as np
import pytest

from conftest import ROOT, assert_report_matches, golden_cases

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import torch.multiprocessing as mp  # noqa: E402

GOLDEN = ["wavefront_big", "sweep4", "hot_address", "random31337_3", "offgrid_groups", "branch_streams_per_group"]
SYNTH = [(1, 4096), (2, 8192), (3, 8192), (4, 2048), (5, 4096)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    from conftest import golden_cases as gc
    from paper_1805_04207_b200 import dist as D
    from paper_1805_04207_b200 import report_to_dict, synth
    from paper_1805_04207_b200.trace import K_WG_BEGIN, ColumnarTrace

    torch.cuda.set_device(0)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    backends = (D.CudaBackend(0), D.CudaBackend(0, force_compact=True))
    try:
        by_name = {c["name"]: (c, t) for c, t in gc()}
        for name in GOLDEN:
            c, tr = by_name[name]
            starts = np.nonzero(tr.kind == K_WG_BEGIN)[0]
            cuts = [0] + [int(starts[len(starts) * r // world]) for r in range(1, world)] + [tr.n_events]
            lo, hi = cuts[rank], cuts[rank + 1]
            shard = ColumnarTrace(torch.from_numpy(tr.kind[lo:hi].copy()).cuda(),
                                  torch.from_numpy(tr.payload[lo:hi].view(np.int64).copy()).cuda(),
                                  tr.kernel_name, tr.invocation, tr.global_size, tr.local_size, tr.opcodes,
                                  tr.extra_groups)
            for backend in backends:
                rep = D.sharded_report(backend, shard, lo, tr.kernel_name, tr.invocation, tr.global_size,
                                       tr.local_size, tr.opcodes)
                q.put((rank, name, report_to_dict(rep), D.LAST_EXCHANGE))
        for cfg, w in SYNTH:
            first, count = synth.shard_range(cfg, w, rank, world)
            shard = synth.device_trace(cfg, w, first=first, count=count)
            for backend in backends:
                rep = D.sharded_report(backend, shard, first, shard.kernel_name, 0, shard.global_size,
                                       shard.local_size, shard.opcodes)
                q.put((rank, f"C{cfg}", report_to_dict(rep), D.LAST_EXCHANGE))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_cuda_backend_matches_whole_trace(world):
    from paper_1805_04207_b200 import consume, finalize, report_to_dict, synth

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    n = 2 * world * (len(GOLDEN) + len(SYNTH))
    got = [q.get(timeout=300) for _ in range(n)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = {c["name"]: c["report"] for c, _ in golden_cases() if c["name"] in GOLDEN}
    for cfg, w in SYNTH:
        want[f"C{cfg}"] = report_to_dict(finalize(consume(synth.device_trace(cfg, w))))
    modes = set()
    for rank, name, rep, mode in got:
        assert_report_matches(rep, want[name])
        modes.add(mode)
    assert {"dense", "runs", "raw"} <= modes  # every address exchange ran through the CUDA engine


def _job_worker(port, q):
    """World 1 over NCCL: the engine's job mode (aiwc_ctx_set_comm) end to end --
    stats all-gather, dense chunk exchange or key-range owners, packed all-reduce,
    list all-gather, the C++ combine."""
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    from conftest import golden_cases as gc
    from paper_1805_04207_b200 import dist as D
    from paper_1805_04207_b200 import report_to_dict, synth
    from paper_1805_04207_b200.trace import ColumnarTrace

    torch.cuda.set_device(0)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    jobs = {"dense": D.NcclJob(0), "compact": D.NcclJob(0, dense_budget_bytes=1)}
    try:
        by_name = {c["name"]: (c, t) for c, t in gc()}
        for name in GOLDEN:
            c, tr = by_name[name]
            shard = ColumnarTrace(torch.from_numpy(tr.kind.copy()).cuda(),
                                  torch.from_numpy(tr.payload.view(np.int64).copy()).cuda(),
                                  tr.kernel_name, tr.invocation, tr.global_size, tr.local_size, tr.opcodes,
                                  tr.extra_groups)
            for mode, job in jobs.items():
                rep = job.report(shard, 0, tr.kernel_name, tr.invocation, tr.global_size, tr.local_size, tr.opcodes)
                q.put((mode, name, report_to_dict(rep)))
        for cfg, w in SYNTH:
            shard = synth.device_trace(cfg, w)
            for mode, job in jobs.items():
                rep = job.report(shard, 0, shard.kernel_name, 0, shard.global_size, shard.local_size, shard.opcodes)
                q.put((mode, f"C{cfg}", report_to_dict(rep)))
        q.put(("done", "", {}))
    finally:
        for job in jobs.values():
            job.close()
        dist.destroy_process_group()


def test_nccl_job_mode_matches_whole_trace():
    from paper_1805_04207_b200 import consume, finalize, report_to_dict, synth

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_job_worker, args=(_free_port(), q))
    p.start()
    got = []
    while True:
        item = q.get(timeout=300)
        if item[0] == "done":
            break
        got.append(item)
    p.join(timeout=60)
    assert p.exitcode == 0
    want = {c["name"]: c["report"] for c, _ in golden_cases() if c["name"] in GOLDEN}
    for cfg, w in SYNTH:
        want[f"C{cfg}"] = report_to_dict(finalize(consume(synth.device_trace(cfg, w))))
    assert len(got) == 2 * (len(GOLDEN) + len(SYNTH))
    for mode, name, rep in got:
        assert_report_matches(rep, want[name])
