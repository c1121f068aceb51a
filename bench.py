"""Benchmark: trace events/s for the full AIWC metric vector (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]

One step = one pass of the hot path (aiwc_reset + aiwc_ingest + aiwc_finalize:
every report field) over one synthetic trace resident in HBM.  The N=1
workload is BASELINE configs[1] (C2, 256 M-event kmeans-like streaming trace,
2^23 work-items, local 256).  `value` is events/s with the trace already on
the device; `e2e` is the same metric through the public Python API
(`consume` + `finalize`) from pinned HOST columns, H2D and the result D2H
inside the timed region.  The trace (2.4 GB) is larger than L2, so no L2 flush
is needed between steps.

`--impl reference` times the reference algorithm's CPU restatement
(oracle/aiwc_oracle_mt.c; the Python reference cannot travel to the GPU box)
on all host threads, on a bounded prefix of the same trace, rank 0 only.  Its
input comes from the pure-numpy generator (oracle/synth_np.py), so that arm
never loads the product library; both arms print the identical `config`.

`--gpus N` (N>1) re-executes itself under torch.distributed.run with one rank
per GPU unless it already runs under torchrun.  Every rank processes its own
work-group shard: `--scaling weak` (default) of an N-times larger trace,
`--scaling strong` of the one fixed-size trace (e.g. `--config 3`, the 2 B-event
north_star target), and the per-rank reductions are combined over NCCL
(paper_1805_04207_b200/dist.py).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "trace events/sec (full AIWC metric vector)"
UNIT = "events/s"
ALG_BYTES_PER_EVENT = 9  # one kind byte + one payload u64


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fp:
            return json.load(fp)
    except OSError:
        return {}


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region (NVML, else nvidia-smi)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._nv = None
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _nvml_open(self) -> bool:
        try:
            import pynvml as nv

            nv.nvmlInit()
            self._nv = nv
            self._h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self._mx = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
            return True
        except Exception:
            self._nv = None
            return False

    def _sample_nvml(self) -> None:
        nv = self._nv
        bits = (0x8, 0x40, 0x20, 0x4)  # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
        try:
            sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            self.samples.append([str(sm), str(self._mx)] + ["Active" if r & b else "Not Active" for b in bits])
        except Exception:
            pass

    def _run_nvml(self) -> bool:
        """NVML sampling every 2 ms (short timed regions still get samples: one is
        also taken synchronously on entry and on exit)."""
        if self._nv is None:
            return False
        while not self._stop.is_set():
            self._sample_nvml()
            self._stop.wait(0.002)
        return True

    def _run(self):
        if self._run_nvml():
            return
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                vals = [v.strip() for v in out.stdout.strip().split(",")]
                if len(vals) == 6:
                    self.samples.append(vals)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        if self._nvml_open():
            self._sample_nvml()
        self._t.start()
        return self

    def __exit__(self, *a):
        if self._nv is not None:
            self._sample_nvml()
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def _dist_env():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


# ---------------------------------------------------------------------------
# reference arm: the C restatement of the reference path on the host cores
# ---------------------------------------------------------------------------
def host_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return max(1, os.cpu_count() or 1)


def reference_sample(cfg: int, total_wi: int, args, threads: int):
    """A bounded prefix of whole work-groups of the same trace (a valid trace),
    sized for ~10 s of CPU work per step: 2^21 work-items per 2 threads.  Built
    by the pure-numpy generator (oracle/synth_np.py, bit-identical to the device
    generator) so the reference arm never loads the product library."""
    from oracle import synth_np

    lv = synth_np.LOCAL[cfg]
    sample_wi = min(total_wi, args.ref_sample_wi * max(1, threads // 2))
    sample_wi -= sample_wi % lv
    kind, payload = synth_np.trace(cfg, sample_wi)
    if sample_wi < total_wi:
        # a prefix of whole work-groups is a valid trace once it is closed by kernel_end
        kind[-1], payload[-1] = synth_np.K_KE, 0
    return sample_wi, kind, payload


def bench_config(cfg: int, world: int, w: int, scaling: str) -> dict:
    """The workload both arms report (identical dict: the driver compares them)."""
    from oracle import synth_np

    total_wi = world * w if scaling == "weak" else w
    n_total = synth_np.n_events(cfg, total_wi)
    return {"workload": f"C{cfg} {synth_np.NAMES[cfg]}: {total_wi} work-items ({n_total} events), "
                        f"local {synth_np.LOCAL[cfg]}",
            "events": n_total, "work_items": total_wi, "scaling": scaling,
            "l2": "trace (9 B/event) larger than the 126 MB L2; no flush needed" if 9 * n_total > (252 << 20) else
                  "trace smaller than L2",
            "parallelism": "replica (N=1)" if world == 1 else f"work-group shards x{world} ({scaling} scaling)"}


def run_reference(args) -> None:
    world, rank, _ = _dist_env()
    if rank != 0:
        return
    from oracle import oracle, synth_np

    oracle.build()
    cfg = args.config
    w = args.work_items or synth_np.FULL_WORK_ITEMS[cfg]
    config = bench_config(cfg, world, w, args.scaling)
    threads = host_threads()
    sample_wi, kind, payload = reference_sample(cfg, config["work_items"], args, threads)
    n = int(kind.shape[0])
    run = lambda: oracle.run(kind, payload, kernel=synth_np.NAMES[cfg], invocation=0,  # noqa: E731
                             n_opcodes=len(synth_np.OPCODES[cfg]), threads=threads)
    for _ in range(args.warmup):
        run()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    dt = statistics.median(times)
    v = n / dt
    whole = sample_wi == config["work_items"]
    sample = (f"{'the whole trace' if whole else f'first {sample_wi} work-items'} of C{cfg} ({n} events, numpy "
              f"generator oracle/synth_np.py); oracle/aiwc_oracle_mt.c: consume+finalize restatement on {threads} "
              "threads (work-group shards + address-owner merge, SURVEY 8d(ii)); median step")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "u8+u64 events, fp64 entropies", "data": "synthetic",
        "config": config,
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def _timed(step, steps, stream, dev, world, local):
    """Barrier + sync, K steps between CUDA events on `stream`, max over ranks."""
    import torch

    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        start.record(stream)
        for _ in range(steps):
            step()
        end.record(stream)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
    ms = start.elapsed_time(end)
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([ms, wall], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, wall = (float(v) for v in t.tolist())
    return ms, wall, clk.summary()


def _timed_lanes(lane_step, streams, steps, phases, kernels, stream, local, world=1, dev=None):
    """K steps split over len(streams) host threads (one engine context and CUDA
    stream each), between CUDA events on `stream` that every lane stream joins;
    barrier before, max over ranks after."""
    import torch

    from paper_1805_04207_b200 import _native

    n = len(streams)
    share = [steps // n + (1 if i < steps % n else 0) for i in range(n)]
    out = [[] for _ in range(n)]
    errs = []

    def run(i):
        try:
            with torch.cuda.stream(streams[i]):
                for _ in range(share[i]):
                    out[i].append(lane_step(i))
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        start.record(stream)
        for s in streams:
            s.wait_event(start)
        th = [threading.Thread(target=run, args=(i,)) for i in range(n)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for s in streams:
            stream.wait_stream(s)
        end.record(stream)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
    if errs:
        raise errs[0]
    for res in out:
        for ph, k in res:
            for i, p in enumerate(_native.PHASES):
                phases[p].append(ph[i])
            kernels[0] += k
    ms = start.elapsed_time(end)
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([ms, wall], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, wall = (float(v) for v in t.tolist())
    return ms, wall, clk.summary()


def run_ours(args) -> None:
    import torch

    from paper_1805_04207_b200 import _native, consume, finalize, synth
    from paper_1805_04207_b200 import dist as D
    from paper_1805_04207_b200.metrics import trace_info
    from paper_1805_04207_b200.trace import ColumnarTrace

    world, rank, local = _dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # the multi-GPU (work-group shard) path; AIWC_BENCH_SHARDED=1 forces it at one
    # rank under torchrun (a single-GPU check of the N>1 code path)
    sharded = world > 1 or os.environ.get("AIWC_BENCH_SHARDED") == "1"
    if sharded:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    cfg = args.config
    w = args.work_items or synth.FULL_WORK_ITEMS[cfg]
    config = bench_config(cfg, world, w, args.scaling)
    # weak scaling: the job is one world*w work-item trace, strong scaling one w
    # work-item trace; rank r owns the contiguous work-group shard
    # synth.shard_range(cfg, total_wi, r, world) of it
    total_wi = config["work_items"]
    first, count = synth.shard_range(cfg, total_wi, rank, world)
    tr = synth.device_trace(cfg, total_wi, first=first, count=count)
    n_total = config["events"]
    stream = torch.cuda.current_stream(dev)

    n_streams = max(1, args.streams if args.streams is not None else (3 if world == 1 else 1))
    if not sharded:
        # one engine context per CUDA stream; with several, concurrent host threads
        # each push whole trace -> report steps (the reference allows distinct
        # streams to run concurrently, pkg/README.md:192-193), so one stream's
        # small kernels and host round trip overlap another stream's ingest.
        # Every lane reads its OWN copy of the trace (no cross-lane L2 reuse).
        # the columns are treated as untrusted: every step also checks StreamChecker's
        # invariants inside the pass (barrier / resume traces included; the separate
        # full validator -- which only locates a violation -- is reported as validate_ms)
        info = trace_info(tr, check=not args.no_stream_check)
        lanes = []
        for i in range(n_streams):
            cs = stream if i == 0 else torch.cuda.Stream(dev)
            ltr = tr if i == 0 else synth.device_trace(cfg, total_wi, first=first, count=count)
            lanes.append((_native.Context(local, flags=_native.OPT_NO_CONSERVATION | _native.OPT_TIMING), cs,
                          _native.Result(), ctypes.c_void_p(ltr.kind.data_ptr()),
                          ctypes.c_void_p(ltr.payload.data_ptr()), ltr))

        def lane_step(i):
            ctx, cs, r, kptr, pptr, _ = lanes[i]
            lib, sptr = ctx.lib, ctypes.c_void_p(cs.cuda_stream)
            ctx.check(lib.aiwc_reset(ctx.h))
            ctx.check(lib.aiwc_ingest(ctx.h, kptr, pptr, ctypes.byref(info), sptr))
            ctx.check(lib.aiwc_finalize(ctx.h, ctypes.byref(r), sptr))
            return list(r.phase_ms), r.kernels_launched

        def step():
            return lane_step(0)
    else:
        # one engine context, CUDA stream, NCCL communicator (process group) and copy of
        # the shard per lane: the lanes' collectives run concurrently on their own
        # communicators, like the single-GPU lanes' whole steps
        # job mode: the engine runs every collective itself over its own NCCL
        # communicator (aiwc_ctx_set_comm); AIWC_BENCH_PYDIST=1 drives the same
        # exchange from Python instead (dist.sharded_result, one collective per call)
        pydist = os.environ.get("AIWC_BENCH_PYDIST") == "1"
        sh_lanes = []
        for i in range(n_streams):
            cs = stream if i == 0 else torch.cuda.Stream(dev)
            ltr = tr if i == 0 else synth.device_trace(cfg, total_wi, first=first, count=count)
            g = None if i == 0 else dist.new_group(list(range(world)))
            eng = D.CudaBackend(local, timing=True) if pydist else D.NcclJob(local, group=g, timing=True)
            sh_lanes.append((eng, cs, ltr, g))
        backend = sh_lanes[0][0]

        def lane_step(i):
            eng, _, ltr, g = sh_lanes[i]
            before = eng.launches
            if pydist:
                D.sharded_result(eng, ltr, first, group=g)
            else:
                eng.result(ltr, first)
            return list(eng.last_phase_ms), eng.launches - before

        def step():
            return lane_step(0)

    phases = {p: [] for p in _native.PHASES}
    kernels = [0]

    def timed_step():
        ph, k = step()
        for i, p in enumerate(_native.PHASES):
            phases[p].append(ph[i])
        kernels[0] += k

    for _ in range(max(3, args.warmup)):
        step()
    if n_streams > 1:
        for i in range(1, n_streams):
            for _ in range(max(3, args.warmup)):
                lane_step(i)
        lane_streams = [c[1] for c in (lanes if not sharded else sh_lanes)]
        ms, _, clocks = _timed_lanes(lane_step, lane_streams, args.steps, {p: [] for p in phases}, kernels,
                                     stream, local, world, dev)
        # per-kernel (phase) times for the roofline come from a separate single-stream
        # run: overlapping streams stretch each kernel's event-to-event duration
        k_timed = kernels[0]
        _timed(timed_step, args.steps, stream, dev, world, local)
        kernels[0] = k_timed
    else:
        ms, _, clocks = _timed(timed_step, args.steps, stream, dev, world, local)
    ms_step = ms / args.steps
    value = n_total / (ms_step / 1e3)
    phase_med = {p: statistics.median(v) for p, v in phases.items()}

    # device stream validation of the same columns (what consume() runs for untrusted columnar input)
    validate_ms = None
    if not sharded:
        vctx = _native.Context(local)
        vout = _native.Violation()
        i64x3 = ctypes.c_int64 * 3
        vinfo = trace_info(tr)
        gsz, lsz = i64x3(*[int(x) for x in tr.global_size]), i64x3(*[int(x) for x in tr.local_size])
        vrun = lambda: vctx.check(vctx.lib.aiwc_validate(vctx.h, ctypes.c_void_p(tr.kind.data_ptr()),  # noqa: E731
                                                         ctypes.c_void_p(tr.payload.data_ptr()), ctypes.byref(vinfo),
                                                         gsz, lsz, ctypes.byref(vout),
                                                         ctypes.c_void_p(stream.cuda_stream)))
        vrun()
        v_ms, _, _ = _timed(vrun, 3, stream, dev, 1, local)
        validate_ms = v_ms / 3
        vctx.close()

    # context for the roofline: the same ingest without the in-pass stream check
    unchecked_ingest_ms = None
    if not sharded and not args.no_stream_check:
        uinfo = trace_info(tr, check=False)
        uctx, ucs, _, ukptr, upptr, _ = lanes[0]
        ur = _native.Result()  # (lane 0's own result keeps the checked step's certification)
        ui = _native.PHASES.index("ingest")
        u_ph = []

        def ustep():
            usptr = ctypes.c_void_p(ucs.cuda_stream)
            uctx.check(uctx.lib.aiwc_reset(uctx.h))
            uctx.check(uctx.lib.aiwc_ingest(uctx.h, ukptr, upptr, ctypes.byref(uinfo), usptr))
            uctx.check(uctx.lib.aiwc_finalize(uctx.h, ctypes.byref(ur), usptr))
            u_ph.append(ur.phase_ms[ui])
        for _ in range(3):
            ustep()
        u_ph.clear()
        for _ in range(args.steps):
            ustep()
        torch.cuda.synchronize()
        unchecked_ingest_ms = statistics.median(u_ph)

    if args.no_e2e:
        if rank == 0:
            print(json.dumps({"ms_per_step": ms_step, "value": value, "phases_ms": phase_med,
                              "validate_ms": validate_ms, "shard_sections_ms": dict(D.LAST_PROFILE),
                              "binned": lanes[0][2].binned_accesses if not sharded else None}), flush=True)
        if sharded:
            dist.destroy_process_group()
        return
    # ---- e2e: the public API from pinned host columns (H2D + result D2H inside) ----
    hk = torch.empty(count, dtype=torch.uint8, pin_memory=True)
    hp = torch.empty(count, dtype=torch.int64, pin_memory=True)
    hk.copy_(tr.kind)
    hp.copy_(tr.payload)
    host_tr = ColumnarTrace(hk, hp, tr.kernel_name, 0, tr.global_size, tr.local_size, tr.opcodes, [], tr.addr_stats)
    if not sharded:
        def e2e_step():
            return finalize(consume(host_tr, max_entries=1 << 62, device=local))
    elif pydist:
        def e2e_step():
            return D.sharded_report(backend, host_tr, first, tr.kernel_name, 0, tr.global_size, tr.local_size,
                                    tr.opcodes)
    else:
        def e2e_step():
            return backend.report(host_tr, first, tr.kernel_name, 0, tr.global_size, tr.local_size, tr.opcodes)
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    out = {}
    for _ in range(2):
        out["rep"] = e2e_step()
    e_ms, e_wall, _ = _timed(lambda: out.__setitem__("rep", e2e_step()), e2e_steps, stream, dev, world, local)
    rep = out["rep"]
    e2e_ms = max(e_ms, e_wall) / e2e_steps
    e2e_value = n_total / (e2e_ms / 1e3)
    # The e2e ceiling is the host link: time a bare pinned-host -> device copy of the same
    # two columns (no compute) so the line says how close the API path gets to it.
    dk = torch.empty(count, dtype=torch.uint8, device=dev)
    dp = torch.empty(count, dtype=torch.int64, device=dev)

    def bare_h2d():
        dk.copy_(hk, non_blocking=True)
        dp.copy_(hp, non_blocking=True)
    bare_h2d()
    h_ms, _, _ = _timed(bare_h2d, 3, torch.cuda.current_stream(dev), dev, 1, local)
    h2d_peak = 9 * count / (h_ms / 3 / 1e3) / 1e9
    del dk, dp

    # ---- roofline of the dominant kernel (the ingest pass), per rank ----
    peaks = measured_peaks()
    peak = peaks.get("hbm_gbs")
    peak_src = "measured" if peak else "fallback"
    peak = peak or 6650.0
    ingest_ms = phase_med["ingest"]
    achieved = ALG_BYTES_PER_EVENT * count / (ingest_ms / 1e3) / 1e9
    step_alg = ALG_BYTES_PER_EVENT * count / (ms_step / 1e3) / 1e9
    traffic, traffic_src = ncu_traffic(cfg) if not sharded else (None, None)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, total_wi, args)
    if rank == 0:
        agg = ALG_BYTES_PER_EVENT * n_total / (ms_step / 1e3) / 1e9
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "u8+u64 events, fp64 entropies",
            "data": "synthetic", "config": config,
            "lanes": {"events_per_rank": count, "streams": n_streams,
                      "how": f"{n_streams} concurrent trace streams (engine ctx + CUDA stream + own copy of the "
                             "trace each)" if not sharded else
                             f"{n_streams} concurrent shard streams per rank (engine ctx with its own NCCL "
                             "communicator + CUDA stream + own copy of the shard each); collectives inside the engine; "
                             "dense exchange of 1024-key chunks"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 9 * count,
                    "d2h_bytes_per_step": lanes[0][2].d2h_bytes if not sharded else backend.last_d2h,
                    "ms_per_step": e2e_ms,
                    "h2d_gbs": 9 * count / (e2e_ms / 1e3) / 1e9, "bare_h2d_gbs": h2d_peak,
                    "link_frac": (9 * count / (e2e_ms / 1e3) / 1e9) / h2d_peak,
                    "path": "consume(ColumnarTrace on pinned host)+finalize" if not sharded else
                            "dist.NcclJob.report(pinned host shard): aiwc_ingest_host + aiwc_finalize in job mode"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_unit": "bytes per launch (ncu dram read+write)",
                         "traffic_source": traffic_src, "alg_bytes": ALG_BYTES_PER_EVENT * count,
                         "kernel": "aiwc::ingest_kernel",
                         "peak_source": peak_src, "alg_bytes_per_event": ALG_BYTES_PER_EVENT,
                         "step_alg_gbs": step_alg, "step_frac": step_alg / peak,
                         "aggregate_frac": agg / (world * peak),
                         "frac_without_stream_check": (ALG_BYTES_PER_EVENT * count / (unchecked_ingest_ms / 1e3) / 1e9)
                         / peak if unchecked_ingest_ms else None,
                         "stream_check_ms": ingest_ms - unchecked_ingest_ms if unchecked_ingest_ms else None},
            "phases_ms": phase_med,
            "validate_ms": validate_ms,
            "stream_check": {"in_pass": not sharded, "certified": bool(lanes[0][2].stream_checked) if not sharded else None,
                             "full_validator_ms": validate_ms,
                             "note": "every timed single-GPU step checks StreamChecker's invariants inside the pass "
                                     "(trace.py:289-424), barrier / resume rules included; the separate device "
                                     "validator (full_validator_ms) only locates a violation"},
            "gpu_launches": kernels[0],
            "clocks": clocks,
            "cpu_baseline": cpu,
            "report_check": {"total_memory_footprint": rep.total_memory_footprint, "gmae": rep.gmae,
                             "footprint_90": rep.footprint_90},
        }
        print(json.dumps(line), flush=True)
    if sharded:
        dist.destroy_process_group()


def ncu_traffic(cfg: int):
    """DRAM bytes (read + write) per launch of the ingest kernel on this config, from the
    committed `ncu --set full` capture (tools/ncu_traffic.py), or None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", f"ncu_traffic_C{cfg}.json")
    try:
        with open(path, encoding="utf-8") as fp:
            d = json.load(fp)
        return d["traffic_bytes"], d.get("source")
    except (OSError, ValueError, KeyError):
        return None, None


def cpu_baseline(cfg, total_wi, args):
    """Oracle (C restatement of the reference path) on all host threads, on a
    bounded prefix of the same trace, rank 0 only (input from the numpy generator)."""
    from oracle import oracle, synth_np

    try:
        oracle.build()
        threads = host_threads()
        sample_wi, kind, payload = reference_sample(cfg, total_wi, args, threads)
        run = lambda: oracle.run(kind, payload, kernel=synth_np.NAMES[cfg], invocation=0,  # noqa: E731
                                 n_opcodes=len(synth_np.OPCODES[cfg]), threads=threads)
        run()
        t0 = time.perf_counter()
        run()
        dt = time.perf_counter() - t0
        return {"value": kind.shape[0] / dt, "unit": UNIT, "cores": threads, "kind": "port",
                "sample": f"{'whole trace' if sample_wi == total_wi else f'first {sample_wi} work-items'} of C{cfg} "
                          f"({kind.shape[0]} events), oracle/aiwc_oracle_mt.c on {threads} threads"}
    except Exception as exc:  # pragma: no cover
        return {"value": None, "unit": UNIT, "cores": None, "kind": "port", "sample": f"failed: {exc}"}


def spawn_ranks(n: int) -> None:
    """`bench.py --gpus N` outside torchrun: re-exec under torch.distributed.run with
    one rank per GPU (127.0.0.1 rendezvous); NCCL prints its communicator lines."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execve(sys.executable, cmd, env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--work-items", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--ref-sample-wi", type=int, default=1 << 21)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N>1: weak = every rank a full-size shard (N-times larger trace); strong = one fixed trace")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--streams", type=int, default=None,
                    help="engine contexts / CUDA streams with whole steps in flight concurrently (default 3 at "
                         "N=1; 1 at N>1, where each would add an NCCL communicator driven from its own thread)")
    ap.add_argument("--no-e2e", action="store_true", help="device-resident timing only (profiling runs)")
    ap.add_argument("--no-stream-check", action="store_true", help="measurement: steps without the in-pass checks")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args.gpus)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
