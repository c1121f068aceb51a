"""Drop-in ``consume`` / ``finalize`` / ``merge_accumulators`` backed by the B200 engine.

Mirrors ``pkg/src/aiwc/metrics.py`` (names, arguments, exceptions, report
fields).  All O(events) work -- every histogram, address set, segment
statistic and branch pattern table -- runs in libaiwc_b200.so on the GPU; this
module only moves the trace in, and turns the engine's exact integers into
report reals with the reference's own expressions (``metrics.py:287-386``), so
ratios, means and the SIMD statistics are bit-identical to the reference.

``consume`` accepts either an iterable of TraceEvent objects (encoded to
columns by the native walker, which also runs the reference's stream
validation) or a ``ColumnarTrace`` whose columns are numpy arrays or torch
tensors (host or CUDA; CUDA columns are processed in place).
"""

from __future__ import annotations

import ctypes
import math
import os
import threading
from collections import Counter
from dataclasses import dataclass, field
from typing import Iterable, NamedTuple

import numpy as np

from . import _native
from .errors import AiwcError, EmptySample, IncompatibleReports, InvalidStream, TraceTooLarge
from .fields import FIELDS, materialize, merge_fields
from .report import AiwcReport, round12
from .trace import ColumnarTrace

MEM_CAP_ENV = "AIWC_MEM_CAP_BYTES"
BYTES_PER_ENTRY = 64
DEFAULT_MEM_CAP_BYTES = 1 << 30


def default_entry_cap() -> int:
    """Entry cap from AIWC_MEM_CAP_BYTES, same rule as the reference (metrics.py:54-57)."""
    raw = os.environ.get(MEM_CAP_ENV)
    cap_bytes = int(raw) if raw else DEFAULT_MEM_CAP_BYTES
    return max(1, cap_bytes // BYTES_PER_ENTRY)


# ---------------------------------------------------------------------------
# engine results
# ---------------------------------------------------------------------------
@dataclass
class EngineResult:
    """Exact integers + unrounded entropies returned by aiwc_finalize."""

    n_events: int
    total_instructions: int
    work_items: int
    barriers_hit: int
    opcode_coverage: int
    itb: tuple  # (n, min, max, sum, mid_lo, mid_hi)
    ipt: tuple
    total_reads: int
    total_writes: int
    unique_reads: int
    unique_writes: int
    footprint: int
    footprint_90: int
    gmae: float
    lmae: list
    branch_executions: int
    branch_observations: int
    branch_excluded: int
    branch_90: int
    yokota: float
    linear: float
    entries: int
    opcode_counts: list
    widths: list  # [(width, count)] first-seen order
    sites: list   # [(site, executions)] ascending site
    used_dense_table: bool
    kernels_launched: int
    binned_accesses: int = 0
    stream_checked: bool = False
    state: object = None  # EngineState for a state merge (merge_accumulators), or None


def _dist(d) -> tuple:
    return (d.n, d.min, d.max, d.sum, d.mid_lo, d.mid_hi)


def _copy_result(r: _native.Result) -> EngineResult:
    return EngineResult(
        n_events=r.n_events, total_instructions=r.total_instructions, work_items=r.work_items,
        barriers_hit=r.barriers_hit, opcode_coverage=r.opcode_coverage, itb=_dist(r.itb), ipt=_dist(r.ipt),
        total_reads=r.total_reads, total_writes=r.total_writes, unique_reads=r.unique_reads,
        unique_writes=r.unique_writes, footprint=r.footprint, footprint_90=r.footprint_90,
        gmae=r.gmae, lmae=list(r.lmae), branch_executions=r.branch_executions,
        branch_observations=r.branch_observations, branch_excluded=r.branch_excluded, branch_90=r.branch_90,
        yokota=r.yokota, linear=r.linear, entries=r.entries,
        opcode_counts=[r.opcode_counts[i] for i in range(r.n_opcodes)],
        widths=[(r.width_values[i], r.width_counts[i]) for i in range(r.n_widths)],
        sites=[(r.site_ids[i], r.site_counts[i]) for i in range(r.n_site_list)],
        used_dense_table=bool(r.used_dense_table), kernels_launched=r.kernels_launched,
        binned_accesses=r.binned_accesses,
    )


_pool: dict[int, list] = {}
_pool_lock = threading.Lock()


def _get_ctx(device: int) -> _native.Context:
    with _pool_lock:
        free = _pool.setdefault(device, [])
        if free:
            return free.pop()
    return _native.Context(device)


def _put_ctx(ctx: _native.Context) -> None:
    with _pool_lock:
        _pool.setdefault(ctx.device, []).append(ctx)


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def trace_info(tr: ColumnarTrace, check: bool = False) -> _native.TraceInfo:
    info = _native.TraceInfo()
    info.check_stream = 1 if check else 0
    info.n_events = tr.n_events
    info.local_volume = max(1, tr.local_volume)
    info.n_opcodes = len(tr.opcodes)
    if tr.addr_stats is not None:
        info.has_addr_stats = 1
        info.addr_min, info.addr_max, info.addr_and, info.addr_or = (int(v) for v in tr.addr_stats)
    if tr.class_counts is not None:
        info.has_counts = 1
        (info.n_instr, info.n_reads, info.n_writes, info.n_branches, info.n_groups,
         info.any_barrier_or_resume) = (int(v) for v in tr.class_counts)
    return info


def ingest_columns(ctx, tr: ColumnarTrace, check: bool = False, export: bool = False):
    """aiwc_ingest (device columns) or aiwc_ingest_host (host columns) of one
    columnar trace into ctx; returns the stream handle the work was queued on.
    check: the pass also checks StreamChecker's invariants (untrusted columns)."""
    kind, payload = tr.kind, tr.payload
    lib = ctx.lib
    info = trace_info(tr, check)
    info.export_state = 1 if export else 0
    if _is_torch(kind) and kind.is_cuda:
        import torch

        if kind.dtype != torch.uint8 or payload.dtype not in (torch.uint64, torch.int64):
            raise AiwcError("CUDA columns must be uint8 kind and (u)int64 payload tensors")
        kind = kind.contiguous()
        payload = payload.contiguous()
        if kind.data_ptr() % 16:
            kind = kind.clone()
        if payload.data_ptr() % 16:
            payload = payload.clone()
        stream = torch.cuda.current_stream(kind.device).cuda_stream
        ctx.check(lib.aiwc_ingest(ctx.h, ctypes.c_void_p(kind.data_ptr()), ctypes.c_void_p(payload.data_ptr()),
                                  ctypes.byref(info), ctypes.c_void_p(stream)))
        return stream
    if _is_torch(kind):
        kind, payload = kind.numpy(), payload.numpy()
    kind = np.ascontiguousarray(kind, dtype=np.uint8)
    payload = np.ascontiguousarray(payload).view(np.uint64)
    ctx.check(lib.aiwc_ingest_host(ctx.h, kind.ctypes.data_as(ctypes.c_void_p),
                                   payload.ctypes.data_as(ctypes.c_void_p), ctypes.byref(info), None))
    return None


def _device_columns(tr: ColumnarTrace, device: int) -> ColumnarTrace:
    """The trace with its columns in CUDA memory on `device` (no copy if already there)."""
    import torch

    kind, payload = tr.kind, tr.payload
    if _is_torch(kind) and kind.is_cuda:
        return tr
    dev = torch.device("cuda", device)
    k = torch.as_tensor(np.ascontiguousarray(kind, dtype=np.uint8) if not _is_torch(kind) else kind).to(dev)
    pl = payload if _is_torch(payload) else torch.from_numpy(np.ascontiguousarray(payload).view(np.int64))
    return ColumnarTrace(k, pl.to(dev), tr.kernel_name, tr.invocation, tr.global_size, tr.local_size, tr.opcodes,
                         tr.extra_groups, tr.addr_stats, tr.validated, tr.class_counts)


def validate_columnar(tr: ColumnarTrace, device: int | None = None) -> tuple | None:
    """First stream violation (event_index, rule, detail) of a columnar trace, as
    StreamChecker would report it for tr.iter_events() (trace.py:289-424), or
    None.  Runs on the device (aiwc_validate); work-groups of more than 1024
    work-items are checked by the native host walker instead."""
    kind = tr.kind
    if device is None:
        device = kind.device.index if (_is_torch(kind) and kind.is_cuda) else _default_device()
    lsz = tuple(int(x) for x in tr.local_size)
    if lsz[0] * lsz[1] * lsz[2] > 1024:
        from .walker import _walker

        v = _walker().validate(tr.iter_events())
        return tuple(v[0]) if v else None
    dtr = _device_columns(tr, device)
    ctx = _get_ctx(device)
    try:
        import torch

        info = trace_info(dtr)
        out = _native.Violation()
        i64x3 = ctypes.c_int64 * 3
        stream = torch.cuda.current_stream(dtr.kind.device).cuda_stream
        rc = ctx.lib.aiwc_validate(ctx.h, ctypes.c_void_p(dtr.kind.data_ptr()), ctypes.c_void_p(dtr.payload.data_ptr()),
                                   ctypes.byref(info), i64x3(*[int(x) for x in tr.global_size]), i64x3(*lsz),
                                   ctypes.byref(out), ctypes.c_void_p(stream))
        if rc == _native.OK:
            return None
        if rc != _native.ERR_INVALID_STREAM:
            ctx.check(rc)
        detail = out.detail.decode(errors="replace")
        if out.detail_code == _native.V_UNFINISHED:  # exact ids, dictionary groups included
            g = tr.group_of_key(out.group_key)
            loc = tr.local_of_id(out.local_id)
            gid = tuple(g[d] * lsz[d] + loc[d] for d in range(3))
            detail = f"work-item {gid} never ended"
        elif out.detail_code == _native.V_DIVERGENCE:
            counts = [int(out.counts[i]) for i in range(out.n_counts)]
            detail = f"work-items of group {tr.group_of_key(out.group_key)} hit differing barrier counts {counts}"
        return (int(out.event_index), out.rule.decode(), detail)
    finally:
        _put_ctx(ctx)


def max_ingest_events() -> int:
    """Events one aiwc_ingest takes (the engine's u32 event indices); larger traces
    are cut at work-group starts and combined exactly (dist.chunked_result).
    AIWC_MAX_INGEST_EVENTS lowers it (tests of the chunked path)."""
    limit = (1 << 32) - 1
    env = os.environ.get("AIWC_MAX_INGEST_EVENTS")
    return min(limit, int(env)) if env else limit


@dataclass
class EngineState:
    """What a later state merge needs of one consumed trace (aiwc_state_export):
    the per-key memory state as device runs over the trace's key map, and the
    histograms / tables finalize consumed."""

    runs: object            # torch int64 [2 * n_runs] on the device (key | len << 32, count | r << 62 | w << 63)
    n_runs: int
    base: int
    low_const: int
    k: int
    addr_stats: tuple | None
    itb_hist: np.ndarray
    ipt_hist: np.ndarray
    itb_ovf: np.ndarray
    ipt_ovf: np.ndarray
    branch_table: np.ndarray
    width_first: list


def _export_state(ctx, res: EngineResult, device: int) -> EngineState | None:
    import torch

    st = _native.State()
    ctx.check(ctx.lib.aiwc_state_export(ctx.h, ctypes.byref(st)))
    if not st.exported:
        return None
    arr = lambda p, n: np.ctypeslib.as_array(p, shape=(n,)).copy() if n else np.zeros(0, np.uint64)  # noqa: E731
    runs = torch.zeros(2, dtype=torch.int64, device=torch.device("cuda", device))
    if st.n_runs:
        iface = {"shape": (2 * st.n_runs,), "typestr": "<i8", "data": (st.runs_dev, False), "version": 3}
        holder = type("_Runs", (), {"__cuda_array_interface__": iface})()
        runs = torch.as_tensor(holder, device=torch.device("cuda", device)).clone()
    m = res.total_reads + res.total_writes
    return EngineState(runs, int(st.n_runs), int(st.base), int(st.low_const), int(st.k),
                       tuple(int(v) for v in st.addr_stats) if m else None,
                       arr(st.itb_hist, 1024), arr(st.ipt_hist, 1024), arr(st.itb_ovf, st.n_itb_ovf),
                       arr(st.ipt_ovf, st.n_ipt_ovf), arr(st.branch_table, st.branch_table_size),
                       [int(v) for v in arr(st.width_first, len(res.widths))])


def run_engine(tr: ColumnarTrace, device: int | None = None, check: bool = False,
               export: bool = False) -> EngineResult:
    """aiwc_reset + aiwc_ingest(_host) + aiwc_finalize on one columnar trace.
    check: StreamChecker's invariants inside the pass (InvalidStream without a
    location on a violation; result.stream_checked when the pass certified it)."""
    kind = tr.kind
    if device is None:
        device = kind.device.index if (_is_torch(kind) and kind.is_cuda) else _default_device()
    limit = max_ingest_events()
    if tr.n_events > limit:
        from . import dist as D

        return D.chunked_result(D.CudaBackend(device), tr, D.chunk_cuts(tr.kind, limit))
    ctx = _get_ctx(device)
    try:
        lib = ctx.lib
        ctx.check(lib.aiwc_reset(ctx.h))
        stream = ingest_columns(ctx, tr, check, export)
        res = _native.Result()
        ctx.check(lib.aiwc_finalize(ctx.h, ctypes.byref(res), ctypes.c_void_p(stream) if stream else None))
        out = _copy_result(res)
        out.stream_checked = bool(res.stream_checked)
        if export:
            out.state = _export_state(ctx, out, device)
        return out
    finally:
        _put_ctx(ctx)


def _default_device() -> int:
    try:
        import torch

        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except ImportError:  # pragma: no cover
        pass
    return 0


# ---------------------------------------------------------------------------
# accumulator
# ---------------------------------------------------------------------------
_OVERRIDABLE = ("opcode_histogram", "simd_width_counts", "itb_samples", "ipt_samples", "total_instructions",
                "work_items", "barriers_hit")


class KernelAccumulator:
    """Device-computed accumulator for one invocation (or a merge of several).

    Field names follow the reference (metrics.py:71-95).  Histogram-valued
    fields are materialised from the engine's exact tables; assigning one of
    them records an override that finalize's conservation checks see, as the
    reference's tampered-accumulator tests expect (test_metrics.py:237-241).
    """

    def __init__(self, kernel_name: str, invocations: list[int], launches: list, result: EngineResult,
                 opcodes: list[str], trace: ColumnarTrace | None = None,
                 lmae_per_invocation: list | None = None, parts: list | None = None):
        object.__setattr__(self, "_over", {})
        object.__setattr__(self, "_fields", None)
        self.parts = parts
        self.kernel_name = kernel_name
        self.invocations = invocations
        self.launches = launches
        self.result = result
        self.opcodes = opcodes
        self.trace = trace
        self.lmae_per_invocation = lmae_per_invocation

    def __setattr__(self, name, value):
        if name in _OVERRIDABLE:
            self._over[name] = value
        else:
            object.__setattr__(self, name, value)

    def __getattr__(self, name):
        over = object.__getattribute__(self, "_over")
        if name in over:
            return over[name]
        r = object.__getattribute__(self, "result")
        if name == "opcode_histogram":
            ops = object.__getattribute__(self, "opcodes")
            return Counter({ops[i]: c for i, c in enumerate(r.opcode_counts) if c})
        if name == "simd_width_counts":
            return Counter(dict(r.widths))
        if name == "total_instructions":
            return r.total_instructions
        if name == "work_items":
            return r.work_items
        if name == "barriers_hit":
            return r.barriers_hit
        if name in FIELDS:
            return self.per_event_fields()[name]
        raise AttributeError(name)

    def per_event_fields(self) -> dict:
        """itb/ipt sample lists, address Counters and branch streams, rebuilt
        from the consumed columns on first access (fields.py)."""
        f = object.__getattribute__(self, "_fields")
        if f is None:
            parts = object.__getattribute__(self, "parts")
            if parts:
                f = merge_fields([q.per_event_fields() for q in parts])
            elif object.__getattribute__(self, "trace") is not None:
                f = materialize(object.__getattribute__(self, "trace"))
            else:
                raise AiwcError("this accumulator was built without its trace columns")
            object.__setattr__(self, "_fields", f)
        return f

    def branch_executions(self) -> dict[int, int]:
        return dict(self.result.sites)


# ---------------------------------------------------------------------------
# consume / finalize / merge
# ---------------------------------------------------------------------------
def consume(events: Iterable | ColumnarTrace, *, max_entries: int | None = None,
            device: int | None = None) -> KernelAccumulator:
    """Fold one trace into an accumulator on the GPU (ref metrics.py:98-196).

    Raises InvalidStream at the first stream-invariant violation (validated
    by the native walker for object streams) and TraceTooLarge when
    unique read addresses + unique write addresses + branch executions exceed
    ``max_entries`` (default from AIWC_MEM_CAP_BYTES), whichever the
    reference would raise first.
    """
    cap = default_entry_cap() if max_entries is None else max_entries
    violation = None
    if isinstance(events, ColumnarTrace):
        tr = events
        if not tr.validated:  # columns from an untrusted producer: StreamChecker on the device
            if device is None:
                kind = tr.kind
                device = kind.device.index if (_is_torch(kind) and kind.is_cuda) else _default_device()
            tr = _device_columns(tr, device)
            res = err = None
            if tr.n_events <= max_ingest_events():
                # the ingest checks StreamChecker's invariants in the same pass (barrier /
                # resume traces: per-work-item order words, aiwc_capi.cu wi_rules_kernel);
                # only a flagged stream goes through the separate device checker, which
                # locates its first violation
                try:
                    res = run_engine(tr, device, check=True, export=True)
                except AiwcError as exc:  # a violation, or malformed data it caused (UnsupportedTrace too)
                    res, err = None, exc
                if res is not None and res.stream_checked:
                    if res.entries > cap:
                        raise TraceTooLarge(cap + 1, cap)
                    return KernelAccumulator(
                        kernel_name=tr.kernel_name, invocations=[tr.invocation],
                        launches=[(tr.invocation, tuple(tr.global_size), tuple(tr.local_size))],
                        result=res, opcodes=list(tr.opcodes), trace=tr)
            violation = validate_columnar(tr, device)
            if violation is None and err is not None:  # a valid stream the engine still refuses
                raise err
            if violation is None and res is not None:  # the pass's result stands (barrier traces)
                if res.entries > cap:
                    raise TraceTooLarge(cap + 1, cap)
                return KernelAccumulator(
                    kernel_name=tr.kernel_name, invocations=[tr.invocation],
                    launches=[(tr.invocation, tuple(tr.global_size), tuple(tr.local_size))],
                    result=res, opcodes=list(tr.opcodes), trace=tr)
            if violation is not None and violation[2] != "stream has no kernel_end":
                # consume() stops before the violating event; finish()'s rule sees every event
                index = violation[0]
                prefix = ColumnarTrace(tr.kind[:index], tr.payload[:index], tr.kernel_name, tr.invocation,
                                       tr.global_size, tr.local_size, tr.opcodes, tr.extra_groups, None)
                tr = prefix if index else None
    else:
        from .walker import encode_events

        tr, violation = encode_events(events)
    if violation is not None:
        # the reference raises whichever of (cap crossing, first violation) comes first
        # in stream order: the prefix before the violation decides
        index, rule, detail = violation
        if tr is not None and tr.n_events:
            res = run_engine(tr, device)
            if res.entries > cap:
                raise TraceTooLarge(cap + 1, cap)
        raise InvalidStream(index, rule, detail)
    res = run_engine(tr, device, export=True)
    if res.entries > cap:
        raise TraceTooLarge(cap + 1, cap)
    return KernelAccumulator(
        kernel_name=tr.kernel_name,
        invocations=[tr.invocation],
        launches=[(tr.invocation, tuple(tr.global_size), tuple(tr.local_size))],
        result=res, opcodes=list(tr.opcodes), trace=tr,
    )


class DistStats(NamedTuple):
    minimum: int
    maximum: int
    median: float
    mean: float
    sd: float


def summarize_distribution(samples: list[int]) -> DistStats:
    """Order statistics, mean, population sd of a host sample list (ref metrics.py:207-223)."""
    if not samples:
        raise EmptySample("cannot summarize an empty sample")
    ordered = sorted(samples)
    n = len(ordered)
    median = float(ordered[n // 2]) if n % 2 else (ordered[n // 2 - 1] + ordered[n // 2]) / 2.0
    mean = sum(ordered) / n
    var = sum((x - mean) ** 2 for x in ordered) / n
    return DistStats(ordered[0], ordered[-1], median, mean, math.sqrt(var))


def _dist_fields(d: tuple):
    """(min, max, median, mean) exactly as summarize_distribution would give."""
    n, lo, hi, total, mid_lo, mid_hi = d
    if not n:
        return 0, 0, 0.0, 0.0
    median = float(mid_hi) if n % 2 else (mid_lo + mid_hi) / 2.0
    return lo, hi, median, total / n


def lmae_profile(acc: KernelAccumulator) -> list[float]:
    """Locality entropy at skip levels 1..10 (ref metrics.py:226-232)."""
    r = acc.result
    if not r.footprint:
        return [0.0] * 10
    return [round12(v) for v in r.lmae]


def finalize(acc: KernelAccumulator) -> AiwcReport:
    """Every metric of the accumulator (ref metrics.py:273-386)."""
    r = acc.result
    over = acc._over
    total = over.get("total_instructions", r.total_instructions)
    # conservation (metrics.py:276-285); overrides model a tampered accumulator
    opc_sum = sum(over["opcode_histogram"].values()) if "opcode_histogram" in over else sum(r.opcode_counts)
    wid_sum = sum(over["simd_width_counts"].values()) if "simd_width_counts" in over else sum(c for _, c in r.widths)
    itb_sum = sum(over["itb_samples"]) if "itb_samples" in over else r.itb[3]
    ipt_sum = sum(over["ipt_samples"]) if "ipt_samples" in over else r.ipt[3]
    ipt_n = len(over["ipt_samples"]) if "ipt_samples" in over else r.ipt[0]
    work_items = over.get("work_items", r.work_items)
    if opc_sum != total:
        raise AiwcError("accumulator inconsistent: opcode counts != total instructions")
    if wid_sum != total:
        raise AiwcError("accumulator inconsistent: width samples != total instructions")
    if itb_sum != total:
        raise AiwcError("accumulator inconsistent: ITB samples do not cover all instructions")
    if ipt_sum != total:
        raise AiwcError("accumulator inconsistent: IPT samples do not cover all instructions")
    if ipt_n != work_items:
        raise AiwcError("accumulator inconsistent: one IPT sample per work-item expected")

    itb_min, itb_max, itb_med, itb_mean = _dist_fields(r.itb)
    ipt_min, ipt_max, ipt_med, _ = _dist_fields(r.ipt)

    # SIMD width statistics: the reference's expressions over first-seen order (metrics.py:298-306)
    widths = r.widths
    width_total = sum(c for _, c in widths)
    if width_total:
        simd_sum = sum(w * c for w, c in widths)
        simd_mean = simd_sum / width_total
        simd_var = sum(c * (w - simd_mean) ** 2 for w, c in widths) / width_total
        simd_max = max(w for w, _ in widths)
        simd_sd = math.sqrt(simd_var)
    else:
        simd_sum, simd_mean, simd_sd, simd_max = 0, 0.0, 0.0, 0

    ur, uw, tr_, tw = r.unique_reads, r.unique_writes, r.total_reads, r.total_writes
    if r.footprint:
        gmae = round12(r.gmae)
        lmae = [round12(v) for v in r.lmae]
        footprint_90 = r.footprint_90
    else:
        gmae, lmae, footprint_90 = 0.0, [0.0] * 10, 0

    executions = r.branch_executions
    no_branches = executions == 0
    if no_branches:
        yokota, linear, warmup = 0.0, 0.0, 0.0
    elif r.branch_observations == 0:  # every stream shorter than the warm-up (NoBranches)
        yokota, linear, warmup = 0.0, 0.0, 1.0
    else:
        yokota, linear = round12(r.yokota), round12(r.linear)
        warmup = round12(r.branch_excluded / executions)

    if acc.lmae_per_invocation is not None:
        per_inv = [{"invocation": inv, "lmae": prof} for inv, prof in acc.lmae_per_invocation]
    else:
        per_inv = [{"invocation": acc.invocations[0], "lmae": list(lmae)}]

    return AiwcReport(
        kernel=acc.kernel_name,
        invocations=list(acc.invocations),
        opcode=r.opcode_coverage,
        total_instruction_count=total,
        work_items=work_items,
        total_barriers_hit=over.get("barriers_hit", r.barriers_hit),
        min_itb=itb_min, max_itb=itb_max, median_itb=round12(itb_med),
        min_ipt=ipt_min, max_ipt=ipt_max, median_ipt=round12(ipt_med),
        max_simd_width=simd_max, mean_simd_width=round12(simd_mean), sd_simd_width=round12(simd_sd),
        total_memory_footprint=r.footprint, footprint_90=footprint_90,
        unique_reads=ur, unique_writes=uw,
        unique_rw_ratio=None if uw == 0 else round12(ur / uw),
        total_reads=tr_, total_writes=tw,
        reread_ratio=0.0 if tr_ == 0 else round12(ur / tr_),
        rewrite_ratio=0.0 if tw == 0 else round12(uw / tw),
        gmae=gmae, lmae=lmae,
        total_unique_branch_instructions=len(r.sites),
        branch_90=r.branch_90 if r.sites else 0,
        yokota_entropy=yokota, linear_entropy=linear,
        mean_itb=round12(itb_mean), simd_width_sum=simd_sum,
        no_branches=no_branches, warmup_excluded_fraction=warmup,
        no_reads=tr_ == 0, no_writes=tw == 0,
        lmae_per_invocation=per_inv,
    )


def merge_accumulators(parts: list[KernelAccumulator], *, allow_name_mismatch: bool = False) -> KernelAccumulator:
    """Application-level merge (ref metrics.py:235-270): histograms add, samples
    concatenate, branch streams stay separate, per-part LMAE profiles are kept.

    The merged accumulator is recomputed on the GPU from the parts' columns
    concatenated in order (opcode dictionaries unified, group keys made
    disjoint so no branch history crosses a part boundary), which is exactly
    the reference's definition of a merge.
    """
    from .merge import concat_traces

    if not parts:
        raise EmptySample("nothing to merge")
    names = {p.kernel_name for p in parts}
    if len(names) > 1 and not allow_name_mismatch:
        raise IncompatibleReports(f"kernel names differ: {sorted(names)}")
    per_inv: list = []
    for p in parts:
        if p.lmae_per_invocation is not None:
            per_inv.extend(p.lmae_per_invocation)
        else:
            per_inv.append((p.invocations[0], lmae_profile(p)))
    invocations = [i for p in parts for i in p.invocations]
    launches = [l for p in parts for l in p.launches]
    leaves = _leaves(parts)
    merged = _state_merge(leaves)  # sums of the parts' exported state: no re-ingest
    if merged is not None:
        res, opcodes = merged
        return KernelAccumulator(parts[0].kernel_name, invocations, launches, res, opcodes, trace=None,
                                 lmae_per_invocation=per_inv, parts=list(parts))
    tr = concat_traces([p.trace for p in leaves])
    res = run_engine(tr)
    return KernelAccumulator(parts[0].kernel_name, invocations, launches, res, list(tr.opcodes), trace=tr,
                             lmae_per_invocation=per_inv, parts=list(parts))


def _leaves(parts: list) -> list:
    """The consumed accumulators under (possibly nested) merges, in order."""
    out = []
    for p in parts:
        if p.parts:
            out.extend(_leaves(p.parts))
        else:
            out.append(p)
    return out


def _state_merge(parts: list):
    """(EngineResult, opcode names) of the parts merged from their exported state
    (EngineState), or None when a part has none (sort-path or random-access
    traces) or the merged address span needs the sort path: the caller re-ingests."""
    from . import dist as D

    states = [p.result.state for p in parts]
    if any(s is None for s in states) or any(p._over for p in parts):
        return None
    idx: dict = {}
    for p in parts:
        for o in p.opcodes:
            idx.setdefault(o, len(idx))
    opcode_counts = [0] * len(idx)
    lists, offset = [], 0
    itb_hist = np.zeros(1024, np.uint64)
    ipt_hist = np.zeros(1024, np.uint64)
    table = None
    for p, st in zip(parts, states):
        r = p.result
        for i, c in enumerate(r.opcode_counts):
            opcode_counts[idx[p.opcodes[i]]] += int(c)
        widths = [(w, c, f + offset) for (w, c), f in zip(r.widths, st.width_first)]
        lists.append((st.itb_ovf.tolist(), st.ipt_ovf.tolist(), widths, dict(r.sites)))
        itb_hist += st.itb_hist
        ipt_hist += st.ipt_hist
        if st.branch_table.size:
            table = st.branch_table.astype(np.uint64) if table is None else table + st.branch_table
        offset += r.n_events
    itb_ovf, ipt_ovf, widths, sites = D._merge_lists(lists)
    tot = lambda f: sum(int(getattr(p.result, f)) for p in parts)  # noqa: E731
    total_reads, total_writes = tot("total_reads"), tot("total_writes")
    total_m = total_reads + total_writes
    mp = D.MemoryPartial(0, 0, 0, np.zeros(11), np.zeros(D.CBINS, np.uint64), np.zeros(0, np.uint64))
    if total_m:
        live = [st for st in states if st.addr_stats is not None]
        aand, aor = (1 << 64) - 1, 0
        for st in live:
            aand &= st.addr_stats[2]
            aor |= st.addr_stats[3]
        stats = (min(st.addr_stats[0] for st in live), max(st.addr_stats[1] for st in live), aand, aor)
        device = live[0].runs.device.index
        ctx = _get_ctx(device)
        try:
            import torch

            rp = (_native.RunsPart * len(live))()
            for i, st in enumerate(live):
                rp[i] = _native.RunsPart(st.runs.data_ptr(), st.n_runs, st.base, st.low_const, st.k, 0)
            out = _native.MemoryPart()
            s4 = (ctypes.c_uint64 * 4)(*stats)
            stream = torch.cuda.current_stream(device).cuda_stream
            rc = ctx.lib.aiwc_memory_merge(ctx.h, rp, len(live), s4, total_m, ctypes.byref(out), ctypes.c_void_p(stream))
            if rc == _native.ERR_UNSUPPORTED:
                return None
            ctx.check(rc)
            big = np.ctypeslib.as_array(out.big, shape=(out.n_big,)).copy() if out.n_big else np.zeros(0, np.uint64)
            mp = D.MemoryPartial(out.unique_reads, out.unique_writes, out.footprint, np.array(out.level_sum[:]),
                                 np.ctypeslib.as_array(out.cnt_hist0, shape=(D.CBINS,)).copy(), big)
        finally:
            _put_ctx(ctx)
    if table is None:
        table = np.zeros(1 << 16, np.uint64)
    res = D._assemble(tot("n_events"), tot("total_instructions"), tot("work_items"), tot("barriers_hit"), total_reads,
                      total_writes, sum(int(p.result.itb[3]) for p in parts), sum(int(p.result.ipt[3]) for p in parts),
                      tot("branch_executions"), opcode_counts, itb_hist, itb_ovf, ipt_hist, ipt_ovf, table, widths,
                      sites, mp.unique_reads, mp.unique_writes, mp.footprint, mp.cnt_hist0.astype(np.uint64),
                      np.sort(mp.big.astype(np.uint64))[::-1], np.asarray(mp.level_sum, dtype=np.float64))
    return res, [o for o, _ in sorted(idx.items(), key=lambda kv: kv[1])]
