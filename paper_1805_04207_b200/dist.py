"""Multi-GPU AIWC: work-group shards, key-range owners, one all-to-all.

Every rank owns a contiguous range of work-groups.  Everything except the
address statistics is local to a work-group -- segments and work-item
lifetimes (ITB / IPT), per-(site, group) branch streams, opcode / width
counts -- so those partials are combined exactly with sums (histograms,
pattern tables) and gathers (overflow lists, site and width lists).  The
reference's own shard-merge equality (`metrics.py:235-270`) is
what makes this exact.

Addresses need one exchange: after an all-reduce of the shards' address
statistics every rank knows the global key map key = (addr - base) >> k;
key ranges aligned to 1024 keys are assigned to owners (so every LSB-skip
level <= 10 groups keys of a single owner), each rank sends its addresses to
their owners with one all-to-all, and each owner computes unique counts,
level-0 count-of-counts and sum(p log2 p) per level for its keys with the
global access count M.  The owners' partials add up to the whole-trace values.

The engine work is behind a small backend interface (`CudaBackend` runs the
C ABI on the local GPU with NCCL; the CPU tests plug in an oracle-backed
backend with gloo), so the exchange and combine logic here is the code the
GPU path runs.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

HBINS = 1024
CBINS = 1024


@dataclass
class ShardPartial:
    """Exact per-shard quantities (everything but the address statistics)."""

    n_events: int
    total_instructions: int
    work_items: int
    barriers_hit: int
    total_reads: int
    total_writes: int
    opcode_counts: np.ndarray            # u64 per opcode id (shared dictionary)
    widths: list                         # [(width, count, first global event index)]
    itb_hist: np.ndarray                 # HBINS u64
    itb_ovf: np.ndarray                  # values >= HBINS
    itb_sum: int
    ipt_hist: np.ndarray
    ipt_ovf: np.ndarray
    ipt_sum: int
    branch_table: np.ndarray             # u64 total << 32 | taken, 2^H entries
    sites: dict                          # site -> executions
    branch_executions: int
    addr_stats: tuple | None             # (min, max, and, or) of the shard's addresses
    handle: object = None                # backend state (device address arrays)


@dataclass
class MemoryPartial:
    unique_reads: int
    unique_writes: int
    footprint: int
    level_sum: np.ndarray                # 11 x f64: sum of p log2 p over owned keys
    cnt_hist0: np.ndarray                # CBINS u64
    big: np.ndarray                      # level-0 counts >= CBINS


@dataclass
class KeyMap:
    base: int
    k: int
    n_keys: int
    keys_per_rank: int

    def owned(self, rank: int) -> tuple[int, int]:
        lo = rank * self.keys_per_rank
        hi = min(self.n_keys, lo + self.keys_per_rank)
        return lo, max(0, hi - lo)


def key_map(stats: tuple, nranks: int) -> KeyMap:
    """Global key map from the all-reduced address statistics (the engine's rule)."""
    amin, amax, aand, aor = stats
    base = amin & ~1023
    vary = aand ^ aor
    k = min((vary & -vary).bit_length() - 1, 32) if vary else 0
    n_keys = ((amax - base) >> k) + 1
    kpr = -(-n_keys // nranks)
    kpr = -(-kpr // 1024) * 1024
    return KeyMap(base, k, n_keys, kpr)


# ---------------------------------------------------------------------------
# host finishing of combined exact integers (same rules as aiwc_finalize)
# ---------------------------------------------------------------------------
def coverage90(big_desc, small_hist, total: int) -> int:
    """Smallest k of the most frequent keys covering 9/10 of total (entropy.py:49-66)."""
    if total == 0:
        return 0
    cum = 0
    k = 0
    for c in big_desc:
        cum += int(c)
        k += 1
        if cum * 10 >= total * 9:
            return k
    if small_hist is not None:
        for c in range(len(small_hist) - 1, 0, -1):
            h = int(small_hist[c])
            if not h:
                continue
            need = total * 9 - cum * 10
            take = -(-need // (c * 10))
            if take <= h:
                return k + take
            cum += h * c
            k += h
    return k


def order_stats(hist: np.ndarray, ovf_sorted: np.ndarray, total_sum: int) -> tuple:
    """(n, min, max, sum, mid_lo, mid_hi) of a histogram + sorted overflow values."""
    small = int(hist.sum())
    n = small + int(len(ovf_sorted))
    if n == 0:
        return (0, 0, 0, total_sum, 0, 0)
    csum = np.cumsum(hist.astype(np.int64))

    def at(rank: int) -> int:
        if rank >= small:
            return int(ovf_sorted[rank - small])
        return int(np.searchsorted(csum, rank, side="right"))

    return (n, at(0), at(n - 1), total_sum, at((n - 1) // 2), at(n // 2))


def branch_entropies(table: np.ndarray):
    """Yokota / linear from the pooled pattern table -- the reference's numpy
    expressions (entropy.py:123-132) on the same integer tables."""
    total_tab = (table >> np.uint64(32)).astype(np.int64)
    taken_tab = (table & np.uint64(0xFFFFFFFF)).astype(np.int64)
    observations = int(total_tab.sum())
    if observations == 0:
        return 0.0, 0.0, 0
    mask = total_tab > 0
    totals = total_tab[mask].astype(np.float64)
    p = taken_tab[mask] / totals
    q = 1.0 - p
    with np.errstate(divide="ignore", invalid="ignore"):
        h = -(np.where(p > 0, p * np.log2(np.where(p > 0, p, 1.0)), 0.0)
              + np.where(q > 0, q * np.log2(np.where(q > 0, q, 1.0)), 0.0))
    weights = totals / observations
    return float((weights * h).sum()), float((weights * np.minimum(p, q)).sum()), observations


# ---------------------------------------------------------------------------
# collectives (torch.distributed: NCCL on GPUs, gloo in the CPU tests)
# ---------------------------------------------------------------------------
def _allreduce_i64(vals: np.ndarray, op, group, device) -> np.ndarray:
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(np.ascontiguousarray(vals).view(np.int64).copy()).to(device)
    dist.all_reduce(t, op=op, group=group)
    return t.cpu().numpy().view(np.uint64)


def _gather_objects(obj, group) -> list:
    import torch.distributed as dist

    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, obj, group=group)
    return out


def allreduce_stats(stats, group, device):
    """(min, max, and, or) over ranks; empty shards contribute identities.  One
    all-gather of the four words (NCCL has no bitwise reductions), combined on
    the host in unsigned arithmetic."""
    import torch
    import torch.distributed as dist

    amin, amax, aand, aor = stats if stats is not None else ((1 << 64) - 1, 0, (1 << 64) - 1, 0)
    mine = torch.from_numpy(np.array([amin, amax, aand, aor], np.uint64).view(np.int64).copy()).to(device)
    parts = [torch.empty_like(mine) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, mine, group=group)
    v = np.stack([p.cpu().numpy().view(np.uint64) for p in parts])
    return (int(v[:, 0].min()), int(v[:, 1].max()), int(np.bitwise_and.reduce(v[:, 2])),
            int(np.bitwise_or.reduce(v[:, 3])))


RUNS_TABLE_BUDGET = 16 << 30  # bytes of one owner's dense table in the run exchange
LAST_EXCHANGE = None  # "runs" or "raw": the address exchange the last sharded_result used
RUN_MIN_AVG = 32      # accesses per run below which the raw exchange is used


def runs_dense_ok(km: KeyMap, total_m: int) -> bool:
    """Owners can hold their key ranges as dense tables (the run exchange needs one)."""
    return km.keys_per_rank * 8 <= RUNS_TABLE_BUDGET and km.n_keys <= 4 * total_m + (1 << 20)


def exchange(entries, counts: list[int], group, device):
    """All-to-all of owner-grouped u64 entries; returns (received tensor, n)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    send_counts = torch.tensor(counts, dtype=torch.int64, device=device)
    recv_counts = torch.empty(world, dtype=torch.int64, device=device)
    dist.all_to_all_single(recv_counts, send_counts, group=group)
    rc = [int(x) for x in recv_counts.cpu().tolist()]
    recv = torch.empty(max(1, sum(rc)), dtype=torch.int64, device=device)
    dist.all_to_all_single(recv[: sum(rc)], entries[: sum(counts)].to(device), rc, list(counts), group=group)
    return recv, sum(rc)


def comm_device(backend, group=None):
    """Where collective buffers live: the backend's device under NCCL, host
    memory under gloo (the CPU tests, and single-GPU tests of CudaBackend)."""
    import torch
    import torch.distributed as dist

    return torch.device("cpu") if dist.get_backend(group) == "gloo" else backend.device


def sharded_result(backend, shard, shard_offset: int, group=None):
    """Every rank: exact whole-trace EngineResult from its work-group shard.

    Collectives: one object all-gather of the small per-shard partials (counts,
    opcode / ITB / IPT histograms, overflow and width / site lists, address
    statistics), the 2^16 branch pattern table all-reduce only when the trace
    has branches, the address exchange (run-count all-reduce + two all-to-alls),
    and one object all-gather of the owners' memory partials."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    device = comm_device(backend, group)
    sp: ShardPartial = backend.shard(shard, shard_offset)

    # ---- small partials: one object all-gather, summed / merged on the host ----
    scalars = [int(sp.n_events), int(sp.total_instructions), int(sp.work_items), int(sp.barriers_hit),
               int(sp.total_reads), int(sp.total_writes), int(sp.itb_sum), int(sp.ipt_sum),
               int(sp.branch_executions)]
    parts = _gather_objects((scalars, sp.opcode_counts.astype(np.uint64), sp.itb_hist, sp.ipt_hist,
                             sp.itb_ovf.tolist(), sp.ipt_ovf.tolist(), sp.widths, sp.sites, sp.addr_stats), group)
    sc = [sum(p[0][i] for p in parts) for i in range(len(scalars))]
    opcode_counts = [int(v) for v in np.sum([p[1] for p in parts], axis=0)]
    itb_hist = np.sum([p[2] for p in parts], axis=0).astype(np.uint64)
    ipt_hist = np.sum([p[3] for p in parts], axis=0).astype(np.uint64)
    itb_ovf, ipt_ovf, widths, sites = _merge_lists([p[4:8] for p in parts])
    n_events, total_instr, work_items, barriers, total_reads, total_writes, itb_sum, ipt_sum, br_exec = sc
    # ---- branch pattern tables (each (site, group) stream is whole on one rank) ----
    if br_exec:
        branch_table = _allreduce_i64(sp.branch_table.astype(np.uint64), dist.ReduceOp.SUM, group, device)
    else:
        branch_table = np.zeros(len(sp.branch_table), np.uint64)

    # ---- addresses: global key map, owner exchange, owner partials ----
    total_m = total_reads + total_writes
    if total_m:
        st = [p[8] for p in parts if p[8] is not None]
        stats = (min(x[0] for x in st), max(x[1] for x in st), int(np.bitwise_and.reduce([np.uint64(x[2]) for x in st])),
                 int(np.bitwise_or.reduce([np.uint64(x[3]) for x in st])))
        km = key_map(stats, world)
        lo, n_owned = km.owned(rank)
        use_runs = False
        if hasattr(backend, "partition_runs") and runs_dense_ok(km, total_m):
            # pre-aggregation: runs of consecutive keys per owner; chosen (on every
            # rank alike) when runs average >= RUN_MIN_AVG accesses (the owner
            # applies one run per warp: short runs would idle its lanes)
            runs, rcounts = backend.partition_runs(sp, km, world)
            tot = _allreduce_i64(np.array([sum(rcounts)], np.uint64), dist.ReduceOp.SUM, group, device)
            use_runs = RUN_MIN_AVG * int(tot[0]) <= total_m
        global LAST_EXCHANGE
        LAST_EXCHANGE = "runs" if use_runs else "raw"
        if use_runs:
            recv, n_words = exchange(runs, [2 * c for c in rcounts], group, device)
            mp = backend.memory_partial_runs(recv, n_words // 2, km, lo, n_owned, total_m)
        else:
            reads, writes, counts = backend.partition(sp, km, world)
            recv_r, n_r = exchange(reads, counts[:world], group, device)
            recv_w, n_w = exchange(writes, counts[world:], group, device)
            mp = backend.memory_partial(recv_r, n_r, recv_w, n_w, km, lo, n_owned, total_m)
    else:
        mp = MemoryPartial(0, 0, 0, np.zeros(11), np.zeros(CBINS, np.uint64), np.zeros(0, np.uint64))
    # ---- owners' partials: one object all-gather (level sums added in rank order) ----
    mparts = _gather_objects((int(mp.unique_reads), int(mp.unique_writes), int(mp.footprint),
                              np.asarray(mp.level_sum, dtype=np.float64), mp.cnt_hist0.astype(np.uint64),
                              mp.big.astype(np.uint64)), group)
    unique_r = sum(m[0] for m in mparts)
    unique_w = sum(m[1] for m in mparts)
    footprint = sum(m[2] for m in mparts)
    level_sum = np.zeros(11)
    for m in mparts:
        level_sum = level_sum + m[3]
    hist0 = np.sum([m[4] for m in mparts], axis=0).astype(np.uint64)
    big = np.sort(np.concatenate([m[5] for m in mparts]).astype(np.uint64))[::-1]
    return _assemble(n_events, total_instr, work_items, barriers, total_reads, total_writes, itb_sum, ipt_sum,
                     br_exec, opcode_counts, itb_hist, itb_ovf, ipt_hist, ipt_ovf, branch_table, widths, sites,
                     unique_r, unique_w, footprint, hist0, big, level_sum)


def _assemble(n_events, total_instr, work_items, barriers, total_reads, total_writes, itb_sum, ipt_sum, br_exec,
              opcode_counts, itb_hist, itb_ovf, ipt_hist, ipt_ovf, branch_table, widths, sites, unique_r, unique_w,
              footprint, hist0, big, level_sum):
    """EngineResult of combined exact integers, finished with the same rules as aiwc_finalize."""
    from .metrics import EngineResult

    total_m = total_reads + total_writes
    yokota, linear, observations = branch_entropies(branch_table)
    ent = [-float(v) for v in level_sum] if total_m else [0.0] * 11
    oc = sorted((c for c in opcode_counts if c), reverse=True)
    return EngineResult(
        n_events=n_events, total_instructions=total_instr, work_items=work_items, barriers_hit=barriers,
        opcode_coverage=coverage90(oc, None, sum(oc)),
        itb=order_stats(itb_hist, itb_ovf, itb_sum), ipt=order_stats(ipt_hist, ipt_ovf, ipt_sum),
        total_reads=total_reads, total_writes=total_writes, unique_reads=unique_r, unique_writes=unique_w,
        footprint=footprint, footprint_90=coverage90(big, hist0, total_m) if total_m else 0,
        gmae=ent[0], lmae=ent[1:], branch_executions=br_exec, branch_observations=observations,
        branch_excluded=br_exec - observations, branch_90=coverage90(sorted((c for _, c in sites), reverse=True), None, br_exec),
        yokota=yokota, linear=linear, entries=unique_r + unique_w + br_exec,
        opcode_counts=opcode_counts, widths=widths, sites=sites, used_dense_table=True, kernels_launched=0,
    )


def _merge_lists(parts):
    """Overflow samples, width list (first appearance order) and site counts of shard partials."""
    itb_ovf = np.sort(np.array([v for p in parts for v in p[0]], dtype=np.uint64))
    ipt_ovf = np.sort(np.array([v for p in parts for v in p[1]], dtype=np.uint64))
    wmap: dict = {}
    for p in parts:
        for w, c, first in p[2]:
            c0, f0 = wmap.get(w, (0, None))
            wmap[w] = (c0 + c, first if f0 is None else min(f0, first))
    widths = [(w, c) for w, (c, _) in sorted(wmap.items(), key=lambda kv: kv[1][1])]
    smap: dict = {}
    for p in parts:
        for s, c in p[3].items():
            smap[s] = smap.get(s, 0) + c
    return itb_ovf, ipt_ovf, widths, sorted(smap.items())


def chunk_cuts(kind, limit: int) -> list[int]:
    """Cut points (event indices) splitting a trace into chunks of at most `limit`
    events, each cut at a wg_begin, so every work-group, segment and (site, group)
    branch stream lies inside one chunk."""
    from .trace import K_WG_BEGIN

    if type(kind).__module__.startswith("torch"):
        import torch

        starts = torch.nonzero(kind == K_WG_BEGIN).flatten().cpu().numpy()
    else:
        starts = np.nonzero(np.asarray(kind) == K_WG_BEGIN)[0]
    n = int(kind.shape[0])
    cuts = [0]
    while n - cuts[-1] > limit:
        # the last group start that keeps this chunk within the limit
        i = int(np.searchsorted(starts, cuts[-1] + limit, side="right")) - 1
        if i < 0 or int(starts[i]) <= cuts[-1]:
            from .errors import UnsupportedTrace

            raise UnsupportedTrace(f"a work-group spans more than {limit} events")
        # prefer a cut at a 16-aligned event (the chunk's device columns then need no
        # aligned copy) among the last few group starts that fit
        for j in range(i, max(i - 64, -1), -1):
            if int(starts[j]) <= cuts[-1]:
                break
            if int(starts[j]) % 16 == 0:
                i = j
                break
        cuts.append(int(starts[i]))
    cuts.append(n)
    return cuts


def chunked_result(backend, tr, cuts: list[int]):
    """One trace larger than one ingest allows, on one GPU: each chunk (whole
    work-groups) is a shard pass; sums and lists combine as across ranks, and the
    chunks' compacted addresses are finished by one owner (this GPU)."""
    import torch

    from .trace import ColumnarTrace

    parts, rd, wr = [], [], []
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        sub = ColumnarTrace(tr.kind[lo:hi], tr.payload[lo:hi], tr.kernel_name, tr.invocation, tr.global_size,
                            tr.local_size, tr.opcodes, tr.extra_groups, None, validated=True)
        sp = backend.shard(sub, lo)
        r, w = backend.addresses(sp)
        parts.append(sp)
        rd.append(r.clone())
        wr.append(w.clone())
    tot = lambda f: sum(int(getattr(p, f)) for p in parts)  # noqa: E731
    n_events, total_instr, work_items, barriers = tot("n_events"), tot("total_instructions"), tot("work_items"), \
        tot("barriers_hit")
    total_reads, total_writes = tot("total_reads"), tot("total_writes")
    itb_sum, ipt_sum, br_exec = tot("itb_sum"), tot("ipt_sum"), tot("branch_executions")
    opcode_counts = [int(v) for v in np.sum([p.opcode_counts.astype(np.uint64) for p in parts], axis=0)]
    itb_hist = np.sum([p.itb_hist for p in parts], axis=0)
    ipt_hist = np.sum([p.ipt_hist for p in parts], axis=0)
    branch_table = np.sum([p.branch_table.astype(np.uint64) for p in parts], axis=0)
    itb_ovf, ipt_ovf, widths, sites = _merge_lists(
        [(p.itb_ovf.tolist(), p.ipt_ovf.tolist(), p.widths, p.sites) for p in parts])
    total_m = total_reads + total_writes
    if total_m:
        st = [p.addr_stats for p in parts if p.addr_stats is not None]
        stats = (min(s[0] for s in st), max(s[1] for s in st), int(np.bitwise_and.reduce([np.uint64(s[2]) for s in st])),
                 int(np.bitwise_or.reduce([np.uint64(s[3]) for s in st])))
        km = key_map(stats, 1)
        reads = torch.cat(rd) if total_reads else torch.zeros(1, dtype=torch.int64, device=backend.device)
        writes = torch.cat(wr) if total_writes else torch.zeros(1, dtype=torch.int64, device=backend.device)
        mp = backend.memory_partial(reads, total_reads, writes, total_writes, km, 0, km.n_keys, total_m)
    else:
        mp = MemoryPartial(0, 0, 0, np.zeros(11), np.zeros(CBINS, np.uint64), np.zeros(0, np.uint64))
    big = np.sort(mp.big.astype(np.uint64))[::-1]
    return _assemble(n_events, total_instr, work_items, barriers, total_reads, total_writes, itb_sum, ipt_sum,
                     br_exec, opcode_counts, itb_hist, itb_ovf, ipt_hist, ipt_ovf, branch_table, widths, sites,
                     mp.unique_reads, mp.unique_writes, mp.footprint, mp.cnt_hist0.astype(np.uint64), big,
                     np.asarray(mp.level_sum, dtype=np.float64))


def sharded_report(backend, shard, shard_offset: int, kernel_name: str, invocation: int, global_size, local_size,
                   opcodes: list[str], group=None):
    """AiwcReport of the whole trace, identical on every rank."""
    from .metrics import KernelAccumulator, finalize

    res = sharded_result(backend, shard, shard_offset, group)
    acc = KernelAccumulator(kernel_name, [invocation], [(invocation, tuple(global_size), tuple(local_size))], res,
                            list(opcodes))
    return finalize(acc)


# ---------------------------------------------------------------------------
# CUDA backend: the C ABI on this rank's GPU
# ---------------------------------------------------------------------------
class _CudaArray:
    """Zero-copy torch view of an engine-owned device buffer."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i8", "data": (ptr, False), "version": 3}


@dataclass
class CudaBackend:
    """The C ABI on this rank's GPU.  `timing` records per-phase CUDA-event
    times of the shard pass (last_phase_ms); `launches` counts the engine
    kernels this backend queued (shard pass + partition + owner partial)."""

    device_index: int = 0
    timing: bool = False
    ctx: object = None
    last_phase_ms: list = field(default_factory=list)
    last_d2h: int = 0
    launches: int = 0

    @property
    def device(self):
        import torch

        return torch.device("cuda", self.device_index)

    def _ctx(self):
        from . import _native

        if self.ctx is None:
            flags = _native.OPT_NO_CONSERVATION | _native.OPT_SHARD | (_native.OPT_TIMING if self.timing else 0)
            self.ctx = _native.Context(self.device_index, flags=flags)
        return self.ctx

    def shard(self, tr, shard_offset: int) -> ShardPartial:
        from . import _native
        from .metrics import _copy_result, ingest_columns

        ctx = self._ctx()
        lib = ctx.lib
        ctx.check(lib.aiwc_reset(ctx.h))
        stream = ingest_columns(ctx, tr)
        res = _native.Result()
        ctx.check(lib.aiwc_finalize(ctx.h, ctypes.byref(res), ctypes.c_void_p(stream) if stream else None))
        self.last_phase_ms = list(res.phase_ms)
        self.last_d2h = res.d2h_bytes
        self.launches += res.kernels_launched
        r = _copy_result(res)
        t = _native.ShardTables()
        ctx.check(lib.aiwc_shard_tables_get(ctx.h, ctypes.byref(t)))
        arr = lambda p, n: np.ctypeslib.as_array(p, shape=(n,)).copy() if n else np.zeros(0, np.uint64)  # noqa: E731
        firsts = arr(t.width_first, len(r.widths))
        return ShardPartial(
            n_events=r.n_events, total_instructions=r.total_instructions, work_items=r.work_items,
            barriers_hit=r.barriers_hit, total_reads=r.total_reads, total_writes=r.total_writes,
            opcode_counts=np.array(r.opcode_counts, dtype=np.uint64),
            widths=[(w, c, int(f) + shard_offset) for (w, c), f in zip(r.widths, firsts)],
            itb_hist=arr(t.itb_hist, HBINS), itb_ovf=arr(t.itb_ovf, t.n_itb_ovf), itb_sum=r.itb[3],
            ipt_hist=arr(t.ipt_hist, HBINS), ipt_ovf=arr(t.ipt_ovf, t.n_ipt_ovf), ipt_sum=r.ipt[3],
            branch_table=arr(t.branch_table, t.branch_table_size) if t.branch_table_size else np.zeros(1 << 16, np.uint64),
            sites=dict(r.sites), branch_executions=r.branch_executions,
            addr_stats=tuple(int(v) for v in t.addr_stats) if (r.total_reads + r.total_writes) else None,
        )

    def addresses(self, sp: ShardPartial):
        """Zero-copy device views of the last shard's compacted read / write addresses."""
        import torch

        from . import _native

        ctx = self._ctx()
        t = _native.ShardTables()
        ctx.check(ctx.lib.aiwc_shard_tables_get(ctx.h, ctypes.byref(t)))
        view = lambda p, n: torch.as_tensor(_CudaArray(ctypes.cast(p, ctypes.c_void_p).value, max(n, 1)),  # noqa: E731
                                            device=self.device)[:n]
        return view(t.rd_dev, int(sp.total_reads)), view(t.wr_dev, int(sp.total_writes))

    def partition_runs(self, sp: ShardPartial, km: KeyMap, nranks: int):
        """Owner-grouped runs of this shard's addresses (two int64 words per run)."""
        import torch

        ctx = self._ctx()
        counts = (ctypes.c_uint64 * nranks)()
        rp = ctypes.POINTER(ctypes.c_uint64)()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        ctx.check(ctx.lib.aiwc_partition_runs(ctx.h, km.base, km.k, km.keys_per_rank, nranks, ctypes.byref(rp), counts,
                                              ctypes.c_void_p(stream)))
        c = [int(x) for x in counts]
        self.launches += 6
        runs = torch.as_tensor(_CudaArray(ctypes.cast(rp, ctypes.c_void_p).value, max(2 * sum(c), 1)),
                               device=self.device)
        return runs, c

    def memory_partial_runs(self, recv, n_runs: int, km: KeyMap, key_lo: int, n_keys: int,
                            total_m: int) -> MemoryPartial:
        import torch

        from . import _native

        ctx = self._ctx()
        out = _native.MemoryPart()
        recv = recv.to(self.device)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        ctx.check(ctx.lib.aiwc_memory_partial_runs(ctx.h, ctypes.c_void_p(recv.data_ptr()), n_runs, km.k, key_lo,
                                                   n_keys, total_m, ctypes.byref(out), ctypes.c_void_p(stream)))
        self.launches += out.kernels_launched
        big = np.ctypeslib.as_array(out.big, shape=(out.n_big,)).copy() if out.n_big else np.zeros(0, np.uint64)
        return MemoryPartial(out.unique_reads, out.unique_writes, out.footprint, np.array(out.level_sum[:]),
                             np.ctypeslib.as_array(out.cnt_hist0, shape=(CBINS,)).copy(), big)

    def partition(self, sp: ShardPartial, km: KeyMap, nranks: int):
        import torch

        ctx = self._ctx()
        counts = (ctypes.c_uint64 * (2 * nranks))()
        rp, wp = ctypes.POINTER(ctypes.c_uint64)(), ctypes.POINTER(ctypes.c_uint64)()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        ctx.check(ctx.lib.aiwc_partition_addresses(ctx.h, km.base, km.k, km.keys_per_rank, nranks, ctypes.byref(rp),
                                                   ctypes.byref(wp), counts, ctypes.c_void_p(stream)))
        c = [int(x) for x in counts]
        self.launches += 2 * (int(sum(c[:nranks]) > 0) + int(sum(c[nranks:]) > 0))  # count + scatter per array
        view = lambda p, n: torch.as_tensor(_CudaArray(ctypes.cast(p, ctypes.c_void_p).value, max(n, 1)),  # noqa: E731
                                            device=self.device)
        return view(rp, sum(c[:nranks])), view(wp, sum(c[nranks:])), c

    def memory_partial(self, recv_r, n_r: int, recv_w, n_w: int, km: KeyMap, key_lo: int, n_keys: int,
                       total_m: int) -> MemoryPartial:
        import torch

        from . import _native

        ctx = self._ctx()
        out = _native.MemoryPart()
        recv_r, recv_w = recv_r.to(self.device), recv_w.to(self.device)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        ctx.check(ctx.lib.aiwc_memory_partial(ctx.h, ctypes.c_void_p(recv_r.data_ptr()), n_r,
                                              ctypes.c_void_p(recv_w.data_ptr()), n_w, km.base, km.k, key_lo, n_keys,
                                              total_m, ctypes.byref(out), ctypes.c_void_p(stream)))
        self.launches += out.kernels_launched
        big = np.ctypeslib.as_array(out.big, shape=(out.n_big,)).copy() if out.n_big else np.zeros(0, np.uint64)
        return MemoryPartial(out.unique_reads, out.unique_writes, out.footprint, np.array(out.level_sum[:]),
                             np.ctypeslib.as_array(out.cnt_hist0, shape=(CBINS,)).copy(), big)
