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
import os
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


PROFILE = os.environ.get("AIWC_SHARD_PROFILE") == "1"  # section timings of sharded_result (synchronizing)
LAST_PROFILE: dict = {}


class _Sections:
    """Wall-clock sections of one sharded_result with a device sync at each mark
    (measurement only: AIWC_SHARD_PROFILE=1)."""

    def __init__(self, device):
        import time

        self.t = time.perf_counter
        self.device = device
        self.last = self.t() if PROFILE else 0.0
        LAST_PROFILE.clear()

    def mark(self, name: str) -> None:
        if not PROFILE:
            return
        import torch

        if self.device.type == "cuda":
            torch.cuda.synchronize(self.device)
        now = self.t()
        LAST_PROFILE[name] = LAST_PROFILE.get(name, 0.0) + (now - self.last) * 1e3
        self.last = now


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


def combine_stats(rows) -> tuple:
    """The job's aiwc_shard_stats from every rank's: (min, max, and, or) over ranks
    with accesses, the summed access count, the smallest dense-table budget, the
    summed branch count."""
    rows = [tuple(int(v) for v in r) for r in rows]
    live = [r for r in rows if r[4]]
    m = sum(r[4] for r in rows)
    budget = min(r[5] for r in rows)
    n_br = sum(r[6] for r in rows)
    if not live:
        return ((1 << 64) - 1, 0, (1 << 64) - 1, 0, 0, budget, n_br)
    aand, aor = (1 << 64) - 1, 0
    for r in live:
        aand &= r[2]
        aor |= r[3]
    return (min(r[0] for r in live), max(r[1] for r in live), aand, aor, m, budget, n_br)


def chunk_owner(all_bits: np.ndarray, c: int) -> int:
    """Owner of 1024-key chunk c (aiwc_internal.cuh chunk_owner): the only rank that
    touched it, else a hash of its index."""
    nranks = all_bits.shape[0]
    w, b = c >> 5, np.uint32(1 << (c & 31))
    touched = [r for r in range(nranks) if int(all_bits[r, w]) & int(b)]
    if len(touched) == 1:
        return touched[0]
    m32 = 0xFFFFFFFF
    h = ((c * 0x9E3779B1) & m32) ^ ((c >> 32) & m32)
    h ^= h >> 15
    h = (h * 0x85EBCA77) & m32
    h ^= h >> 13
    return h % nranks


def _all_gather_u64(vals: np.ndarray, group, device) -> np.ndarray:
    """[world, len] of every rank's equal-length u64 vector (one all-gather)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    mine = torch.from_numpy(np.ascontiguousarray(vals, dtype=np.uint64).view(np.int64).copy()).to(device)
    out = torch.empty(world * mine.numel(), dtype=torch.int64, device=device)  # flat: gloo and NCCL alike
    dist.all_gather_into_tensor(out, mine, group=group)
    return out.cpu().numpy().view(np.uint64).reshape(world, -1)


def sharded_result(backend, shard, shard_offset: int, group=None):
    """Every rank: exact whole-trace EngineResult from its work-group shard.

    1. pass 1 of the shard; one all-gather of every rank's address statistics and
       access count fixes the job's key map;
    2. the ingest fills a dense table over that key map (the single-GPU ingest) and
       marks the 1024-key chunks it touched; one all-gather of the chunk bitmaps;
    3. chunks several ranks touched travel to their owner as runs of equal table
       entries (one all-to-all); the owner sweeps its chunks with the single-GPU
       statistics kernel;
    4. one device all-reduce of a packed u64 buffer (scalars, opcode / ITB / IPT /
       count-of-counts histograms, the 2^H branch pattern table) and one all-gather
       of the variable parts (overflow lists, width / site lists, fp64 level sums,
       added in rank order).
    A job whose key span does not fit a dense table keeps its addresses compacted
    and exchanges them with key-range owners (runs or raw addresses)."""
    import torch.distributed as dist

    global LAST_EXCHANGE
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    device = comm_device(backend, group)
    sec = _Sections(getattr(backend, "device", device))
    local = backend.prepare(shard, shard_offset)
    sec.mark("prepare")
    job = combine_stats(_all_gather_u64(np.array(local, np.uint64), group, device))
    sec.mark("stats_allgather")
    dense = backend.ingest(job)
    sec.mark("ingest")
    sp: ShardPartial = backend.finish()
    sec.mark("finalize")
    total_m = job[4]
    if total_m and dense:
        LAST_EXCHANGE = "dense"
        bits = backend.chunk_bits()
        all_bits = _all_gather_u32(bits, group, device)
        sec.mark("bitmap_allgather")
        runs, rcounts = backend.pack(all_bits, rank, world)
        sec.mark("pack")
        recv, n_words = exchange(runs, [2 * c for c in rcounts], group, device)
        sec.mark("alltoall")
        mp = backend.owned(recv, n_words // 2, all_bits, rank, world, total_m)
        sec.mark("owned")
    elif total_m:
        km = key_map(job[:4], world)
        lo, n_owned = km.owned(rank)
        use_runs = False
        if hasattr(backend, "partition_runs") and runs_dense_ok(km, total_m):
            # pre-aggregation: runs of consecutive keys per owner; chosen (on every
            # rank alike) when runs average >= RUN_MIN_AVG accesses
            runs, rcounts = backend.partition_runs(sp, km, world)
            tot = _allreduce_i64(np.array([sum(rcounts)], np.uint64), dist.ReduceOp.SUM, group, device)
            use_runs = RUN_MIN_AVG * int(tot[0]) <= total_m
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

    # ---- one packed all-reduce: every summable integer (the 2^H branch pattern table
    # only when the job has branches), plus every rank's list lengths in its own row
    # of a [world, 5] block (zeros elsewhere), so the sum hands everyone all lengths ----
    n_opc = len(sp.opcode_counts)
    scalars = np.array([sp.n_events, sp.total_instructions, sp.work_items, sp.barriers_hit, sp.total_reads,
                        sp.total_writes, sp.itb_sum, sp.ipt_sum, sp.branch_executions, mp.unique_reads,
                        mp.unique_writes, mp.footprint], dtype=np.uint64)
    lens = np.zeros((world, 5), np.uint64)
    lens[rank] = (len(sp.itb_ovf), len(sp.ipt_ovf), len(mp.big), len(sp.widths), len(sp.sites))
    has_br = job[6] > 0
    packed = np.concatenate([scalars, np.asarray(sp.opcode_counts, np.uint64), np.asarray(sp.itb_hist, np.uint64),
                             np.asarray(sp.ipt_hist, np.uint64), np.asarray(mp.cnt_hist0, np.uint64),
                             lens.reshape(-1), np.asarray(sp.branch_table, np.uint64) if has_br else
                             np.zeros(0, np.uint64)])
    tot = _allreduce_i64(packed, dist.ReduceOp.SUM, group, device)
    sec.mark("packed_allreduce")
    o = 0

    def take(n):
        nonlocal o
        o += n
        return tot[o - n:o]

    (n_events, total_instr, work_items, barriers, total_reads, total_writes, itb_sum, ipt_sum, br_exec, unique_r,
     unique_w, footprint) = (int(v) for v in take(len(scalars)))
    opcode_counts = [int(v) for v in take(n_opc)]
    itb_hist, ipt_hist, hist0 = take(HBINS).copy(), take(HBINS).copy(), take(CBINS).copy()
    all_lens = take(5 * world).reshape(world, 5).astype(np.int64)
    branch_table = take(len(sp.branch_table)).copy() if has_br else np.zeros(len(sp.branch_table), np.uint64)

    # ---- one all-gather of the variable parts (blobs padded to the longest) ----
    blob = np.concatenate([
        np.asarray(mp.level_sum, np.float64).view(np.uint64),
        np.asarray(sp.itb_ovf, np.uint64), np.asarray(sp.ipt_ovf, np.uint64), np.asarray(mp.big, np.uint64),
        np.array([v for w in sp.widths for v in w], np.uint64),
        np.array([v for it in sorted(sp.sites.items()) for v in it], np.uint64)])
    level_sum = np.zeros(11)
    lists, bigs = [], []
    width = int(max(11 + n[0] + n[1] + n[2] + 3 * n[3] + 2 * n[4] for n in all_lens))
    padded = np.zeros(width, np.uint64)
    padded[:blob.size] = blob
    for r, b in enumerate(_all_gather_u64(padded, group, device)):
        n_i, n_p, n_b, n_w, n_s = (int(v) for v in all_lens[r])
        level_sum = level_sum + b[:11].view(np.float64)  # rank order: deterministic
        q = 11
        itb_o = b[q:q + n_i]; q += n_i
        ipt_o = b[q:q + n_p]; q += n_p
        bigs.append(b[q:q + n_b]); q += n_b
        widths = [tuple(int(x) for x in b[q + 3 * i:q + 3 * i + 3]) for i in range(n_w)]; q += 3 * n_w
        sites = {int(b[q + 2 * i]): int(b[q + 2 * i + 1]) for i in range(n_s)}
        lists.append((itb_o.tolist(), ipt_o.tolist(), widths, sites))
    itb_ovf, ipt_ovf, widths, sites = _merge_lists(lists)
    big = np.sort(np.concatenate(bigs).astype(np.uint64))[::-1]
    sec.mark("lists_allgather")
    return _assemble(n_events, total_instr, work_items, barriers, total_reads, total_writes, itb_sum, ipt_sum,
                     br_exec, opcode_counts, itb_hist, itb_ovf, ipt_hist, ipt_ovf, branch_table, widths, sites,
                     unique_r, unique_w, footprint, hist0, big, level_sum)


def _all_gather_u32(bits, group, device) -> object:
    """[world, words] int32 tensor of every rank's chunk bitmap (on the collective device)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    mine = bits.to(device)
    out = torch.empty(world * mine.numel(), dtype=mine.dtype, device=device)
    dist.all_gather_into_tensor(out, mine.contiguous(), group=group)
    return out.view(world, -1)


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


def _check_groups_unique_across(tr, cuts: list[int]) -> None:
    """A (site, group) branch stream continues across work-groups that repeat the
    group id (metrics.py:145-152 keys streams by group): split at a cut it would
    become two streams.  Chunks that share a work-group id are refused."""
    from .errors import UnsupportedTrace
    from .trace import K_WG_BEGIN

    if len(cuts) <= 2:
        return
    if type(tr.kind).__module__.startswith("torch"):
        import torch

        keys = []
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            k = tr.kind[lo:hi]
            keys.append(torch.unique(tr.payload[lo:hi][k == K_WG_BEGIN]))
        allk = torch.cat(keys)
        repeated = int(torch.unique(allk).numel()) != int(allk.numel())
    else:
        kind, pay = np.asarray(tr.kind), np.asarray(tr.payload)
        keys = [np.unique(pay[lo:hi][kind[lo:hi] == K_WG_BEGIN]) for lo, hi in zip(cuts[:-1], cuts[1:])]
        allk = np.concatenate(keys)
        repeated = np.unique(allk).size != allk.size
    if repeated:
        raise UnsupportedTrace("a work-group id repeats in more than one ingest chunk: its branch streams would split "
                               "at the cut")


def chunked_result(backend, tr, cuts: list[int]):
    """One trace larger than one ingest allows, on one GPU: each chunk (whole
    work-groups) is a shard pass; sums and lists combine as across ranks, and the
    chunks' compacted addresses are finished by one owner (this GPU)."""
    import torch

    from .trace import ColumnarTrace

    _check_groups_unique_across(tr, cuts)
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
# job mode: NCCL inside the engine (aiwc_ctx_set_comm) -- the multi-GPU product path
# ---------------------------------------------------------------------------
class NcclJob:
    """One engine context joined to the job's NCCL communicator.  torch.distributed
    only bootstraps it (rank 0's ncclUniqueId is broadcast once); from then on
    `result` is aiwc_ingest of this rank's shard + aiwc_finalize, and every
    collective of the exchange and the combine runs inside the engine (no Python
    between them).  One NcclJob per concurrent trace stream (its own communicator)."""

    def __init__(self, device_index: int = 0, group=None, timing: bool = False, dense_budget_bytes: int = 0):
        import torch.distributed as dist

        from . import _native

        self.device_index = device_index
        flags = _native.OPT_NO_CONSERVATION | (_native.OPT_TIMING if timing else 0)
        # dense_budget_bytes=1 (tests) forces the compacted-address exchange
        self.ctx = _native.Context(device_index, flags=flags, dense_budget_bytes=dense_budget_bytes)
        lib = self.ctx.lib
        uid = (ctypes.c_uint8 * 128)()
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        if rank == 0:
            self.ctx.check(lib.aiwc_nccl_unique_id(uid))
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        uid = (ctypes.c_uint8 * 128).from_buffer_copy(box[0])
        import torch

        torch.cuda.set_device(device_index)
        self.ctx.check(lib.aiwc_ctx_set_comm(self.ctx.h, uid, rank, world))
        self.rank, self.world = rank, world
        self.last_phase_ms: list = []
        self.last_d2h = 0
        self.launches = 0

    def result(self, shard, shard_offset: int):
        """The whole job's EngineResult from this rank's work-group shard."""
        from . import _native
        from .metrics import _copy_result, _is_torch, trace_info

        ctx = self.ctx
        lib = ctx.lib
        ctx.check(lib.aiwc_reset(ctx.h))
        info = trace_info(shard)
        info.first_event = shard_offset
        kind, payload = shard.kind, shard.payload
        if _is_torch(kind) and kind.is_cuda:
            import torch

            kind, payload = kind.contiguous(), payload.contiguous()
            stream = torch.cuda.current_stream(kind.device).cuda_stream
            ctx.check(lib.aiwc_ingest(ctx.h, ctypes.c_void_p(kind.data_ptr()), ctypes.c_void_p(payload.data_ptr()),
                                      ctypes.byref(info), ctypes.c_void_p(stream)))
        else:
            if _is_torch(kind):
                kind, payload = kind.numpy(), payload.numpy()
            kind = np.ascontiguousarray(kind, dtype=np.uint8)
            payload = np.ascontiguousarray(payload).view(np.uint64)
            import torch

            stream = torch.cuda.current_stream(self.device_index).cuda_stream
            ctx.check(lib.aiwc_ingest_host(ctx.h, kind.ctypes.data_as(ctypes.c_void_p),
                                           payload.ctypes.data_as(ctypes.c_void_p), ctypes.byref(info),
                                           ctypes.c_void_p(stream)))
        res = _native.Result()
        ctx.check(lib.aiwc_finalize(ctx.h, ctypes.byref(res), ctypes.c_void_p(stream)))
        self.last_phase_ms = list(res.phase_ms)
        self.last_d2h = res.d2h_bytes
        self.launches += res.kernels_launched
        return _copy_result(res)

    def report(self, shard, shard_offset: int, kernel_name: str, invocation: int, global_size, local_size,
               opcodes: list[str]):
        """AiwcReport of the whole trace, identical on every rank."""
        from .metrics import KernelAccumulator, finalize

        res = self.result(shard, shard_offset)
        acc = KernelAccumulator(kernel_name, [invocation], [(invocation, tuple(global_size), tuple(local_size))], res,
                                list(opcodes))
        return finalize(acc)

    def close(self):
        self.ctx.close()


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
    force_compact: bool = False  # tests: take the compacted-address exchange even when a dense table fits
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

    # ---- the dense exchange (aiwc_shard_*) ----
    def prepare(self, tr, shard_offset: int) -> tuple:
        """Pass 1 of the shard (device columns; host columns are copied first): its
        aiwc_shard_stats as six ints."""
        import torch

        from . import _native
        from .metrics import _device_columns, trace_info

        ctx = self._ctx()
        ctx.check(ctx.lib.aiwc_reset(ctx.h))
        dtr = _device_columns(tr, self.device_index)
        kind, payload = dtr.kind.contiguous(), dtr.payload.contiguous()
        if kind.data_ptr() % 16:
            kind = kind.clone()
        if payload.data_ptr() % 16:
            payload = payload.clone()
        self._cols = (kind, payload)  # alive until the ingest has run
        self._offset = shard_offset
        self._stream = torch.cuda.current_stream(self.device).cuda_stream
        out = _native.ShardStats()
        info = trace_info(dtr)
        ctx.check(ctx.lib.aiwc_shard_prepare(ctx.h, ctypes.c_void_p(kind.data_ptr()), ctypes.c_void_p(payload.data_ptr()),
                                             ctypes.byref(info), ctypes.byref(out), ctypes.c_void_p(self._stream)))
        return (out.addr_min, out.addr_max, out.addr_and, out.addr_or, out.n_accesses, out.dense_budget_bytes,
                out.n_branches)

    def ingest(self, job: tuple) -> bool:
        from . import _native

        ctx = self._ctx()
        st = _native.ShardStats(*[int(v) for v in job[:5]], 0 if self.force_compact else int(job[5]), int(job[6]))
        dense = ctypes.c_uint32(0)
        ctx.check(ctx.lib.aiwc_shard_ingest(ctx.h, ctypes.byref(st), ctypes.byref(dense), ctypes.c_void_p(self._stream)))
        return bool(dense.value)

    def finish(self) -> ShardPartial:
        from . import _native

        ctx = self._ctx()
        res = _native.Result()
        ctx.check(ctx.lib.aiwc_finalize(ctx.h, ctypes.byref(res), ctypes.c_void_p(self._stream)))
        self._cols = None
        return self._partial(res, self._offset)

    def chunk_bits(self):
        import torch

        ctx = self._ctx()
        p, n = ctypes.c_void_p(), ctypes.c_uint64()
        ctx.check(ctx.lib.aiwc_shard_chunks(ctx.h, ctypes.byref(p), ctypes.byref(n)))
        iface = {"shape": (max(int(n.value), 1),), "typestr": "<i4", "data": (p.value, False), "version": 3}
        holder = type("_Bits", (), {"__cuda_array_interface__": iface})()
        return torch.as_tensor(holder, device=self.device)[: int(n.value)]

    def pack(self, all_bits, rank: int, nranks: int):
        import torch

        ctx = self._ctx()
        all_bits = all_bits.to(self.device).contiguous()
        counts = (ctypes.c_uint64 * nranks)()
        rp = ctypes.c_void_p()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        ctx.check(ctx.lib.aiwc_shard_pack(ctx.h, ctypes.c_void_p(all_bits.data_ptr()), rank, nranks, ctypes.byref(rp),
                                          counts, ctypes.c_void_p(stream)))
        c = [int(x) for x in counts]
        self.launches += 1 + int(sum(c) > 0)
        runs = torch.as_tensor(_CudaArray(rp.value, max(2 * sum(c), 1)), device=self.device)
        return runs, c

    def owned(self, recv, n_runs: int, all_bits, rank: int, nranks: int, total_m: int) -> MemoryPartial:
        import torch

        from . import _native

        ctx = self._ctx()
        out = _native.MemoryPart()
        recv = recv.to(self.device)
        all_bits = all_bits.to(self.device).contiguous()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        ctx.check(ctx.lib.aiwc_shard_owned(ctx.h, ctypes.c_void_p(recv.data_ptr()), n_runs,
                                           ctypes.c_void_p(all_bits.data_ptr()), rank, nranks, total_m,
                                           ctypes.byref(out), ctypes.c_void_p(stream)))
        self.launches += out.kernels_launched
        big = np.ctypeslib.as_array(out.big, shape=(out.n_big,)).copy() if out.n_big else np.zeros(0, np.uint64)
        return MemoryPartial(out.unique_reads, out.unique_writes, out.footprint, np.array(out.level_sum[:]),
                             np.ctypeslib.as_array(out.cnt_hist0, shape=(CBINS,)).copy(), big)

    def _partial(self, res, shard_offset: int) -> ShardPartial:
        from . import _native
        from .metrics import _copy_result

        ctx = self._ctx()
        self.last_phase_ms = list(res.phase_ms)
        self.last_d2h = res.d2h_bytes
        self.launches += res.kernels_launched
        r = _copy_result(res)
        t = _native.ShardTables()
        ctx.check(ctx.lib.aiwc_shard_tables_get(ctx.h, ctypes.byref(t)))
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

    # ---- one ingest of a whole (sub)trace in shard mode: compacted addresses (chunked_result) ----
    def shard(self, tr, shard_offset: int) -> ShardPartial:
        from . import _native
        from .metrics import ingest_columns

        ctx = self._ctx()
        lib = ctx.lib
        ctx.check(lib.aiwc_reset(ctx.h))
        stream = ingest_columns(ctx, tr)
        res = _native.Result()
        ctx.check(lib.aiwc_finalize(ctx.h, ctypes.byref(res), ctypes.c_void_p(stream) if stream else None))
        return self._partial(res, shard_offset)

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
