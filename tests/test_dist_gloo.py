"""Multi-rank path on CPU: two gloo ranks, each holding one work-group shard
of a golden trace, run paper_1805_04207_b200.dist (address statistics
all-reduce, key-range owners, all-to-all of addresses, owner partials,
exact combine).  The engine steps are served by an oracle-backed test
backend; the combined report must equal the reference's own report."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import ROOT, assert_report_matches, golden_cases

CASES = ["wavefront_big", "bfs_flags", "sweep4", "long_segments", "hot_address", "random31337_3", "random202_5",
         "coin_20k", "offgrid_groups", "branch_streams_per_group"]


class OracleBackend:
    """Test double for dist.CudaBackend: the C oracle's accumulator + numpy.  The
    dense exchange keeps a {key: (reads, writes)} table over the job's key map and
    packs every key of a chunk owned elsewhere as a one-key run (runs need not be
    maximal); force_compact takes the compacted-address exchange instead."""

    device = torch.device("cpu")

    def __init__(self, n_opcodes, force_compact=False):
        self.n_opcodes = n_opcodes
        self.force_compact = force_compact

    # ---- dense exchange ----
    def prepare(self, tr, offset):
        self.sp = self.shard(tr, offset)
        m = self.sp.total_reads + self.sp.total_writes
        st = self.sp.addr_stats or ((1 << 64) - 1, 0, (1 << 64) - 1, 0)
        return (*st, m, 1 << 40, self.sp.branch_executions)

    def ingest(self, job):
        from paper_1805_04207_b200.dist import key_map

        self.km = key_map(job[:4], 1)
        m = job[4]
        if self.force_compact or not m or self.km.n_keys > 4 * m + (1 << 20) or self.km.n_keys >= (1 << 31) - 2:
            return False
        rd_a, rd_c, wr_a, wr_c = self.sp.handle
        tab = {}
        for a, c, w in ((rd_a, rd_c, 0), (wr_a, wr_c, 1)):
            for key, n in zip(((a - np.uint64(self.km.base)) >> np.uint64(self.km.k)).tolist(), c.tolist()):
                r0, w0 = tab.get(key, (0, 0))
                tab[key] = (r0 + (0 if w else n), w0 + (n if w else 0))
        self.tab = tab
        return True

    def finish(self):
        return self.sp

    def chunk_bits(self):
        words = ((self.km.n_keys + 1 + 1023) // 1024 + 31) // 32
        bits = np.zeros(words, np.uint32)
        for key in self.tab:
            c = key >> 10
            bits[c >> 5] |= np.uint32(1 << (c & 31))
        return torch.from_numpy(bits.view(np.int32).copy())

    def pack(self, all_bits, rank, nranks):
        from paper_1805_04207_b200.dist import chunk_owner

        ab = all_bits.numpy().view(np.uint32)
        by_owner = [[] for _ in range(nranks)]
        for key in sorted(self.tab):
            o = chunk_owner(ab, key >> 10)
            if o != rank:
                r, w = self.tab[key]
                by_owner[o].append((key | (1 << 32), r | (w << 32)))
        flat = [v for lst in by_owner for run in lst for v in run]
        arr = np.array(flat, dtype=np.uint64) if flat else np.zeros(1, np.uint64)
        return torch.from_numpy(arr.view(np.int64).copy()), [len(lst) for lst in by_owner]

    def owned(self, recv, n_runs, all_bits, rank, nranks, total_m):
        from paper_1805_04207_b200.dist import chunk_owner

        ab = all_bits.numpy().view(np.uint32)
        tot = {k: v for k, v in self.tab.items() if chunk_owner(ab, k >> 10) == rank}
        r = recv[: 2 * n_runs].numpy().view(np.uint64).reshape(-1, 2)
        for w0, v in r.tolist():
            key, n = w0 & 0xFFFFFFFF, w0 >> 32
            assert chunk_owner(ab, key >> 10) == rank
            for i in range(n):
                r0, w_0 = tot.get(key + i, (0, 0))
                tot[key + i] = (r0 + (v & 0xFFFFFFFF), w_0 + (v >> 32))
        return self._partial_from_counts(tot, self.km, total_m)

    def _partial_from_counts(self, tot, km, total_m):
        from paper_1805_04207_b200.dist import CBINS, MemoryPartial

        keys = np.array(sorted(tot), dtype=np.uint64)
        rw = np.array([tot[int(k)] for k in keys], dtype=np.int64).reshape(-1, 2)
        c = rw.sum(axis=1) if keys.size else np.zeros(0, np.int64)
        sums = []
        for lvl in range(11):
            j = max(0, lvl - km.k)
            if not keys.size:
                sums.append(0.0)
                continue
            g = np.unique(keys >> np.uint64(j), return_inverse=True)[1]
            p = np.bincount(g, weights=c) / total_m
            sums.append(float((p * np.log2(p)).sum()))
        return MemoryPartial(int((rw[:, 0] > 0).sum()) if keys.size else 0, int((rw[:, 1] > 0).sum()) if keys.size else 0,
                             int(keys.size), np.array(sums), np.bincount(c[c < CBINS], minlength=CBINS).astype(np.uint64),
                             c[c >= CBINS].astype(np.uint64))

    def shard(self, tr, offset):
        from oracle import oracle
        from paper_1805_04207_b200.dist import HBINS, ShardPartial

        acc = oracle.accumulator(tr.kind, tr.payload, self.n_opcodes)

        def hist(v):
            v = v.astype(np.int64)
            return (np.bincount(v[v < HBINS], minlength=HBINS).astype(np.uint64), np.sort(v[v >= HBINS]).astype(np.uint64))

        ih, io = hist(acc["itb"])
        ph, po = hist(acc["ipt"])
        rd_a, rd_c = acc["rd"]
        wr_a, wr_c = acc["wr"]
        addrs = np.concatenate([rd_a, wr_a])
        stats = None
        if addrs.size:
            stats = (int(addrs.min()), int(addrs.max()), int(np.bitwise_and.reduce(addrs)), int(np.bitwise_or.reduce(addrs)))
        table = (acc["total"].astype(np.uint64) << np.uint64(32)) | acc["taken"].astype(np.uint64)
        return ShardPartial(
            n_events=tr.n_events, total_instructions=acc["total_instructions"], work_items=acc["work_items"],
            barriers_hit=acc["barriers"], total_reads=int(rd_c.sum()), total_writes=int(wr_c.sum()),
            opcode_counts=acc["opc"], widths=[(w, c, f + offset) for w, c, f in acc["widths"]],
            itb_hist=ih, itb_ovf=io, itb_sum=int(acc["itb"].sum()), ipt_hist=ph, ipt_ovf=po,
            ipt_sum=int(acc["ipt"].sum()), branch_table=table, sites=acc["sites"], branch_executions=acc["executions"],
            addr_stats=stats, handle=(rd_a, rd_c, wr_a, wr_c))

    def partition(self, sp, km, nranks):
        rd_a, rd_c, wr_a, wr_c = sp.handle
        out, counts = [], []
        for a, c in ((rd_a, rd_c), (wr_a, wr_c)):
            a = np.repeat(a, c.astype(np.int64))
            keys = (a - np.uint64(km.base)) >> np.uint64(km.k)
            own = np.minimum(keys // np.uint64(km.keys_per_rank), np.uint64(nranks - 1)).astype(np.int64)
            order = np.argsort(own, kind="stable")
            out.append(torch.from_numpy(a[order].view(np.int64).copy()))
            counts += np.bincount(own, minlength=nranks).tolist()
        return out[0], out[1], counts

    def partition_runs(self, sp, km, nranks):
        """Runs of consecutive keys with one owner (the engine's aiwc_partition_runs)."""
        rd_a, rd_c, wr_a, wr_c = sp.handle
        runs = []
        for w, (a, c) in enumerate(((rd_a, rd_c), (wr_a, wr_c))):
            a = np.sort(np.repeat(a, c.astype(np.int64)))  # the oracle's address order is arbitrary
            if not a.size:
                continue
            keys = ((a - np.uint64(km.base)) >> np.uint64(km.k)).astype(np.int64)
            own = np.minimum(keys // km.keys_per_rank, nranks - 1)
            idx = np.arange(keys.size)
            head = np.ones(keys.size, bool)
            head[1:] = (keys[1:] != keys[:-1] + 1) | (own[1:] != own[:-1]) | (idx[1:] % 65536 == 0)
            hp = np.nonzero(head)[0]
            lens = np.diff(np.append(hp, keys.size))
            for h, n in zip(hp, lens):
                runs.append((int(own[h]), int(keys[h]), int(n) | (w << 63)))
        runs.sort(key=lambda r: r[0])  # owner-grouped
        flat = np.array([[k, lw] for _, k, lw in runs], dtype=np.uint64).reshape(-1)
        counts = np.bincount([r[0] for r in runs], minlength=nranks).tolist() if runs else [0] * nranks
        return torch.from_numpy(flat.view(np.int64).copy() if flat.size else np.zeros(1, np.int64)), counts

    def memory_partial_runs(self, recv, n_runs, km, lo, n_owned, total_m):
        r = recv[: 2 * n_runs].numpy().view(np.uint64).reshape(-1, 2)
        keys = [np.zeros(0, np.uint64), np.zeros(0, np.uint64)]
        for w in (0, 1):
            sel = r[(r[:, 1] >> np.uint64(63)) == np.uint64(w)]
            if sel.size:
                lens = (sel[:, 1] & np.uint64(0xFFFFFFFF)).astype(np.int64)
                starts = np.repeat(sel[:, 0], lens)
                offs = np.arange(lens.sum()) - np.repeat(np.cumsum(lens) - lens, lens)
                keys[w] = starts + offs.astype(np.uint64)
        return self._partial_from_keys(keys, km, lo, n_owned, total_m)

    def memory_partial(self, recv_r, n_r, recv_w, n_w, km, lo, n_owned, total_m):
        rd = recv_r[:n_r].numpy().view(np.uint64)
        wr = recv_w[:n_w].numpy().view(np.uint64)
        keys = [((a - np.uint64(km.base)) >> np.uint64(km.k)) for a in (rd, wr)]
        return self._partial_from_keys(keys, km, lo, n_owned, total_m)

    def _partial_from_keys(self, keys, km, lo, n_owned, total_m):
        from paper_1805_04207_b200.dist import CBINS, MemoryPartial

        for kk in keys:  # every received address belongs to this owner's key range
            assert ((kk >= np.uint64(lo)) & (kk - np.uint64(lo) < np.uint64(max(n_owned, 1)))).all()
        allk = np.concatenate(keys)
        uk, c = np.unique(allk, return_counts=True)
        sums = []
        for lvl in range(11):
            j = max(0, lvl - km.k)
            if not uk.size:
                sums.append(0.0)
                continue
            g = np.unique(uk >> np.uint64(j), return_inverse=True)[1]
            tot = np.bincount(g, weights=c)
            p = tot / total_m
            sums.append(float((p * np.log2(p)).sum()))
        return MemoryPartial(int(np.unique(keys[0]).size), int(np.unique(keys[1]).size), int(uk.size), np.array(sums),
                             np.bincount(c[c < CBINS], minlength=CBINS).astype(np.uint64),
                             c[c >= CBINS].astype(np.uint64))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, names, q):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    from conftest import golden_cases as gc
    from paper_1805_04207_b200 import dist as D
    from paper_1805_04207_b200 import report_to_dict
    from paper_1805_04207_b200.trace import ColumnarTrace, K_WG_BEGIN

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        by_name = {c["name"]: (c, t) for c, t in gc()}
        for name in names:
            c, tr = by_name[name]
            starts = np.nonzero(tr.kind == K_WG_BEGIN)[0]
            # contiguous work-group ranges, one per rank (a rank may get none)
            cuts = [0] + [int(starts[len(starts) * r // world]) for r in range(1, world)] + [tr.n_events]
            lo, hi = cuts[rank], cuts[rank + 1]
            shard = ColumnarTrace(tr.kind[lo:hi], tr.payload[lo:hi], tr.kernel_name, tr.invocation, tr.global_size,
                                  tr.local_size, tr.opcodes, tr.extra_groups)
            for compact in (False, True):
                rep = D.sharded_report(OracleBackend(len(tr.opcodes), compact), shard, lo, tr.kernel_name,
                                       tr.invocation, tr.global_size, tr.local_size, tr.opcodes)
                q.put((rank, name, report_to_dict(rep), D.LAST_EXCHANGE))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_reports_match_reference(world):
    from oracle import oracle

    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, CASES, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=240) for _ in range(2 * world * len(CASES))]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = {c["name"]: c["report"] for c, _ in golden_cases() if c["name"] in CASES}
    modes = set()
    for rank, name, rep, mode in got:
        assert_report_matches(rep, want[name])
        modes.add(mode)
    assert {"dense", "runs", "raw"} <= modes  # every address exchange was exercised


def test_key_map_owner_ranges_are_block_aligned():
    from paper_1805_04207_b200.dist import key_map

    km = key_map((4096 + 4, 4096 + 4 * 99999, 0, ~3 & ((1 << 64) - 1)), 3)
    assert km.k == 2 and km.keys_per_rank % 1024 == 0
    assert sum(km.owned(r)[1] for r in range(3)) == km.n_keys
