"""Per-event accumulator fields, materialised on demand.

The reference's KernelAccumulator holds Python lists and Counters built event
by event (pkg/src/aiwc/metrics.py:110-196): ``itb_samples`` / ``ipt_samples``
in stream order, ``read_addresses`` / ``write_addresses`` Counters in
first-appearance order, and ``branch_records`` = site -> [(group, bits)].
The engine never needs them -- finalize runs from the device's exact tables --
so they are rebuilt here, only when a caller reads them, from the columns the
accumulator was consumed from.  Vectorised numpy over the columnar trace; this
is API parity for inspection-sized traces, not part of the metric path.
"""

from __future__ import annotations

from collections import Counter

import numpy as np

from .trace import (K_BARRIER, K_BRANCH, K_INSTR, K_WG_BEGIN, K_WI_BEGIN, K_WI_END, K_WI_RESUME, ColumnarTrace)

FIELDS = ("itb_samples", "ipt_samples", "read_addresses", "write_addresses", "branch_records")


def _counter_in_first_order(addrs: np.ndarray) -> Counter:
    if not addrs.size:
        return Counter()
    u, first, cnt = np.unique(addrs, return_index=True, return_counts=True)
    order = np.argsort(first, kind="stable")
    return Counter(dict(zip(u[order].tolist(), cnt[order].tolist())))


def materialize(tr: ColumnarTrace) -> dict:
    """The five per-event fields of one consumed (valid) trace."""
    t = tr.to_numpy()
    k = np.ascontiguousarray(t.kind, dtype=np.uint8)
    p = np.ascontiguousarray(t.payload).view(np.uint64)

    # segments (metrics.py:131-133,156-174): a close (barrier / wi_end) ends the
    # segment opened by the latest wi_begin / wi_resume; segments never interleave
    instr_cum = np.cumsum(k == K_INSTR, dtype=np.int64)
    opens = np.flatnonzero((k == K_WI_BEGIN) | (k == K_WI_RESUME))
    closes = np.flatnonzero((k == K_BARRIER) | (k == K_WI_END))
    if closes.size:
        oi = np.searchsorted(opens, closes) - 1
        seg = instr_cum[closes] - instr_cum[opens[oi]]
        is_bar = k[closes] == K_BARRIER
        itb = seg[is_bar | (seg > 0)]
        # IPT: a work-item's lifetime is (group sequence, local id) of its opens;
        # the sample is the lifetime total at its wi_end, in wi_end order
        gseq = np.cumsum(k == K_WG_BEGIN, dtype=np.int64)
        life = (gseq[opens[oi]].astype(np.uint64) << np.uint64(32)) | (p[opens[oi]] & np.uint64(0xFFFFFFFF))
        _, inv = np.unique(life, return_inverse=True)
        totals = np.zeros(int(inv.max()) + 1, dtype=np.int64)
        np.add.at(totals, inv, seg)
        ipt = totals[inv[~is_bar]]
    else:
        itb = ipt = np.zeros(0, dtype=np.int64)

    # memory (metrics.py:137-144): atomics fold into reads / writes
    reads = _counter_in_first_order(p[(k & 0x7F) == 0x02])
    writes = _counter_in_first_order(p[(k & 0x7F) == 0x04])

    # branch streams (metrics.py:145-155): per site in first-appearance order, one
    # (group, bits) stream per consecutive run of the same group
    records: dict = {}
    bi = np.flatnonzero(k == K_BRANCH)
    if bi.size:
        site = p[bi] >> np.uint64(1)
        bits = (p[bi] & np.uint64(1)).astype(np.int64)
        wgb = np.flatnonzero(k == K_WG_BEGIN)
        gpos = np.searchsorted(wgb, bi) - 1
        gkey = np.where(gpos >= 0, p[wgb[np.maximum(gpos, 0)]], np.uint64(2**63))
        su, sfirst, sinv = np.unique(site, return_index=True, return_inverse=True)
        rank = np.empty(su.size, dtype=np.int64)
        rank[np.argsort(sfirst, kind="stable")] = np.arange(su.size)
        order = np.lexsort((bi, rank[sinv]))
        s_o, g_o, b_o = site[order], gkey[order], bits[order]
        cut = np.flatnonzero((s_o[1:] != s_o[:-1]) | (g_o[1:] != g_o[:-1])) + 1
        starts = np.concatenate([[0], cut])
        ends = np.concatenate([cut, [s_o.size]])
        for a, b in zip(starts.tolist(), ends.tolist()):
            g = int(g_o[a])
            group = tr.group_of_key(g) if g != 2**63 else None
            records.setdefault(int(s_o[a]), []).append((group, b_o[a:b].tolist()))
    return {"itb_samples": itb.tolist(), "ipt_samples": ipt.tolist(), "read_addresses": reads,
            "write_addresses": writes, "branch_records": records}


def merge_fields(parts: list[dict]) -> dict:
    """The reference's merge of the same fields (metrics.py:252-262)."""
    out = {"itb_samples": [], "ipt_samples": [], "read_addresses": Counter(), "write_addresses": Counter(),
           "branch_records": {}}
    for f in parts:
        out["itb_samples"].extend(f["itb_samples"])
        out["ipt_samples"].extend(f["ipt_samples"])
        out["read_addresses"].update(f["read_addresses"])
        out["write_addresses"].update(f["write_addresses"])
        for site, streams in f["branch_records"].items():
            out["branch_records"].setdefault(site, []).extend(streams)
    return out
