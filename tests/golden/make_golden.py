"""Generate the golden parity fixtures from the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package read-only from /root/reference/pkg/src (and
its own test helpers generators.py / reference.py), builds the traces the
reference's tests use, runs the reference's ``consume`` + ``finalize`` +
``derive`` on each, and writes:

    tests/golden/traces.npz     columnar traces (kind u8 / payload u64, concatenated)
    tests/golden/cases.json     per-trace header, dictionaries and the expected
                                reference report (or expected exception)

The columnar encoder below is deliberately a separate pure-Python
restatement of the layout in include/aiwc_b200.h, so the fixtures do not
depend on the product's native walker.  Nothing here runs on the GPU box.
"""

from __future__ import annotations

import json
import os
import random
import sys
from itertools import product

import numpy as np

REF = "/root/reference/pkg"
sys.path[:0] = [os.path.join(REF, "src"), os.path.join(REF, "tests")]

from aiwc import errors as E  # noqa: E402
from aiwc.buffers import make_buffer  # noqa: E402
from aiwc.ir import parse_kernel  # noqa: E402
from aiwc.metrics import consume, finalize  # noqa: E402
from aiwc.report import derive, emit_report, report_to_dict  # noqa: E402
from aiwc.sim import NDRangeConfig, simulate  # noqa: E402
from aiwc.trace import (  # noqa: E402
    Barrier, Branch, Instruction, KernelBegin, KernelEnd, Memory, WorkGroupBegin, WorkGroupEnd,
    WorkItemBegin, WorkItemEnd, WorkItemId, WorkItemResume,
)
from generators import random_events  # noqa: E402  (reference test helper)

OUT = os.path.dirname(os.path.abspath(__file__))

KIND = {"load": 0x02, "atomic_load": 0x82, "store": 0x04, "atomic_store": 0x84}


def encode(events):
    """Pure-Python columnar encoder (layout of include/aiwc_b200.h)."""
    hdr = events[0]
    gsz, lsz = hdr.global_size, hdr.local_size
    grid = tuple(-(-gsz[d] // lsz[d]) for d in range(3))
    n_grid = grid[0] * grid[1] * grid[2]
    opcodes: dict[str, int] = {}
    extra: dict[tuple, int] = {}

    def gkey(g):
        if all(g[d] < grid[d] for d in range(3)):
            return g[0] + grid[0] * (g[1] + grid[1] * g[2])
        if g not in extra:
            extra[g] = n_grid + len(extra)
        return extra[g]

    def lid(wi):
        l = wi.local_id
        return l[0] + lsz[0] * (l[1] + lsz[1] * l[2])

    kinds, pays = [], []
    for ev in events:
        t = type(ev)
        if t is Instruction:
            oid = opcodes.setdefault(ev.opcode, len(opcodes))
            kinds.append(0x01); pays.append((oid << 32) | ev.width)
        elif t is Memory:
            kinds.append(KIND[ev.op]); pays.append(ev.addr)
        elif t is Branch:
            kinds.append(0x08); pays.append((ev.site << 1) | int(ev.taken))
        elif t is Barrier:
            kinds.append(0x90); pays.append(0)
        elif t is WorkItemBegin:
            kinds.append(0x30); pays.append(lid(ev.work_item))
        elif t is WorkItemResume:
            kinds.append(0xB0); pays.append(lid(ev.work_item))
        elif t is WorkItemEnd:
            kinds.append(0x10); pays.append(lid(ev.work_item))
        elif t is WorkGroupBegin:
            kinds.append(0x40); pays.append(gkey(ev.group_id))
        elif t is WorkGroupEnd:
            kinds.append(0xC0); pays.append(gkey(ev.group_id))
        elif t is KernelBegin:
            kinds.append(0x20); pays.append(0)
        elif t is KernelEnd:
            kinds.append(0xA0); pays.append(0)
        else:
            raise TypeError(ev)
    meta = {
        "kernel": hdr.kernel_name, "invocation": hdr.invocation,
        "global_size": list(gsz), "local_size": list(lsz),
        "opcodes": sorted(opcodes, key=opcodes.get),
        "extra_groups": [list(g) for g in sorted(extra, key=extra.get)],
    }
    return np.array(kinds, np.uint8), np.array(pays, np.uint64), meta


def repr_events(events):
    """JSON-able event list: [class name, *fields] with nested tuples as lists."""
    def conv(x):
        if isinstance(x, tuple):
            return [conv(v) for v in x]
        return x
    return [[type(e).__name__, *[conv(v) for v in e]] for e in events]


def load_kernel(name):
    with open(os.path.join(REF, "kernels", name), encoding="utf-8") as fp:
        return parse_kernel(fp.read())


def sim(kernel, gsz, lsz, bufs):
    volume = gsz[0] * gsz[1] * gsz[2]
    cfg = NDRangeConfig(gsz, lsz, {k: make_buffer(v, volume) for k, v in bufs.items()})
    return simulate(load_kernel(kernel), cfg)


def sim_inv(kernel, n, invocation):
    from aiwc.sim import simulate as _sim

    cfg = NDRangeConfig((n, 1, 1), (min(n, 64), 1, 1), {"a": make_buffer("iota", n)})
    return _sim(load_kernel(kernel), cfg, invocation=invocation)


WI0 = WorkItemId((0, 0, 0), (0, 0, 0), (0, 0, 0))
WI1 = WorkItemId((1, 0, 0), (1, 0, 0), (0, 0, 0))


def stream(body, local=(2, 1, 1), name="k", invocation=0):
    return [KernelBegin(name, invocation, local, local), WorkGroupBegin((0, 0, 0)), *body,
            WorkGroupEnd((0, 0, 0)), KernelEnd()]


def one_item(inside, **kw):
    return stream([WorkItemBegin(WI0), *inside, WorkItemEnd(WI0)], local=(1, 1, 1), **kw)


def instrs(n, opcode="add", width=1):
    return [Instruction(opcode, width)] * n


def unit_cases():
    """Hand-built streams mirroring pkg/tests/test_metrics.py and SURVEY App. C."""
    c = {}
    c["single_item_no_barriers"] = one_item(instrs(10))
    c["segment_split"] = stream([WorkItemBegin(WI0), *instrs(25), Barrier(), WorkItemResume(WI0),
                                 *instrs(5), WorkItemEnd(WI0)], local=(1, 1, 1))
    c["two_items_ipt"] = stream([WorkItemBegin(WI0), *instrs(7), WorkItemEnd(WI0),
                                 WorkItemBegin(WI1), *instrs(13), WorkItemEnd(WI1)])
    c["empty_final_segment"] = stream([WorkItemBegin(WI0), *instrs(24), Instruction("barrier", 1), Barrier(),
                                       WorkItemResume(WI0), WorkItemEnd(WI0)], local=(1, 1, 1))
    c["atomics_folded"] = one_item([Instruction("aload", 1), Memory("atomic_load", 64),
                                    Instruction("astore", 1), Memory("atomic_store", 64),
                                    Instruction("load", 1), Memory("load", 128)])
    c["single_address_store"] = one_item([e for _ in range(100) for e in (Instruction("store", 1), Memory("store", 4096))])
    c["stride_sweep"] = one_item([e for i in range(1024) for e in (Instruction("load", 1), Memory("load", 4096 + 4 * i))])
    body = [WorkItemBegin(WI0)]
    for _ in range(4):
        body += instrs(24) + [Instruction("barrier", 1), Barrier(), WorkItemResume(WI0)]
    body += instrs(25) + [WorkItemEnd(WI0)]
    c["uniform_itb"] = stream(body, local=(1, 1, 1))
    c["no_writes"] = one_item([Instruction("load", 1), Memory("load", 8)])
    c["simd_stats"] = one_item([Instruction("add", 1), Instruction("fmul", 4), Instruction("mad", 4)])
    c["opcode_coverage"] = one_item(instrs(90, "add") + instrs(6, "mul") + instrs(4, "xor"))
    c["no_branches"] = one_item(instrs(3))
    c["short_branch_streams"] = one_item([Instruction("br", 1), Branch(4, True)] * 3)
    c["per_invocation_lmae"] = one_item([Instruction("load", 1), Memory("load", 4096)], invocation=3)
    wa = WorkItemId((0, 0, 0), (0, 0, 0), (0, 0, 0))
    wb = WorkItemId((1, 0, 0), (0, 0, 0), (1, 0, 0))
    c["branch_streams_per_group"] = [
        KernelBegin("k", 0, (2, 1, 1), (1, 1, 1)),
        WorkGroupBegin((0, 0, 0)), WorkItemBegin(wa), Instruction("br", 1), Branch(9, True), WorkItemEnd(wa), WorkGroupEnd((0, 0, 0)),
        WorkGroupBegin((1, 0, 0)), WorkItemBegin(wb), Instruction("br", 1), Branch(9, False), WorkItemEnd(wb), WorkGroupEnd((1, 0, 0)),
        KernelEnd()]
    # App. C #6: zero-length barrier segment is sampled, empty trailing is not
    c["zero_length_barrier_segment"] = stream([
        WorkItemBegin(WI0), Instruction("add", 1), Instruction("barrier", 1), Barrier(),
        WorkItemResume(WI0), Barrier(), WorkItemResume(WI0), Instruction("add", 1), WorkItemEnd(WI0)], local=(1, 1, 1))
    # App. C #8: repeated group id continues the site's history; WI tallies restart
    rep = [KernelBegin("rep", 0, (1, 1, 1), (1, 1, 1))]
    rng = random.Random(5)
    for _ in range(2):
        rep += [WorkGroupBegin((0, 0, 0)), WorkItemBegin(WI0)]
        for _ in range(10):
            rep += [Instruction("br", 1), Branch(3, rng.random() < 0.5)]
        rep += [WorkItemEnd(WI0), WorkGroupEnd((0, 0, 0))]
    rep.append(KernelEnd())
    c["repeated_group_id"] = rep
    # A, B, A group order with one site: the third block's stream continues the first
    aba = [KernelBegin("aba", 0, (2, 1, 1), (1, 1, 1))]
    bits = [rng.random() < 0.7 for _ in range(60)]
    for blk, g in enumerate(((0, 0, 0), (1, 0, 0), (0, 0, 0))):
        wi = WorkItemId(g, (0, 0, 0), g)
        aba += [WorkGroupBegin(g), WorkItemBegin(wi)]
        for b in bits[blk * 20:(blk + 1) * 20]:
            aba += [Instruction("br", 1), Branch(7 if blk != 1 else 8, b)]
        aba += [WorkItemEnd(wi), WorkGroupEnd(g)]
    aba.append(KernelEnd())
    c["group_aba"] = aba
    # groups outside the launch grid get dictionary keys
    og = [KernelBegin("offgrid", 0, (2, 1, 1), (1, 1, 1))]
    for g in ((5, 0, 0), (0, 0, 0), (5, 0, 0)):
        wi = WorkItemId(g, (0, 0, 0), g)
        og += [WorkGroupBegin(g), WorkItemBegin(wi), Instruction("br", 1), Branch(2, True),
               Instruction("store", 2), Memory("store", 4096 + g[0]), WorkItemEnd(wi), WorkGroupEnd(g)]
    og.append(KernelEnd())
    c["offgrid_groups"] = og
    # long always-taken / alternating streams (entropy 0) and a coin
    alt = [KernelBegin("alt", 0, (1, 1, 1), (1, 1, 1)), WorkGroupBegin((0, 0, 0)), WorkItemBegin(WI0)]
    for t in range(3000):
        alt += [Instruction("br", 1), Branch(1, t % 2 == 0), Instruction("br", 1), Branch(2, True)]
    alt += [WorkItemEnd(WI0), WorkGroupEnd((0, 0, 0)), KernelEnd()]
    c["alternating_and_always"] = alt
    coin = [KernelBegin("coin", 0, (1, 1, 1), (1, 1, 1)), WorkGroupBegin((0, 0, 0)), WorkItemBegin(WI0)]
    for _ in range(20000):
        coin += [Instruction("br", 1), Branch(11, rng.random() < 0.5)]
    coin += [WorkItemEnd(WI0), WorkGroupEnd((0, 0, 0)), KernelEnd()]
    c["coin_20k"] = coin
    # big counts: one hot address hit far more often than any histogram bin
    hot = [KernelBegin("hot", 0, (1, 1, 1), (1, 1, 1)), WorkGroupBegin((0, 0, 0)), WorkItemBegin(WI0)]
    for i in range(6000):
        hot += [Instruction("atomic", 1), Memory("atomic_store", 1 << 40), Instruction("load", 1), Memory("load", (1 << 40) + 4 * (i % 700))]
    hot += [WorkItemEnd(WI0), WorkGroupEnd((0, 0, 0)), KernelEnd()]
    c["hot_address"] = hot
    # extreme addresses / widths
    ext = [KernelBegin("ext", 0, (1, 1, 1), (1, 1, 1)), WorkGroupBegin((0, 0, 0)), WorkItemBegin(WI0)]
    for a in (0, 1, (1 << 64) - 1, (1 << 63), 4096, (1 << 64) - 1024, 12345678901234):
        ext += [Instruction("load", 1024), Memory("load", a), Instruction("st", 3), Memory("store", a ^ 1)]
    ext += [WorkItemEnd(WI0), WorkGroupEnd((0, 0, 0)), KernelEnd()]
    c["extreme_addresses"] = ext
    # long segments: ITB / IPT above any small histogram
    longseg = [KernelBegin("long", 0, (3, 1, 1), (3, 1, 1)), WorkGroupBegin((0, 0, 0))]
    wis = [WorkItemId((i, 0, 0), (i, 0, 0), (0, 0, 0)) for i in range(3)]
    for sec in range(3):
        for j, wi in enumerate(wis):
            longseg.append(WorkItemBegin(wi) if sec == 0 else WorkItemResume(wi))
            longseg += instrs(1500 * (j + 1) + 37 * sec, "fma", 2)
            longseg += [Instruction("barrier", 1), Barrier()] if sec < 2 else [WorkItemEnd(wi)]
    longseg += [WorkGroupEnd((0, 0, 0)), KernelEnd()]
    c["long_segments"] = longseg
    return c


def expected(events, cap=None):
    try:
        acc = consume(events, max_entries=cap)
        rep = finalize(acc)
    except E.TraceTooLarge as exc:
        return {"error": "TraceTooLarge", "entries": exc.entries, "cap": exc.cap}
    return {"report": report_to_dict(rep, derive(rep)),
            "json": emit_report(rep).decode("utf-8"), "csv": emit_report(rep, format="csv").decode("utf-8")}


def invalid_cases():
    """Streams violating one StreamChecker rule each (trace.py:278-286), with the
    reference's InvalidStream (event index, rule, message) or TraceTooLarge."""
    base = one_item(instrs(2) + [Instruction("load", 1), Memory("load", 64)])
    wi_b = WorkItemId((1, 0, 0), (1, 0, 0), (0, 0, 0))
    out = {
        "not_kernel_begin_first": [Instruction("add", 1)] + base,
        "empty": [],
        "event_after_end": base + [Instruction("add", 1)],
        "no_kernel_end": base[:-1],
        "duplicate_kernel_begin": base[:1] + base,
        "outside_segment_instr": base[:2] + [Instruction("add", 1)] + base[2:],
        "outside_segment_mem": base[:2] + [Memory("load", 4)] + base[2:],
        "outside_segment_branch": base[:2] + [Branch(3, True)] + base[2:],
        "outside_segment_barrier": base[:2] + [Barrier()] + base[2:],
        "kernel_end_open_group": base[:-2] + [KernelEnd()],
        "wg_begin_nested": base[:2] + [WorkGroupBegin((0, 0, 0))] + base[2:],
        "wg_end_mismatch": base[:-2] + [WorkGroupEnd((1, 0, 0)), KernelEnd()],
        "wg_end_open_segment": base[:-3] + [WorkGroupEnd((0, 0, 0)), KernelEnd()],
        "wi_outside_group": [base[0], WorkItemBegin(WI0)] + base[1:],
        "wi_other_group": [KernelBegin("k", 0, (2, 1, 1), (1, 1, 1)), WorkGroupBegin((0, 0, 0)),
                           WorkItemBegin(WorkItemId((1, 0, 0), (0, 0, 0), (1, 0, 0))), WorkItemEnd(WI0),
                           WorkGroupEnd((0, 0, 0)), KernelEnd()],
        "wi_local_range": [KernelBegin("k", 0, (2, 1, 1), (1, 1, 1)), WorkGroupBegin((0, 0, 0)),
                           WorkItemBegin(WorkItemId((1, 0, 0), (1, 0, 0), (0, 0, 0))), WorkItemEnd(WI0),
                           WorkGroupEnd((0, 0, 0)), KernelEnd()],
        "wi_gid_arith": [KernelBegin("k", 0, (2, 1, 1), (2, 1, 1)), WorkGroupBegin((0, 0, 0)),
                         WorkItemBegin(WorkItemId((0, 0, 0), (1, 0, 0), (0, 0, 0))),
                         WorkGroupEnd((0, 0, 0)), KernelEnd()],
        "segment_while_open": stream([WorkItemBegin(WI0), WorkItemBegin(wi_b), WorkItemEnd(wi_b), WorkItemEnd(WI0)]),
        "wi_begin_twice": stream([WorkItemBegin(WI0), WorkItemEnd(WI0), WorkItemBegin(WI0), WorkItemEnd(WI0)]),
        "resume_without_barrier": stream([WorkItemBegin(WI0), WorkItemEnd(WI0), WorkItemResume(WI0), WorkItemEnd(WI0)]),
        "end_without_open": stream([WorkItemBegin(WI0), WorkItemEnd(WI0), WorkItemEnd(WI0)]),
        "unfinished": stream([WorkItemBegin(WI0), Barrier(), WorkItemBegin(wi_b), WorkItemEnd(wi_b)]),
        "barrier_divergence": stream([WorkItemBegin(WI0), Barrier(), WorkItemBegin(wi_b), WorkItemEnd(wi_b),
                                      WorkItemResume(WI0), WorkItemEnd(WI0)]),
        # cap crossing before a violation wins; after it, the violation wins
        "cap_before_violation": [KernelBegin("k", 0, (1, 1, 1), (1, 1, 1)), WorkGroupBegin((0, 0, 0)), WorkItemBegin(WI0)]
                                + [e for k in range(6) for e in (Instruction("load", 1), Memory("load", 8 * k))]
                                + [WorkItemEnd(WI0), Barrier(), WorkGroupEnd((0, 0, 0)), KernelEnd()],
        "branch_cap_then_violation": [KernelBegin("k", 0, (1, 1, 1), (1, 1, 1)), WorkGroupBegin((0, 0, 0)),
                                      WorkItemBegin(WI0)] + [Instruction("br", 1), Branch(2, True)] * 5
                                     + [WorkItemEnd(WI0), Instruction("add", 1), WorkGroupEnd((0, 0, 0)), KernelEnd()],
    }
    return out


def expected_error(events, cap=None):
    try:
        acc = consume(iter(events), max_entries=cap)
        finalize(acc)
    except E.InvalidStream as exc:
        return {"error": "InvalidStream", "event_index": exc.event_index, "rule": exc.rule, "message": str(exc)}
    except E.TraceTooLarge as exc:
        return {"error": "TraceTooLarge", "entries": exc.entries, "cap": exc.cap}
    return {"error": None}


def main():
    cases = []
    kinds, pays = [], []
    offset = 0

    def add(name, events, cap=None, store_trace=True):
        nonlocal offset
        k, p, meta = encode(events)
        exp = expected(events, cap)
        rec = {"name": name, "n_events": int(k.shape[0]), "cap": cap, **meta, **exp}
        if store_trace:
            rec["offset"] = offset
            kinds.append(k); pays.append(p)
            offset += int(k.shape[0])
        cases.append(rec)

    for name, ev in unit_cases().items():
        add(name, ev)
    add("memory_cap_3", one_item([e for k in range(6) for e in (Instruction("load", 1), Memory("load", 64 * k))]), cap=3)
    add("branch_cap_2", one_item([Instruction("br", 1), Branch(4, True)] * 3), cap=2)

    fixtures = [
        ("wavefront", "wavefront.aiwck", (4, 1, 1), (4, 1, 1), {"a": "zeros:len=8"}),
        ("bfs_flags", "bfs_flags.aiwck", (16384, 1, 1), (256, 1, 1), {"flags": "bernoulli:0.5:seed=7", "out": "zeros"}),
        ("sweep4", "sweep4.aiwck", (1024, 1, 1), (64, 1, 1), {"a": "iota"}),
        ("sweep64", "sweep64.aiwck", (1024, 1, 1), (64, 1, 1), {"a": "iota:len=16384"}),
        ("bfs_const1", "bfs_flags.aiwck", (4096, 1, 1), (256, 1, 1), {"flags": "const:1", "out": "zeros"}),
        ("wavefront_big", "wavefront.aiwck", (64, 1, 1), (16, 1, 1), {"a": "zeros:len=128"}),
    ]
    for name, kern, g, l, bufs in fixtures:
        add(name, sim(kern, g, l, bufs))
    # C1 = BASELINE.json configs[0]: expected report only; the trace is regenerated
    # on device by the synthetic generator (checked against the simulator below).
    add("C1_sweep4_262144", sim("sweep4.aiwck", (262144, 1, 1), (64, 1, 1), {"a": "iota"}), store_trace=False)

    # merges (metrics.py:235-270; pkg/tests/test_metrics.py:264-303, test_acceptance.py:228-243)
    from aiwc.metrics import merge_accumulators

    def sweep_part(offset, n, invocation=0, name="k"):
        return one_item([e for i in range(n) for e in (Instruction("load", 1), Memory("load", offset + 4 * i))],
                        invocation=invocation, name=name)

    merges = {
        "self": ([sweep_part(4096, 256, 0), sweep_part(4096, 256, 1)], False),
        "disjoint": ([sweep_part(4096, 256, 0), sweep_part(4096 + 4 * 256, 256, 1)], False),
        "names": ([sweep_part(4096, 8, 0, "x"), sweep_part(8192, 8, 1, "y")], True),
        "invocations": ([sim_inv("sweep4.aiwck", n, inv) for inv, n in enumerate((1024, 512, 256, 128))], False),
        "random": ([random_events(random.Random(70 + i), 3000) for i in range(3)], True),
        "branchy": ([sim("bfs_flags.aiwck", (2048, 1, 1), (256, 1, 1), {"flags": "bernoulli:0.5:seed=%d" % s,
                                                                          "out": "zeros"}) for s in (1, 2)], False),
    }
    for mname, (parts, allow) in merges.items():
        names = []
        for i, ev in enumerate(parts):
            names.append(f"merge_{mname}_part{i}")
            add(names[-1], ev)
        rep = finalize(merge_accumulators([consume(ev) for ev in parts], allow_name_mismatch=allow))
        cases.append({"name": f"merge_{mname}", "merge": names, "allow_name_mismatch": allow,
                      "report": report_to_dict(rep, derive(rep))})

    rng = random.Random(202)  # pkg/tests/test_metrics.py:306-313
    for i in range(60):
        add(f"random202_{i}", random_events(rng, 2500))
    rng = random.Random(31337)  # pkg/tests/test_acceptance.py:134-144 (first 40)
    for i in range(40):
        add(f"random31337_{i}", random_events(rng, rng.choice([300, 1000, 4000, 10_000]), seg_cap=400))

    np.savez_compressed(os.path.join(OUT, "traces.npz"),
                        kind=np.concatenate(kinds), payload=np.concatenate(pays))


    inv = []
    for name, ev in invalid_cases().items():
        for cap in (None, 3):
            inv.append({"name": f"{name}_cap{cap}", "cap": cap, "events": repr_events(ev), **expected_error(ev, cap)})
    with open(os.path.join(OUT, "invalid.json"), "w", encoding="utf-8") as fp:
        json.dump(inv, fp, indent=1)
    with open(os.path.join(OUT, "cases.json"), "w", encoding="utf-8") as fp:
        json.dump({"generator": "tests/golden/make_golden.py", "reference": "/root/reference/pkg (aiwc 0.1.0)",
                   "cases": cases}, fp, indent=1)
    print(f"{len(cases)} cases, {offset} stored events")


if __name__ == "__main__":
    main()
