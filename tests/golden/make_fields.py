"""Golden per-event accumulator fields from the REFERENCE (build container only).

    python tests/golden/make_fields.py

Runs the reference's ``consume`` (and ``merge_accumulators``) on a subset of
the traces make_golden.py stores and writes their itb_samples, ipt_samples,
read/write address Counters (first-appearance order) and branch_records to
tests/golden/fields.json, keyed by the case names of cases.json.
"""

from __future__ import annotations

import json
import os
import random

import make_golden as G

OUT = os.path.dirname(os.path.abspath(__file__))


def fields_of(acc):
    return {
        "itb_samples": list(acc.itb_samples),
        "ipt_samples": list(acc.ipt_samples),
        "read_addresses": [[a, c] for a, c in acc.read_addresses.items()],
        "write_addresses": [[a, c] for a, c in acc.write_addresses.items()],
        "branch_records": [[site, [[list(g) if g is not None else None, bits] for g, bits in streams]]
                           for site, streams in acc.branch_records.items()],
    }


def main():
    from aiwc.metrics import consume, merge_accumulators

    out = {}
    for name, ev in G.unit_cases().items():
        out[name] = fields_of(consume(ev))
    for name, kern, g, l, bufs in [
        ("wavefront", "wavefront.aiwck", (4, 1, 1), (4, 1, 1), {"a": "zeros:len=8"}),
        ("sweep4", "sweep4.aiwck", (1024, 1, 1), (64, 1, 1), {"a": "iota"}),
        ("wavefront_big", "wavefront.aiwck", (64, 1, 1), (16, 1, 1), {"a": "zeros:len=128"}),
        ("bfs_const1", "bfs_flags.aiwck", (4096, 1, 1), (256, 1, 1), {"flags": "const:1", "out": "zeros"}),
    ]:
        out[name] = fields_of(consume(G.sim(kern, g, l, bufs)))
    rng = random.Random(202)  # the same sequence make_golden.py draws
    for i in range(60):
        ev = G.random_events(rng, 2500)
        if i < 20:
            out[f"random202_{i}"] = fields_of(consume(ev))
    parts = [G.sim("bfs_flags.aiwck", (2048, 1, 1), (256, 1, 1), {"flags": "bernoulli:0.5:seed=%d" % s, "out": "zeros"})
             for s in (1, 2)]
    accs = [consume(ev) for ev in parts]
    for i, a in enumerate(accs):
        out[f"merge_branchy_part{i}"] = fields_of(a)
    out["merge_branchy"] = fields_of(merge_accumulators(accs))
    with open(os.path.join(OUT, "fields.json"), "w", encoding="utf-8") as fp:
        json.dump({"generator": "tests/golden/make_fields.py", "fields": out}, fp)
    print(f"{len(out)} field sets")


if __name__ == "__main__":
    main()
