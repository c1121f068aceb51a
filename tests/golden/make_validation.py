"""Golden validate_stream reports from the REFERENCE (build container only).

    python tests/golden/make_validation.py

The reference's validate_stream (pkg/src/aiwc/trace.py:427-437) collects every
violation; this records its reports for the invalid streams of invalid.json
and for randomly mutated valid streams (events dropped, duplicated, swapped).
"""

from __future__ import annotations

import json
import os
import random
import sys

import make_golden as G

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    from aiwc.trace import validate_stream

    cases = []
    for name, ev in G.invalid_cases().items():
        cases.append({"name": name, "events": G.repr_events(ev),
                      "violations": [list(v) for v in validate_stream(ev).violations]})
    rng = random.Random(4242)
    bases = [G.sim("wavefront.aiwck", (8, 1, 1), (4, 1, 1), {"a": "zeros:len=16"}),
             G.sim("bfs_flags.aiwck", (64, 1, 1), (16, 1, 1), {"flags": "bernoulli:0.5:seed=3", "out": "zeros"})]
    bases += [G.random_events(random.Random(900 + i), 400) for i in range(4)]
    for b, base in enumerate(bases):
        for m in range(12):
            ev = list(base)
            for _ in range(rng.randint(1, 3)):
                op = rng.choice(("drop", "dup", "swap"))
                k = rng.randrange(len(ev))
                if op == "drop":
                    del ev[k]
                elif op == "dup":
                    ev.insert(k, ev[k])
                elif k + 1 < len(ev):
                    ev[k], ev[k + 1] = ev[k + 1], ev[k]
            cases.append({"name": f"mut{b}_{m}", "events": G.repr_events(ev),
                          "violations": [list(v) for v in validate_stream(ev).violations]})
    with open(os.path.join(OUT, "validation.json"), "w", encoding="utf-8") as fp:
        json.dump(cases, fp)
    print(f"{len(cases)} streams, {sum(len(c['violations']) for c in cases)} violations")


if __name__ == "__main__":
    main()
