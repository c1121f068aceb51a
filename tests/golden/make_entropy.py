"""Golden values of the reference's entropy helpers (build container only).

    python tests/golden/make_entropy.py

Random histograms and branch-record sets through the reference's
shannon_entropy / local_entropy / coverage_count / branch_entropy
(pkg/src/aiwc/entropy.py:20-133), including its error cases.
"""

from __future__ import annotations

import json
import os
import random
import sys

REF = "/root/reference/pkg"
sys.path[:0] = [os.path.join(REF, "src")]

from aiwc import entropy as E  # noqa: E402
from aiwc.errors import AiwcError  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def call(fn, *a):
    try:
        r = fn(*a)
        return {"value": list(r) if isinstance(r, tuple) else r}
    except (AiwcError, ValueError) as exc:
        return {"error": type(exc).__name__, "message": str(exc)}


def main():
    rng = random.Random(99)
    hists = [{}, {5: 1}, {1: 2, 2: 2}, {0: 3, 1: 0}]
    for _ in range(40):
        n = rng.choice([1, 2, 5, 50, 400])
        span = rng.choice([16, 1024, 1 << 20, 1 << 40])
        hists.append({rng.randrange(span): rng.randint(1, rng.choice([1, 5, 1000])) for _ in range(n)})
    out = {"hist": [], "branch": []}
    for h in hists:
        row = {"items": [[k, v] for k, v in h.items()], "shannon": call(E.shannon_entropy, h),
               "coverage": call(E.coverage_count, h), "coverage_half": call(E.coverage_count, h, 0.5),
               "local": [call(E.local_entropy, h, s) for s in (1, 3, 10)], "local_bad": call(E.local_entropy, h, 11)}
        out["hist"].append(row)
    for _ in range(20):
        recs = {}
        for s in range(rng.randint(0, 4)):
            bias = rng.random()
            recs[rng.randrange(1000)] = [int(rng.random() < bias) for _ in range(rng.choice([0, 5, 17, 40, 300]))]
        for hl in (1, 4, 16):
            out["branch"].append({"records": [[k, v] for k, v in recs.items()], "history_len": hl,
                                  "result": call(E.branch_entropy, recs, hl)})
    with open(os.path.join(OUT, "entropy.json"), "w", encoding="utf-8") as fp:
        json.dump(out, fp)
    print(len(out["hist"]), "histograms,", len(out["branch"]), "branch sets")


if __name__ == "__main__":
    main()
