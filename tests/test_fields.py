"""Per-event accumulator fields (itb_samples, ipt_samples, read/write address
Counters, branch_records) against the reference's own consume() output
(tests/golden/fields.json, made by make_fields.py).  The CPU tests check the
materialiser on the golden columns; the GPU tests read the fields through
KernelAccumulator after consume / merge_accumulators, as the reference's
test_metrics.py does."""

import json
import os

import pytest

from conftest import GOLDEN, golden_cases

with open(os.path.join(GOLDEN, "fields.json"), encoding="utf-8") as _fp:
    REF = json.load(_fp)["fields"]


def as_plain(f):
    return {
        "itb_samples": list(f["itb_samples"]),
        "ipt_samples": list(f["ipt_samples"]),
        "read_addresses": [[a, c] for a, c in f["read_addresses"].items()],
        "write_addresses": [[a, c] for a, c in f["write_addresses"].items()],
        "branch_records": [[site, [[list(g) if g is not None else None, bits] for g, bits in streams]]
                           for site, streams in f["branch_records"].items()],
    }


def _traces():
    return {c["name"]: t for c, t in golden_cases() if t is not None}


@pytest.mark.parametrize("name", sorted(n for n in REF if not n.startswith("merge_branchy") or "part" in n))
def test_materialized_fields_match_reference(name):
    from paper_1805_04207_b200.fields import materialize

    got = as_plain(materialize(_traces()[name]))
    assert got == REF[name]


def test_merged_fields_match_reference_merge():
    from paper_1805_04207_b200.fields import materialize, merge_fields

    tr = _traces()
    got = merge_fields([materialize(tr[f"merge_branchy_part{i}"]) for i in range(2)])
    assert as_plain(got) == REF["merge_branchy"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["segment_split", "two_items_ipt", "empty_final_segment", "atomics_folded",
                                  "wavefront_big", "random202_3"])
def test_accumulator_fields_after_consume(name):
    from paper_1805_04207_b200 import consume

    acc = consume(_traces()[name])
    assert as_plain({f: getattr(acc, f) for f in REF[name]}) == REF[name]


@pytest.mark.gpu
def test_accumulator_fields_after_merge():
    from paper_1805_04207_b200 import consume, merge_accumulators

    tr = _traces()
    acc = merge_accumulators([consume(tr[f"merge_branchy_part{i}"]) for i in range(2)])
    assert as_plain({f: getattr(acc, f) for f in REF["merge_branchy"]}) == REF["merge_branchy"]
