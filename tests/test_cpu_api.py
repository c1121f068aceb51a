"""CPU-only tests: the C ABI library loads and exports every declared symbol,
the native walker encodes / validates exactly like the reference, and the
report artifact is byte-identical to the reference's emit_report output.
No CUDA device is touched here."""

import json
import os
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, golden_cases
from paper_1805_04207_b200 import (
    Barrier, Branch, Instruction, KernelBegin, KernelEnd, Memory, WorkGroupBegin, WorkGroupEnd, WorkItemBegin,
    WorkItemEnd, WorkItemId, WorkItemResume, emit_report, report_from_dict, report_to_dict, summarize_distribution,
)
from paper_1805_04207_b200 import _native, default_entry_cap, derive
from paper_1805_04207_b200.errors import EmptySample
from paper_1805_04207_b200.report import AiwcReport, CSV_COLUMNS
from paper_1805_04207_b200.walker import encode_events


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_1805_04207_b200 import build

    build.build_all()


def test_library_exports_every_declared_symbol():
    with open(os.path.join(ROOT, "include", "aiwc_b200.h"), encoding="utf-8") as fp:
        header = fp.read()
    declared = set(re.findall(r"\b(aiwc_[a-z_0-9]+)\s*\(", header))
    assert declared >= set(_native.EXPORTS)
    lib = _native.load_library()
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert lib.aiwc_abi_version() == 2


def test_result_struct_matches_header_layout():
    import ctypes

    # aiwc_result: 2x dist (6 u64) + scalars; pointer / phase tail must line up with the header
    assert ctypes.sizeof(_native.Result) % 8 == 0
    assert _native.Result.phase_ms.offset == _native.Result.d2h_bytes.offset + 8


_CLS = {c.__name__: c for c in (KernelBegin, KernelEnd, WorkGroupBegin, WorkGroupEnd, WorkItemBegin, WorkItemResume,
                                WorkItemEnd, Instruction, Branch, Memory, Barrier)}


def _tup(x):
    return tuple(_tup(v) for v in x) if isinstance(x, list) else x


def events_from_json(rows):
    out = []
    for name, *fields in rows:
        if name in ("WorkItemBegin", "WorkItemResume", "WorkItemEnd"):
            out.append(_CLS[name](WorkItemId(*_tup(fields[0]))))
        else:
            out.append(_CLS[name](*[_tup(f) for f in fields]))
    return out


def _invalid_cases():
    with open(os.path.join(GOLDEN, "invalid.json"), encoding="utf-8") as fp:
        return json.load(fp)


@pytest.mark.parametrize("case", [c for c in _invalid_cases() if c["cap"] is None], ids=lambda c: c["name"])
def test_walker_first_violation_matches_reference(case):
    """StreamChecker parity: same first event index, rule and message text."""
    tr, violation = encode_events(iter(events_from_json(case["events"])))
    assert violation is not None
    index, rule, detail = violation
    assert (index, rule) == (case["event_index"], case["rule"])
    msg = f"event {index}: {rule}" + (f" ({detail})" if detail else "")
    assert msg == case["message"]
    if tr is not None:  # the encoded prefix = the events consume() folded before raising
        assert tr.n_events <= index + 1


@pytest.mark.parametrize("case,trace", [(c, t) for c, t in golden_cases() if t is not None and "error" not in c][:60],
                         ids=lambda x: x["name"] if isinstance(x, dict) else "")
def test_walker_round_trip(case, trace):
    """decode (ColumnarTrace.iter_events) -> native walker -> identical columns."""
    tr, violation = encode_events(trace.iter_events())
    assert violation is None
    assert np.array_equal(tr.kind, trace.kind)
    assert np.array_equal(tr.payload, trace.payload)
    assert tr.opcodes == trace.opcodes
    assert [tuple(g) for g in tr.extra_groups] == [tuple(g) for g in trace.extra_groups]


def test_walker_accepts_generators_and_rejects_non_events():
    def gen():
        yield KernelBegin("k", 0, (1, 1, 1), (1, 1, 1))
        yield KernelEnd()
    tr, v = encode_events(gen())
    assert v is None and tr.n_events == 2
    with pytest.raises(TypeError):
        encode_events([KernelBegin("k", 0, (1, 1, 1), (1, 1, 1)), object()])


def test_walker_memory_op_fold_and_stats():
    wi = WorkItemId((0, 0, 0), (0, 0, 0), (0, 0, 0))
    ev = [KernelBegin("k", 0, (1, 1, 1), (1, 1, 1)), WorkGroupBegin((0, 0, 0)), WorkItemBegin(wi),
          Instruction("x", 1), Memory("atomic_load", 64), Instruction("x", 1), Memory("atomic_store", 96),
          Instruction("x", 1), Memory("weird_op", 128), WorkItemEnd(wi), WorkGroupEnd((0, 0, 0)), KernelEnd()]
    tr, v = encode_events(ev)
    assert v is None
    assert list(tr.kind[[4, 6, 8]]) == [0x82, 0x84, 0x04]  # anything not a read op is a write (metrics.py:138)
    assert tr.addr_stats == (64, 128, 64 & 96 & 128, 64 | 96 | 128)


@pytest.mark.parametrize("case", [c for c, _ in golden_cases() if "json" in c][:40], ids=lambda c: c["name"])
def test_emit_report_bytes_match_reference(case):
    rep = report_from_dict(case["report"])
    assert emit_report(rep).decode("utf-8") == case["json"]
    assert emit_report(rep, format="csv").decode("utf-8") == case["csv"]


def test_report_key_order_is_the_reference_schema():
    case = next(c for c, _ in golden_cases() if "report" in c)
    rep = report_from_dict(case["report"])
    assert list(report_to_dict(rep)) == list(case["report"])
    assert len(CSV_COLUMNS) == 49


def test_summarize_distribution_semantics():
    s = summarize_distribution([2, 4, 4, 4, 5, 5, 7, 9])
    assert (s.minimum, s.maximum, s.median, s.mean, s.sd) == (2, 9, 4.5, 5.0, 2.0)
    assert summarize_distribution([5]).median == 5.0
    with pytest.raises(EmptySample):
        summarize_distribution([])


def test_default_entry_cap_env(monkeypatch):
    monkeypatch.delenv("AIWC_MEM_CAP_BYTES", raising=False)
    assert default_entry_cap() == (1 << 30) // 64
    monkeypatch.setenv("AIWC_MEM_CAP_BYTES", "256")
    assert default_entry_cap() == 4
    monkeypatch.setenv("AIWC_MEM_CAP_BYTES", "1")
    assert default_entry_cap() == 1


def test_derive_degenerate():
    case = next(c for c, _ in golden_cases() if c["name"] == "wavefront")
    rep = report_from_dict(case["report"])
    d = derive(rep)
    assert d.barriers_per_instruction == 0.04
    assert isinstance(rep, AiwcReport)


def test_chunk_cuts_split_at_work_group_starts():
    from paper_1805_04207_b200.dist import chunk_cuts
    from paper_1805_04207_b200.errors import UnsupportedTrace
    from paper_1805_04207_b200.trace import K_WG_BEGIN

    kind = np.zeros(100, np.uint8)
    starts = [1, 12, 30, 31, 55, 80, 97]
    kind[starts] = K_WG_BEGIN
    cuts = chunk_cuts(kind, 30)
    assert cuts[0] == 0 and cuts[-1] == 100
    assert all(b - a <= 30 for a, b in zip(cuts, cuts[1:]))
    assert all(c in starts for c in cuts[1:-1])
    assert chunk_cuts(kind, 100) == [0, 100]
    with pytest.raises(UnsupportedTrace):
        chunk_cuts(kind, 20)  # 55..80 is one 25-event group
