"""The drop-in API end to end on the GPU: TraceEvent object streams (native
walker -> CUDA engine), the reference's error ordering between InvalidStream
and TraceTooLarge, merge_accumulators, and tampered-accumulator checks --
each against the reference's own recorded behaviour (tests/golden)."""

import json
import os

import pytest

from conftest import GOLDEN, assert_report_matches, golden_cases
from test_cpu_api import events_from_json

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1805_04207_b200 import (  # noqa: E402
    AiwcError, IncompatibleReports, InvalidStream, TraceTooLarge, consume, finalize, merge_accumulators,
    report_to_dict,
)


def _stored():
    return [(c, t) for c, t in golden_cases() if t is not None and "error" not in c]


@pytest.mark.parametrize("case,trace", _stored()[:80], ids=lambda x: x["name"] if isinstance(x, dict) else "")
def test_object_stream_matches_reference(case, trace):
    """consume(Iterable[TraceEvent]) -- a generator, never materialised."""
    got = report_to_dict(finalize(consume(trace.iter_events())))
    assert_report_matches(got, case["report"])


def _invalid():
    with open(os.path.join(GOLDEN, "invalid.json"), encoding="utf-8") as fp:
        return json.load(fp)


@pytest.mark.parametrize("case", _invalid(), ids=lambda c: c["name"])
def test_error_parity(case):
    events = events_from_json(case["events"])
    if case["error"] == "TraceTooLarge":
        with pytest.raises(TraceTooLarge) as ei:
            consume(iter(events), max_entries=case["cap"])
        assert (ei.value.entries, ei.value.cap) == (case["entries"], case["cap"])
    else:
        with pytest.raises(InvalidStream) as ei:
            consume(iter(events), max_entries=case["cap"])
        assert (ei.value.event_index, ei.value.rule, str(ei.value)) == (
            case["event_index"], case["rule"], case["message"])


_by_name = {c["name"]: (c, t) for c, t in golden_cases()}


@pytest.mark.parametrize("case", [c for c, _ in golden_cases() if "merge" in c], ids=lambda c: c["name"])
def test_merge_matches_reference(case):
    parts = [consume(_by_name[n][1]) for n in case["merge"]]
    merged = merge_accumulators(parts, allow_name_mismatch=case["allow_name_mismatch"])
    assert_report_matches(report_to_dict(finalize(merged)), case["report"])


def test_merge_name_mismatch_rejected():
    c = next(c for c in golden_cases() if c[0]["name"] == "merge_names")[0]
    parts = [consume(_by_name[n][1]) for n in c["merge"]]
    with pytest.raises(IncompatibleReports):
        merge_accumulators(parts)


def test_tampered_accumulator_rejected():
    """finalize re-checks conservation (ref test_metrics.py:237-241)."""
    _, tr = _by_name["single_item_no_barriers"]
    acc = consume(tr)
    acc.itb_samples = [4]
    with pytest.raises(AiwcError, match="ITB"):
        finalize(acc)


def test_accumulator_fields():
    _, tr = _by_name["simd_stats"]
    acc = consume(tr)
    assert acc.total_instructions == 3 and acc.work_items == 1 and acc.barriers_hit == 0
    assert dict(acc.opcode_histogram) == {"add": 1, "fmul": 1, "mad": 1}
    assert list(acc.simd_width_counts.items()) == [(1, 1), (4, 2)]  # first-appearance order
