"""Traces larger than one engine ingest (2^32 - 1 events) are cut at
work-group starts and combined exactly (dist.chunked_result).  The limit is
lowered here (AIWC_MAX_INGEST_EVENTS) so golden traces and the synthetic
configs take the chunked path; reports must equal the reference's / the
single-ingest engine's."""

import numpy as np
import pytest

from conftest import assert_report_matches, golden_cases

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

NAMES = ["wavefront_big", "sweep4", "hot_address", "random31337_3", "offgrid_groups", "branch_streams_per_group",
         "bfs_flags", "segment_split"]


@pytest.mark.parametrize("limit", [700, 5000])
def test_golden_traces_chunked_match_reference(limit, monkeypatch):
    from paper_1805_04207_b200 import consume, finalize, report_to_dict

    by_name = {c["name"]: (c, t) for c, t in golden_cases()}
    ran = 0
    for name in NAMES:
        if name not in by_name:
            continue
        c, tr = by_name[name]
        monkeypatch.setenv("AIWC_MAX_INGEST_EVENTS", str(limit))
        try:
            got = report_to_dict(finalize(consume(tr, max_entries=1 << 40)))
        except Exception as exc:  # a work-group longer than the limit cannot be cut
            assert "work-group spans" in str(exc)
            continue
        assert_report_matches(got, c["report"])
        ran += 1
    assert ran >= 3


@pytest.mark.parametrize("cfg,w", [(2, 8192), (3, 4096), (4, 4096), (5, 2048)])
def test_synthetic_chunked_match_single_ingest(cfg, w, monkeypatch):
    from paper_1805_04207_b200 import consume, finalize, report_to_dict, synth

    tr = synth.device_trace(cfg, w)
    want = report_to_dict(finalize(consume(tr, max_entries=1 << 40)))
    monkeypatch.setenv("AIWC_MAX_INGEST_EVENTS", str(tr.n_events // 3))
    got = report_to_dict(finalize(consume(tr, max_entries=1 << 40)))
    assert_report_matches(got, want)


def test_repeated_group_id_across_chunks_is_refused(monkeypatch):
    """A work-group id that repeats on both sides of a cut would split its (site,
    group) branch stream (metrics.py:145-152): refused, not silently wrong."""
    from paper_1805_04207_b200 import UnsupportedTrace, consume, finalize, report_to_dict
    from paper_1805_04207_b200.trace import K_WG_BEGIN

    c, tr = next((c, t) for c, t in golden_cases() if c["name"] == "repeated_group_id")
    starts = np.nonzero(tr.kind == K_WG_BEGIN)[0].tolist() + [tr.n_events]
    longest = max(b - a for a, b in zip(starts[:-1], starts[1:]))
    monkeypatch.setenv("AIWC_MAX_INGEST_EVENTS", str(longest + 2))
    with pytest.raises(UnsupportedTrace, match="repeats"):
        finalize(consume(tr, max_entries=1 << 40))
    monkeypatch.delenv("AIWC_MAX_INGEST_EVENTS")
    assert_report_matches(report_to_dict(finalize(consume(tr, max_entries=1 << 40))), c["report"])
