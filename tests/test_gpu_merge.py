"""merge_accumulators as a STATE merge (ref metrics.py:235-270): the parts'
exported state (per-key runs over each trace's key map, histograms, pattern
tables) is summed -- no re-ingest of the parts' columns.  Results must equal the
reference's merge reports and the re-ingest of the concatenated columns, nested
merges included; the state merge must cost far less than one ingest."""

import time

import pytest

from conftest import assert_report_matches, golden_cases

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1805_04207_b200 import consume, finalize, merge_accumulators, report_to_dict  # noqa: E402

_by_name = {c["name"]: (c, t) for c, t in golden_cases()}


@pytest.mark.parametrize("case", [c for c, _ in golden_cases() if "merge" in c], ids=lambda c: c["name"])
def test_state_merge_matches_reference(case):
    parts = [consume(_by_name[n][1]) for n in case["merge"]]
    merged = merge_accumulators(parts, allow_name_mismatch=case["allow_name_mismatch"])
    if case["name"] != "merge_random":  # random parts span too wide a union: that merge re-ingests
        assert merged.trace is None, "the state merge re-ingested"
    assert_report_matches(report_to_dict(finalize(merged)), case["report"])
    # nested: merge(merge(p0, p1), p2, ...) == merge(p0, p1, p2, ...)
    if len(parts) >= 3:
        inner = merge_accumulators(parts[:2], allow_name_mismatch=case["allow_name_mismatch"])
        outer = merge_accumulators([inner] + parts[2:], allow_name_mismatch=case["allow_name_mismatch"])
        assert_report_matches(report_to_dict(finalize(outer)), case["report"])


def test_state_merge_of_synthetic_halves_matches_reingest_and_is_cheaper():
    """Two C2-shaped accumulators (2^22 work-items each): the state merge equals the
    re-ingest of the concatenated columns and costs less than that re-ingest."""
    from paper_1805_04207_b200 import synth
    from paper_1805_04207_b200.merge import concat_traces
    from paper_1805_04207_b200.metrics import KernelAccumulator, run_engine

    w = 1 << 22
    a = synth.device_trace(2, w)
    b = synth.device_trace(5, w // 4)
    pa, pb = consume(a, max_entries=1 << 40), consume(b, max_entries=1 << 40)
    assert pa.result.state is not None and pb.result.state is not None
    for _ in range(2):
        merged = merge_accumulators([pa, pb], allow_name_mismatch=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    merged = merge_accumulators([pa, pb], allow_name_mismatch=True)
    t_merge = time.perf_counter() - t0
    assert merged.trace is None
    run_engine(concat_traces([a, b]))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tr = concat_traces([a, b])  # the re-ingest merge: concatenated columns, one engine pass
    res = run_engine(tr)
    torch.cuda.synchronize()
    t_reingest = time.perf_counter() - t0
    want = KernelAccumulator(pa.kernel_name, [0, 0], merged.launches, res, list(tr.opcodes))
    want.lmae_per_invocation = merged.lmae_per_invocation
    assert_report_matches(report_to_dict(finalize(merged)), report_to_dict(finalize(want)))
    assert t_merge < t_reingest, (t_merge, t_reingest)
