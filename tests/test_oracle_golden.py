"""Pin the C oracle against reports produced by the reference itself.

tests/golden/cases.json holds the reference's own ``finalize`` output for
every fixture (tests/golden/make_golden.py).  The oracle is only trusted as
the GPU path's checker because it reproduces all of them.
"""

import pytest

from conftest import assert_report_matches, golden_cases
from oracle import oracle


@pytest.fixture(scope="module", autouse=True)
def _built():
    oracle.build()


def _cases():
    return [(c, t) for c, t in golden_cases() if t is not None]


@pytest.mark.parametrize("case,trace", _cases(), ids=[c["name"] for c, _ in _cases()])
def test_oracle_matches_reference(case, trace):
    if "error" in case:
        with pytest.raises(oracle.OracleTooLarge) as ei:
            oracle.run_trace(trace, entry_cap=case["cap"])
        assert (ei.value.entries, ei.value.cap) == (case["entries"], case["cap"])
        return
    got = oracle.run_trace(trace, entry_cap=case["cap"] or 0)
    want = dict(case["report"])
    for k in ("granularity", "barriers_per_instruction", "instructions_per_operand", "load_imbalance"):
        want.pop(k)
    assert_report_matches(got, want)


def test_c1_expected_report_present():
    names = [c["name"] for c, _ in golden_cases()]
    assert "C1_sweep4_262144" in names
