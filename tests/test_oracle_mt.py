"""The multi-threaded oracle (bench.py's CPU baseline) against the
single-threaded oracle and the reference's golden reports: work-group shards
merge exactly, so integers match bit for bit and entropies to 1e-9."""

import pytest

from conftest import assert_report_matches, golden_cases
from oracle import oracle


@pytest.fixture(scope="module", autouse=True)
def _built():
    oracle.build()


CASES = ["wavefront_big", "bfs_flags", "sweep4", "sweep64", "bfs_const1", "hot_address", "random202_5",
         "random31337_3", "random31337_7", "branch_streams_per_group", "offgrid_groups", "long_segments"]


@pytest.mark.parametrize("threads", [2, 3, 8])
def test_mt_oracle_matches_reference(threads):
    by = {c["name"]: (c, t) for c, t in golden_cases()}
    for name in CASES:
        if name not in by:
            continue
        c, t = by[name]
        got = oracle.run(t.kind, t.payload, kernel=t.kernel_name, invocation=t.invocation, n_opcodes=len(t.opcodes),
                         threads=threads)
        want = {k: v for k, v in c["report"].items()
                if k not in ("granularity", "barriers_per_instruction", "instructions_per_operand", "load_imbalance")}
        assert_report_matches(got, want)


def test_mt_oracle_matches_single_thread_on_synthetic():
    from paper_1805_04207_b200 import synth

    for cfg, w in [(2, 1 << 13), (3, 1 << 12), (4, 1 << 11), (5, 1 << 12)]:
        t = synth.python_trace(cfg, w)
        one = oracle.run_trace(t)
        many = oracle.run(t.kind, t.payload, kernel=t.kernel_name, invocation=0, n_opcodes=len(t.opcodes), threads=6)
        assert_report_matches(many, one)
