"""NDRange producer on the device against the reference simulator's own
outputs (tests/golden/sim.json from tests/golden/make_sim.py).

Every golden launch -- the reference's kernels and test programs, semantic
edge cases (Python floor division / modulo, INT64_MIN, shifts, vector lanes)
and 120 seeded random programs with loops, diamonds, barriers, private and
shared memory, faults, divergence and step limits -- runs through both device
modes (speculative with automatic fallback, forced group, forced sequential).  The event stream must be
byte-identical to the reference's canonical lines (count + sha256, lines
where recorded), the fault must be the same class with the same message and
line, and it must come after exactly the same events.  Valid traces also go
through consume/finalize on the device and must match the oracle."""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import assert_report_matches

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "sim.json")))


def _run(case, schedule):
    from paper_1805_04207_b200 import encode_event, ir, sim

    prog = ir.parse_kernel(case["source"])
    cfg = sim.NDRangeConfig(tuple(case["global"]), tuple(case["local"]), case["buffers"], case["bases"])
    lines, err = [], None
    try:
        for ev in sim.simulate_events(prog, cfg, step_limit=case["step_limit"], invocation=case["invocation"],
                                      schedule=schedule):
            lines.append(encode_event(ev))
    except Exception as exc:  # noqa: BLE001
        err = {"type": type(exc).__name__, "message": str(exc), "line": getattr(exc, "line", None)}
    return lines, err


@pytest.mark.parametrize("schedule", ["auto", "group", "sequential"])
@pytest.mark.parametrize("case", GOLD["cases"], ids=lambda c: c["name"])
def test_events_match_reference(case, schedule):
    lines, err = _run(case, schedule)
    if "lines" in case and lines != case["lines"]:
        for i, (a, b) in enumerate(zip(lines, case["lines"])):
            assert a == b, f"event {i}"
        assert len(lines) == len(case["lines"])
    assert len(lines) == case["n_events"]
    assert hashlib.sha256("\n".join(lines).encode()).hexdigest() == case["sha256"]
    assert err == case["error"]


@pytest.mark.parametrize("case", [c for c in GOLD["cases"] if c["error"] is None], ids=lambda c: c["name"])
def test_simulated_trace_report_matches_oracle(case):
    from oracle import oracle

    from paper_1805_04207_b200 import consume, finalize, ir, report_to_dict, sim

    oracle.build()
    prog = ir.parse_kernel(case["source"])
    cfg = sim.NDRangeConfig(tuple(case["global"]), tuple(case["local"]), case["buffers"], case["bases"])
    tr = sim.simulate_trace(prog, cfg, step_limit=case["step_limit"], invocation=case["invocation"])
    assert tr.kind.is_cuda and tr.validated and tr.class_counts is not None
    assert tr.n_events == case["n_events"]
    want = oracle.run_trace(tr.to_numpy())
    assert_report_matches(report_to_dict(finalize(consume(tr))), want)


def test_faults_raise_through_simulate_trace():
    from paper_1805_04207_b200 import errors, ir, sim

    prog = ir.parse_kernel("kernel k(a)\nentry:\n  load r0, buf[a][gid0]\n  ret\n")
    with pytest.raises(errors.OutOfBoundsAccess, match="'a' at index 3"):
        sim.simulate_trace(prog, sim.NDRangeConfig((8, 1, 1), (4, 1, 1), {"a": [0] * 3}))
    loop = ir.parse_kernel("kernel k()\nentry:\n  jmp entry\n")
    with pytest.raises(errors.StepLimitExceeded):
        sim.simulate_trace(loop, sim.NDRangeConfig((4, 1, 1), (2, 1, 1), {}), step_limit=10_000)


def test_large_launch_matches_sequential_mode():
    """A launch big enough to fill the GPU: speculative and sequential device
    modes agree byte for byte (the sequential mode is the reference's schedule
    literally), and the report equals the oracle's."""
    from oracle import oracle

    from paper_1805_04207_b200 import consume, finalize, ir, report_to_dict, sim

    oracle.build()
    src = ("kernel big(a, b)\nentry:\n  load r0, buf[b][gid0]\n  and r1, r0, 1\n  mov r2, 0\n  br r1, odd, even\n"
           "odd:\n  add r2, r2, r0\n  mul r3, gid0, 2\n  store.x2 buf[a][r3], r2\n  jmp fin\n"
           "even:\n  load.x4 r4, buf[b][lid0]\n  add.x4 r4, r4, 7\n  jmp fin\nfin:\n  barrier\n  ret\n")
    n = 1 << 16
    rng = np.random.default_rng(5)
    cfg = sim.NDRangeConfig((n, 1, 1), (256, 1, 1), {"a": [0] * (2 * n), "b": rng.integers(0, 1 << 20, n).tolist()})
    prog = ir.parse_kernel(src)
    a = sim.simulate_trace(prog, cfg)
    for schedule in ("group", "sequential"):
        b = sim.simulate_trace(prog, cfg, schedule=schedule)
        assert torch.equal(a.kind, b.kind) and torch.equal(a.payload, b.payload)
    assert_report_matches(report_to_dict(finalize(consume(a))), oracle.run_trace(a.to_numpy()))


def test_schedule_selection():
    """Private stores stay speculative; a neighbour read after a barrier (a
    dependence inside the group) takes the group schedule; a chain across
    groups takes the sequential one."""
    from paper_1805_04207_b200 import ir, sim

    def schedule_of(src, gsz, lsz, bufs):
        cfg = sim.NDRangeConfig(gsz, lsz, bufs)
        launch = sim._Launch(ir.parse_kernel(src), cfg, sim._prepare(ir.parse_kernel(src), cfg), 10 ** 8, 0)
        try:
            return launch.schedule
        finally:
            launch.close()

    private = "kernel p(a)\nentry:\n  store buf[a][gid0], 1\n  load r0, buf[a][gid0]\n  ret\n"
    assert schedule_of(private, (64, 1, 1), (8, 1, 1), {"a": [0] * 64}) == "speculative"
    nb = ("kernel nb(a)\nentry:\n  store buf[a][gid0], gid0\n  barrier\n  add r0, lid0, 1\n  rem r0, r0, lsz0\n"
          "  sub r1, gid0, lid0\n  add r0, r0, r1\n  load r1, buf[a][r0]\n  ret\n")
    assert schedule_of(nb, (64, 1, 1), (8, 1, 1), {"a": [0] * 64}) == "group"
    chain = "kernel c(a)\nentry:\n  load r0, buf[a][gid0]\n  add r1, gid0, 1\n  store buf[a][r1], r0\n  ret\n"
    assert schedule_of(chain, (64, 1, 1), (8, 1, 1), {"a": [0] * 65}) == "sequential"
