""".aiwctrace files: the reference's line rules (tests/golden/tracefile_lines.json,
made by the reference's decode_event) and the columnar fast path (native
canonical parser + Python fallback) against the object path, on CPU; reports
from consume_file against the reference's goldens on the GPU."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, assert_report_matches, golden_cases

with open(os.path.join(GOLDEN, "tracefile_lines.json"), encoding="utf-8") as _fp:
    LINES = json.load(_fp)

DERIVED = ("granularity", "barriers_per_instruction", "instructions_per_operand", "load_imbalance")


@pytest.mark.parametrize("i", range(len(LINES)))
def test_decode_event_matches_reference(i):
    from paper_1805_04207_b200 import MalformedEvent
    from paper_1805_04207_b200.tracefile import decode_event, encode_event

    case = LINES[i]
    if "error" in case:
        with pytest.raises(MalformedEvent) as ei:
            decode_event(case["line"], i + 1)
        assert str(ei.value) == case["error"]
    else:
        assert encode_event(decode_event(case["line"], i + 1)) == case["event"]


def _events(tr):
    return list(tr.iter_events())


def _write(path, lines):
    with open(path, "w", encoding="utf-8", newline="\n") as fp:
        for ln in lines:
            fp.write(ln + "\n")


def _same_columns(a, b):
    assert a.kernel_name == b.kernel_name and a.invocation == b.invocation
    assert tuple(a.global_size) == tuple(b.global_size) and tuple(a.local_size) == tuple(b.local_size)
    assert list(a.opcodes) == list(b.opcodes)
    assert [tuple(g) for g in a.extra_groups] == [tuple(g) for g in b.extra_groups]
    np.testing.assert_array_equal(np.asarray(a.kind), np.asarray(b.kind))
    np.testing.assert_array_equal(np.asarray(a.payload).view(np.uint64), np.asarray(b.payload).view(np.uint64))


CASES = ["wavefront_big", "bfs_flags", "sweep4", "hot_address", "offgrid_groups", "branch_streams_per_group",
         "random202_1", "random31337_4", "long_segments", "merge_branchy_part0"]


@pytest.mark.parametrize("name", CASES)
def test_file_columns_equal_object_path(name, tmp_path):
    from paper_1805_04207_b200.tracefile import encode_event, load_trace
    from paper_1805_04207_b200.walker import encode_events

    tr = {c["name"]: t for c, t in golden_cases() if t is not None}[name]
    events = _events(tr)
    path = tmp_path / "t.aiwctrace"
    _write(path, ["# produced by test_tracefile"] + [encode_event(e) for e in events])
    got, violation, err, last = load_trace(str(path))
    assert violation is None and err is None
    want, v2 = encode_events(events)
    assert v2 is None
    _same_columns(got, want)
    assert last == len(events) + 1


def test_non_canonical_lines_fall_back_to_the_reference_rules(tmp_path):
    """Re-ordered keys, spaces, escapes, non-ASCII and CRLF lines decode like json.loads."""
    from paper_1805_04207_b200.tracefile import encode_event, load_trace
    from paper_1805_04207_b200.walker import encode_events

    tr = {c["name"]: t for c, t in golden_cases() if t is not None}["random202_2"]
    events = _events(tr)
    lines = []
    for k, e in enumerate(events):
        ln = encode_event(e)
        obj = json.loads(ln)
        if k % 5 == 1:
            ln = json.dumps(dict(reversed(list(obj.items()))))  # other key order, spaces
        elif k % 5 == 2:
            ln = json.dumps(obj, ensure_ascii=True, indent=None, separators=(", ", ": "))
        elif k % 5 == 3 and obj["ev"] == "instr":
            obj["opcode"] = obj["opcode"] + "é\"q"
            ln = json.dumps(obj, separators=(",", ":"), ensure_ascii=False)
        lines.append(ln)
    path = tmp_path / "t.aiwctrace"
    _write(path, lines)
    got, violation, err, _ = load_trace(str(path))
    ev2 = []
    for k, e in enumerate(events):
        if k % 5 == 3 and type(e).__name__ == "Instruction":
            e = type(e)(e.opcode + "é\"q", e.width)
        ev2.append(e)
    want, _ = encode_events(ev2)
    assert violation is None and err is None
    _same_columns(got, want)
    # CRLF / lone-CR files are read in text mode, like the reference
    with open(path, "w", encoding="utf-8", newline="\r\n") as fp:
        fp.write("\n".join(lines) + "\n")
    got2, violation, err, _ = load_trace(str(path))
    assert violation is None and err is None
    _same_columns(got2, want)


def test_malformed_line_and_blank_line_errors(tmp_path):
    from paper_1805_04207_b200 import MalformedEvent
    from paper_1805_04207_b200.tracefile import load_trace

    head = ['{"ev":"kernel_begin","kernel":"k","invocation":0,"global_size":[2,1,1],"local_size":[2,1,1]}',
            '{"ev":"wg_begin","group":[0,0,0]}',
            '{"ev":"wi_begin","global":[0,0,0],"local":[0,0,0],"group":[0,0,0]}']
    for bad, msg in [("", "line 5: blank line"), ("   ", "line 5: blank line"),
                     ('{"ev":"instr","opcode":"add","width":0}', "line 5: field 'width' must be >= 1"),
                     ('{"ev":"mem","op":"load","addr":4096.0}', "line 5: field 'addr' must be a non-negative integer")]:
        path = tmp_path / "b.aiwctrace"
        _write(path, head + ['# comment', bad, '{"ev":"kernel_end"}'])
        tr, violation, err, last = load_trace(str(path))
        assert isinstance(err, MalformedEvent) and str(err) == msg
        assert tr.n_events == 3 and last == 5


@pytest.mark.parametrize("case", [c for c in json.load(open(os.path.join(GOLDEN, "invalid.json"), encoding="utf-8"))
                                  if c.get("cap") is None][:25], ids=lambda c: c["name"])
def test_stream_violations_from_files(case, tmp_path):
    """The reference's InvalidStream (index, rule) for invalid streams written to files."""
    from test_cpu_api import events_from_json  # the invalid fixtures' event decoder

    from paper_1805_04207_b200.tracefile import encode_event, load_trace

    events = events_from_json(case["events"])
    path = tmp_path / "v.aiwctrace"
    _write(path, [encode_event(e) for e in events])
    _, violation, err, _ = load_trace(str(path))
    assert err is None
    if case.get("error") == "InvalidStream":
        assert violation is not None and (violation[0], violation[1]) == (case["event_index"], case["rule"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["wavefront_big", "bfs_flags", "sweep4", "random31337_4", "branch_streams_per_group"])
def test_consume_file_report_matches_reference(name, tmp_path):
    from paper_1805_04207_b200 import finalize, report_to_dict
    from paper_1805_04207_b200.tracefile import consume_file, encode_event

    c, tr = {c["name"]: (c, t) for c, t in golden_cases() if t is not None}[name]
    path = tmp_path / "t.aiwctrace"
    _write(path, [encode_event(e) for e in _events(tr)])
    rep = report_to_dict(finalize(consume_file(str(path), max_entries=1 << 40)))
    assert_report_matches(rep, {k: v for k, v in c["report"].items() if k not in DERIVED})


@pytest.mark.gpu
def test_consume_file_cap_before_malformed_line(tmp_path):
    """TraceTooLarge wins when the cap is crossed before a malformed line (lazy consume order)."""
    from paper_1805_04207_b200 import MalformedEvent, TraceTooLarge
    from paper_1805_04207_b200.tracefile import consume_file

    head = ['{"ev":"kernel_begin","kernel":"k","invocation":0,"global_size":[1,1,1],"local_size":[1,1,1]}',
            '{"ev":"wg_begin","group":[0,0,0]}',
            '{"ev":"wi_begin","global":[0,0,0],"local":[0,0,0],"group":[0,0,0]}']
    mem = [f'{{"ev":"mem","op":"load","addr":{64 * k}}}' for k in range(6)]
    path = tmp_path / "c.aiwctrace"
    _write(path, head + mem + ["{oops", '{"ev":"kernel_end"}'])
    with pytest.raises(TraceTooLarge):
        consume_file(str(path), max_entries=3)
    with pytest.raises(MalformedEvent):
        consume_file(str(path), max_entries=100)


@pytest.mark.parametrize("name", ["wavefront_big", "bfs_flags", "random31337_4", "offgrid_groups", "branch_streams_per_group"])
def test_fast_parallel_parse_matches_walker(name, tmp_path):
    """encode_lines_fast (all host threads, chunk-local dictionaries merged in
    first-appearance order) gives the sequential walker's columns exactly."""
    from paper_1805_04207_b200.tracefile import encode_event, fast_trace, load_trace

    c, tr = {c["name"]: (c, t) for c, t in golden_cases() if t is not None}[name]
    path = tmp_path / "f.aiwctrace"
    _write(path, [encode_event(e) for e in _events(tr)])
    want, violation, err, _ = load_trace(str(path))
    assert violation is None and err is None
    for threads in (1, 3, 16):
        got = fast_trace(str(path), threads)
        assert got is not None and not got.validated
        assert np.array_equal(np.asarray(got.kind), np.asarray(want.kind))
        assert np.array_equal(np.asarray(got.payload).view(np.uint64), np.asarray(want.payload).view(np.uint64))
        assert got.opcodes == want.opcodes and got.extra_groups == want.extra_groups
        assert got.addr_stats == want.addr_stats and got.class_counts == want.class_counts


def test_fast_parse_declines_what_the_walker_must_decide(tmp_path):
    from paper_1805_04207_b200.tracefile import fast_trace

    head = ['{"ev":"kernel_begin","kernel":"k","invocation":0,"global_size":[2,1,1],"local_size":[2,1,1]}',
            '{"ev":"wg_begin","group":[0,0,0]}']
    cases = {
        "comment": head + ["# c", '{"ev":"kernel_end"}'],
        "bad_id": head + ['{"ev":"wi_begin","global":[1,0,0],"local":[0,0,0],"group":[0,0,0]}'],
        "other_group": head + ['{"ev":"wi_begin","global":[2,0,0],"local":[0,0,0],"group":[1,0,0]}'],
        "noncanonical": head + ['{"ev": "kernel_end"}'],
    }
    for name, lines in cases.items():
        path = tmp_path / f"{name}.aiwctrace"
        _write(path, lines)
        assert fast_trace(str(path), 4) is None, name


@pytest.mark.parametrize("name", ["wavefront_big", "bfs_flags", "offgrid_groups", "branch_streams_per_group", "single_item_no_barriers"])
def test_columnar_file_round_trip(name, tmp_path):
    """write_columnar / read_columnar: the columns and the launch metadata come back
    exactly, memory-mapped and untrusted."""
    from paper_1805_04207_b200.tracefile import is_columnar_file, read_columnar, write_columnar

    cases = {c["name"]: t for c, t in golden_cases() if t is not None}
    if name not in cases:
        pytest.skip(f"no golden trace {name}")
    tr = cases[name]
    path = str(tmp_path / "t.aiwcc")
    write_columnar(tr, path)
    assert is_columnar_file(path) and os.path.getsize(path) % 8 == 0
    got = read_columnar(path)
    assert not got.validated
    assert np.array_equal(np.asarray(got.kind), np.asarray(tr.kind))
    assert np.array_equal(np.asarray(got.payload).view(np.uint64), np.asarray(tr.payload).view(np.uint64))
    assert (got.kernel_name, got.invocation, tuple(got.global_size), tuple(got.local_size)) == \
        (tr.kernel_name, tr.invocation, tuple(tr.global_size), tuple(tr.local_size))
    assert got.opcodes == list(tr.opcodes) and got.extra_groups == [tuple(g) for g in tr.extra_groups]
    assert got.addr_stats == (tuple(tr.addr_stats) if tr.addr_stats is not None else None)


def test_columnar_file_rejects_damage(tmp_path):
    from paper_1805_04207_b200.tracefile import read_columnar, write_columnar

    tr = next(t for c, t in golden_cases() if t is not None and t.n_events > 100)
    path = tmp_path / "t.aiwcc"
    write_columnar(tr, str(path))
    data = path.read_bytes()
    (tmp_path / "short.aiwcc").write_bytes(data[:-9])
    with pytest.raises(ValueError, match="truncated"):
        read_columnar(str(tmp_path / "short.aiwcc"))
    (tmp_path / "magic.aiwcc").write_bytes(b"X" + data[1:])
    with pytest.raises(ValueError, match="not a columnar"):
        read_columnar(str(tmp_path / "magic.aiwcc"))
    (tmp_path / "head.aiwcc").write_bytes(data[:16] + b"X" + data[17:])
    with pytest.raises(ValueError, match="bad columnar header"):
        read_columnar(str(tmp_path / "head.aiwcc"))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["wavefront_big", "bfs_flags", "random31337_4", "branch_streams_per_group"])
def test_consume_columnar_file_matches_reference(name, tmp_path):
    """consume_file on the binary columnar form: the reference's report; a damaged
    stream inside a columnar file raises InvalidStream (the engine checks it)."""
    from paper_1805_04207_b200 import InvalidStream, finalize, report_to_dict
    from paper_1805_04207_b200.tracefile import consume_file, write_columnar
    from paper_1805_04207_b200.trace import ColumnarTrace

    c, tr = {c["name"]: (c, t) for c, t in golden_cases() if t is not None}[name]
    path = str(tmp_path / "t.aiwcc")
    write_columnar(tr, path)
    rep = report_to_dict(finalize(consume_file(path, max_entries=1 << 40)))
    assert_report_matches(rep, {k: v for k, v in c["report"].items() if k not in DERIVED})
    k = np.array(tr.kind, dtype=np.uint8).copy()
    k[-1] = 0x40  # kernel_end -> wg_begin
    bad = ColumnarTrace(k, tr.payload, tr.kernel_name, tr.invocation, tr.global_size, tr.local_size, tr.opcodes,
                        tr.extra_groups)
    write_columnar(bad, path)
    with pytest.raises(InvalidStream):
        consume_file(path, max_entries=1 << 40)
