"""Host side of the NDRange producer against the reference's own outputs
(tests/golden/sim.json, written by tests/golden/make_sim.py): the `.aiwck`
parser (ir.py:300-374) -- program structure or error class / line / message --
the buffer specs (buffers.py:27-72), launch validation and buffer bases
(sim.py:88-141), and the bytecode lowering."""

import json
import os

import numpy as np
import pytest

from paper_1805_04207_b200 import buffers, errors, ir, sim

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "sim.json")))


@pytest.mark.parametrize("case", GOLD["parse"], ids=lambda c: repr(c["source"][:40]))
def test_parse_matches_reference(case):
    if "program" in case:
        assert repr(ir.parse_kernel(case["source"])) == case["program"]
        return
    with pytest.raises(errors.ParseError) as exc:
        ir.parse_kernel(case["source"])
    assert type(exc.value).__name__ == case["error"]
    assert exc.value.line == case["line"]
    assert str(exc.value) == case["message"]


def test_sim_case_sources_parse_like_reference():
    # every simulator golden's kernel parses, and lowers to bytecode
    for case in GOLD["cases"]:
        cp = ir.compile_program(ir.parse_kernel(case["source"]))
        assert cp.code.shape[1] == ir.SIM_WORDS and cp.code.dtype == np.int32
        assert len(cp.lines) == cp.code.shape[0]


@pytest.mark.parametrize("case", GOLD["buffers"], ids=lambda c: c["spec"])
def test_buffer_specs_match_reference(case):
    if "values" in case:
        assert buffers.make_buffer(case["spec"], 12, 5) == case["values"]
        return
    with pytest.raises(Exception) as exc:
        buffers.make_buffer(case["spec"], 12, 5)
    assert type(exc.value).__name__ == case["error"]
    assert str(exc.value) == case["message"]


def test_buffer_file_spec(tmp_path):
    p = tmp_path / "v.txt"
    p.write_text("1 0x10 -1\n7")
    assert buffers.make_buffer(f"file:{p}", 3) == [1, 16, (1 << 64) - 1, 7]


def test_assign_bases_reference_layout():
    # test_sim.py:379-383
    bases = sim.assign_bases(("a", "b", "c"), {"a": [0] * 3000, "b": [0], "c": [0] * 10})
    assert bases["a"] == 4096
    assert bases["b"] == 4096 + 12288
    assert all(b % 4096 == 0 for b in bases.values())


@pytest.mark.parametrize("cfg,match", [
    (sim.NDRangeConfig((10, 1, 1), (4, 1, 1)), "divide"),
    (sim.NDRangeConfig((0, 1, 1), (1, 1, 1)), "global_size must be three positive integers"),
    (sim.NDRangeConfig((4, 1), (1, 1, 1)), "global_size"),
    (sim.NDRangeConfig((4, 1, 1), (1, 1, 1), {"a": [0] * 4, "b": [0]}, {"a": 4096, "b": 4100}), "overlap"),
    (sim.NDRangeConfig((4, 1, 1), (1, 1, 1), {"a": [0]}, {}), "no base address"),
    (sim.NDRangeConfig((4, 1, 1), (1, 1, 1), {"a": [0] * 2}, {"a": (1 << 64) - 4}), "does not fit"),
])
def test_config_rejections(cfg, match):
    with pytest.raises(errors.ConfigError, match=match):
        cfg.validate()


def test_missing_buffer_rejected_at_call_time():
    prog = ir.parse_kernel("kernel k(a)\nentry:\n  load r0, buf[a][0]\n  ret\n")
    with pytest.raises(errors.ConfigError, match="'a'"):
        sim.simulate_events(prog, sim.NDRangeConfig((1, 1, 1), (1, 1, 1), {}))


def test_bytecode_layout():
    prog = ir.parse_kernel("kernel k(a)\nentry:\n  fmul.x2 r1, 5, gid0\n  aload r0, buf[a][r1]\n"
                           "  br r0, entry, out\nout:\n  ret\n")
    cp = ir.compile_program(prog)
    assert cp.opcodes == ["fmul", "aload", "br"]
    mul, ld, br, ret = cp.code.tolist()
    assert mul[:4] == [ir.K_COMPUTE, ir.SEM_IDS["mul"], 2, 1]
    assert mul[4] == (ir.OPND_IMM << 30) | 0 and cp.imm[0] == 5
    assert mul[5] & 0xFFFFFFFF == (ir.OPND_BUILTIN << 30) | 0  # int32 storage, read as u32
    assert ld[:2] == [ir.K_LOAD, 1] and ld[4] == 1 and ld[7] == 0
    assert br[0] == ir.K_BR and br[8:10] == [0, 3] and br[11] == 5
    assert ret[0] == ir.K_RET
    assert cp.max_width == 2 and cp.n_regs == 2
