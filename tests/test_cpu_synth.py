"""Synthetic BASELINE configs on the CPU: the Python twin of the device
generator run through the C oracle reproduces the closed forms of SURVEY.md
§8d / Appendix B (recipe checks run with the reference there)."""

import math

import pytest

from oracle import oracle
from paper_1805_04207_b200 import synth


@pytest.fixture(scope="module", autouse=True)
def _built():
    oracle.build()


def test_c2_recipe_closed_forms():
    w = 1 << 14
    r = oracle.run_trace(synth.python_trace(2, w))
    assert r["total_memory_footprint"] == 9 * w == 147456
    assert r["footprint_90"] == math.ceil(0.9 * 9 * w) == 132711
    assert r["gmae"] == 17.1699250014  # log2(9 * 2^14), SURVEY App. B
    # 4-byte elements: skip levels 1, 2 keep every address distinct; level 3 drops one bit
    assert r["lmae"][0] == r["lmae"][1] == r["gmae"]
    assert abs(r["lmae"][2] - (r["lmae"][1] - 1.0)) < 1e-9
    assert r["opcode"] == 3 and r["min_itb"] == r["max_ipt"] == 21
    assert r["max_simd_width"] == 4 and r["mean_simd_width"] == 1.57142857143


def test_c4_recipe_closed_forms():
    r = oracle.run_trace(synth.python_trace(4, 1024))
    assert r["warmup_excluded_fraction"] == 0.001953125  # 16 / 8192 per stream... 16/(32*...) -> App. B
    assert r["total_unique_branch_instructions"] == 3
    assert r["min_itb"] == r["max_ipt"] == 192
    assert 0.0 < r["linear_entropy"] < 0.5 and 0.0 < r["yokota_entropy"] < 1.0


def test_c5_recipe_closed_forms():
    r = oracle.run_trace(synth.python_trace(5, 1024))
    assert r["min_itb"] == r["max_itb"] == 25 and r["mean_itb"] == 25.0
    assert r["min_ipt"] == r["max_ipt"] == 100
    assert r["total_barriers_hit"] * 25 == r["total_instruction_count"]
    assert r["mean_simd_width"] == 2.12


def test_c1_size_matches_reference_trace():
    # BASELINE configs[0]: sweep4 g=262144 l=64 has 1,056,770 events
    assert 2 + (262144 // 64) * (2 + 64 * 4) == 1056770


def test_event_counts_match_survey():
    per_group = {2: 2 + 256 * 32, 3: 2 + 256 * 32, 4: 2 + 256 * 322, 5: 2 + 256 * 122}
    want = {2: 268500994, 3: 2148007938, 4: 337649666, 5: 2046951426}
    for cfg, n in want.items():
        assert 2 + synth.FULL_WORK_ITEMS[cfg] // 256 * per_group[cfg] == n


@pytest.mark.parametrize("cfg,w", [(1, 4096), (2, 8192), (5, 4096)])
def test_shard_ranges_tile_the_trace_at_work_group_boundaries(cfg, w):
    from paper_1805_04207_b200.trace import K_WG_BEGIN

    tr = synth.python_trace(cfg, w)
    for world in (1, 2, 3, 8):
        pos = 0
        for r in range(world):
            first, count = synth.shard_range(cfg, w, r, world)
            assert first == pos
            assert first == 0 or tr.kind[first] == K_WG_BEGIN
            pos += count
        assert pos == tr.n_events
