"""Synthetic BASELINE configs on the GPU: generator agreement, the C1 oracle
config against the reference's own report, and small-scale parity of C2-C5
against the C oracle plus their closed forms."""

import math

import numpy as np
import pytest

from conftest import assert_report_matches, golden_cases

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle import oracle  # noqa: E402
from paper_1805_04207_b200 import consume, finalize, report_to_dict  # noqa: E402
from paper_1805_04207_b200 import synth  # noqa: E402

SMALL = {1: 4096, 2: 4096, 3: 2048, 4: 1024, 5: 1024}


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_device_generator_matches_python_twin(cfg):
    w = SMALL[cfg]
    dev = synth.device_trace(cfg, w)
    ref = synth.python_trace(cfg, w)
    assert np.array_equal(dev.kind.cpu().numpy(), ref.kind)
    assert np.array_equal(dev.payload.cpu().numpy().view(np.uint64), ref.payload)
    assert synth.n_events(cfg, w) == ref.n_events


@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_numpy_generator_matches_device_generator(cfg):
    """oracle/synth_np.py (the reference arm's input) against the device generator."""
    from oracle import synth_np

    w = 1 << 14
    dev = synth.device_trace(cfg, w)
    kind, payload = synth_np.trace(cfg, w)
    assert np.array_equal(dev.kind.cpu().numpy(), kind)
    assert np.array_equal(dev.payload.cpu().numpy().view(np.uint64), payload)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_small_configs_match_oracle(cfg):
    tr = synth.device_trace(cfg, SMALL[cfg])
    got = report_to_dict(finalize(consume(tr, max_entries=1 << 40)))
    host = tr.to_numpy()
    want = oracle.run(host.kind, host.payload.view(np.uint64), kernel=host.kernel_name, invocation=0,
                      n_opcodes=len(host.opcodes))
    assert_report_matches(got, want)


def test_c1_full_matches_reference_report():
    """BASELINE configs[0]: the reference's report for sweep4 g=262144 l=64."""
    case = next(c for c, _ in golden_cases() if c["name"] == "C1_sweep4_262144")
    tr = synth.device_trace(1, 262144)
    assert tr.n_events == case["n_events"] == 1056770
    got = report_to_dict(finalize(consume(tr, max_entries=1 << 40)))
    assert_report_matches(got, case["report"])


def test_c2_closed_forms_scaled():
    w = 1 << 16
    r = finalize(consume(synth.device_trace(2, w), max_entries=1 << 40))
    u = 9 * w
    assert r.total_memory_footprint == u and r.unique_reads == 8 * w and r.unique_writes == w
    assert r.footprint_90 == math.ceil(0.9 * u)
    assert abs(r.gmae - math.log2(u)) < 1e-9
    assert r.reread_ratio == 1.0 and r.rewrite_ratio == 1.0
    assert r.min_itb == r.max_itb == 21 and r.min_ipt == r.max_ipt == 21
    assert r.opcode == 3


def test_c5_barrier_density_scaled():
    r = finalize(consume(synth.device_trace(5, 4096), max_entries=1 << 40))
    assert r.min_itb == r.max_itb == 25 and r.mean_itb == 25.0
    assert r.min_ipt == r.max_ipt == 100
    assert r.total_barriers_hit * 25 == r.total_instruction_count
