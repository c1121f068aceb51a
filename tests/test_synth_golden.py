"""Scaled samples of the synthetic BASELINE configs C1..C5 against the
REFERENCE implementation's own reports (tests/golden/synth.json, written by
tests/golden/make_synth_golden.py): the C oracle on the numpy generator's
trace (CPU), and the CUDA engine on the device generator's trace (GPU)."""

import json
import os

import numpy as np
import pytest

from conftest import ROOT, assert_report_matches

with open(os.path.join(ROOT, "tests", "golden", "synth.json"), encoding="utf-8") as fp:
    SAMPLES = json.load(fp)["samples"]
IDS = [f"C{s['config']}_{s['work_items']}" for s in SAMPLES]
DERIVED = ("granularity", "barriers_per_instruction", "instructions_per_operand", "load_imbalance")


@pytest.mark.parametrize("s", SAMPLES, ids=IDS)
def test_oracle_matches_reference_on_synthetic_samples(s):
    from oracle import oracle, synth_np

    oracle.build()
    kind, payload = synth_np.trace(s["config"], s["work_items"])
    assert kind.shape[0] == s["n_events"]
    got = oracle.run(kind, payload, kernel=synth_np.NAMES[s["config"]], invocation=0,
                     n_opcodes=len(synth_np.OPCODES[s["config"]]))
    assert_report_matches(got, s["report"], skip=DERIVED)  # the oracle reports the AiwcReport fields only


@pytest.mark.gpu
@pytest.mark.parametrize("s", SAMPLES, ids=IDS)
def test_engine_matches_reference_on_synthetic_samples(s):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():  # pragma: no cover
        pytest.skip("no CUDA device")
    from paper_1805_04207_b200 import consume, finalize, report_to_dict, synth

    tr = synth.device_trace(s["config"], s["work_items"])
    assert tr.n_events == s["n_events"]
    got = report_to_dict(finalize(consume(tr, max_entries=1 << 40)))
    assert_report_matches(got, s["report"])
