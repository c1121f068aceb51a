"""BASELINE configs at their full sizes on the GPU against the multi-threaded
oracle (pinned to the reference by test_oracle_golden.py / test_oracle_mt.py):
C2 (268,500,994 events, the bench workload), C3 (2,148,007,938 events: dense
table with the hot-key window, u32 entries, 2^28-key random gathers), C4
(337,649,666 events: 100.7 M branch records, 12,288 streams) and C5
(2,046,951,426 events: 67 M barriers, lifetime IPT slots).  Counts must match
exactly, entropies to 1e-9.  The oracle uses every host thread (~30 s per
2 B-event config on a 16-core host)."""

import os

import numpy as np
import pytest

from conftest import assert_report_matches

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)


@pytest.mark.parametrize("cfg", [2, 4, 3, 5])
def test_full_size_config_matches_oracle(cfg):
    from oracle import oracle

    from paper_1805_04207_b200 import consume, finalize, report_to_dict, synth

    oracle.build()
    w = synth.FULL_WORK_ITEMS[cfg]
    tr = synth.device_trace(cfg, w)
    got = report_to_dict(finalize(consume(tr, max_entries=1 << 40)))
    kind = tr.kind.cpu().numpy()
    payload = tr.payload.cpu().numpy().view(np.uint64)
    del tr
    torch.cuda.empty_cache()
    want = oracle.run(kind, payload, kernel=got["kernel"], invocation=0, n_opcodes=len(synth.OPCODES[cfg]),
                      threads=max(1, os.cpu_count() or 1))
    want = {k: v for k, v in want.items() if k in got}
    assert_report_matches(got, want)
