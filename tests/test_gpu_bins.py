"""Key-block bins (aiwc_bins.cu): accesses into key zones the sampler finds
random are appended to per-warp bin segments, partitioned by key block and
counted in shared memory instead of REDed into a table far larger than L2.
AIWC_BINS=2 makes small traces eligible; reports must equal the engine's
without bins (AIWC_BINS=0), the C oracle's and, for golden traces, the
reference's."""

import subprocess
import sys
import json

import pytest

from conftest import ROOT, assert_report_matches, golden_cases

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

PROBE = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
import numpy as np, torch
from paper_1805_04207_b200 import consume, finalize, report_to_dict, synth
from paper_1805_04207_b200.trace import ColumnarTrace
sys.path.insert(0, sys.argv[1] + "/tests")
from conftest import golden_cases
out = {}
for cfg, w in ((3, 1 << 16), (3, 1 << 14), (2, 1 << 15), (5, 1 << 13)):
    acc = consume(synth.device_trace(cfg, w), max_entries=1 << 40)
    out[f"C{cfg}_{w}"] = report_to_dict(finalize(acc))
    out[f"C{cfg}_{w}"]["__binned"] = acc.result.binned_accesses
for c, tr in golden_cases():
    if tr is None or "error" in c or not c["name"].startswith(("random31337", "hot_address", "bfs")):
        continue
    dev = ColumnarTrace(torch.from_numpy(tr.kind.copy()).cuda(), torch.from_numpy(tr.payload.view(np.int64).copy()).cuda(),
                        tr.kernel_name, tr.invocation, tr.global_size, tr.local_size, tr.opcodes, tr.extra_groups)
    out[c["name"]] = report_to_dict(finalize(consume(dev, max_entries=1 << 40)))
print(json.dumps(out))
"""


def _run(bins: str):
    env = {"AIWC_BINS": bins}
    import os

    out = subprocess.run([sys.executable, "-c", PROBE, ROOT], capture_output=True, text=True, timeout=600,
                         env={**os.environ, **env})
    assert out.returncode == 0, out.stderr[-3000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_binned_reports_match_unbinned_and_reference():
    binned, plain = _run("2"), _run("0")
    assert binned.keys() == plain.keys()
    # C3's gathers are random: the sampler bins them (and only with AIWC_BINS != 0)
    assert binned["C3_65536"].pop("__binned") > 0 and plain["C3_65536"].pop("__binned") == 0
    for name in binned:
        binned[name].pop("__binned", None)
        plain[name].pop("__binned", None)
    want = {c["name"]: c["report"] for c, _ in golden_cases() if "report" in c}
    for name, rep in binned.items():
        assert_report_matches(rep, plain[name])
        if name in want:
            assert_report_matches(rep, want[name])
