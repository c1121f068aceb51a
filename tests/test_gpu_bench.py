"""bench.py end to end on the GPU at a small size: the driver's JSON contract
(keys, units, roofline / e2e / clocks objects) and the multi-GPU shard path
under torchrun + NCCL at one rank (AIWC_BENCH_SHARDED=1: NCCL collectives,
the address exchange, the sharded e2e report), whose report must equal the
single-GPU path's."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

ARGS = ["--config", "2", "--work-items", "65536", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"]


def _line(cmd, env=None):
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600,
                         env={**os.environ, **(env or {})})
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_bench_contract_and_sharded_path_agree():
    single = _line([sys.executable, "bench.py", *ARGS])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "clocks", "gpu_launches"):
        assert key in single, key
    assert single["value"] > 0 and single["e2e"]["value"] > 0 and single["gpu_launches"] > 0
    assert single["roofline"]["bound"] == "hbm" and 0 < single["roofline"]["frac"] < 1
    # the timed steps checked the stream inside the pass and certified it
    assert single["stream_check"]["in_pass"] and single["stream_check"]["certified"] is True
    assert single["roofline"]["frac"] <= single["roofline"]["frac_without_stream_check"] < 1
    e2e = single["e2e"]
    assert e2e["h2d_bytes_per_step"] > 0 and e2e["bare_h2d_gbs"] > 0 and 0 < e2e["link_frac"] < 1.2
    sharded = _line([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                     "--master-addr", "127.0.0.1", "--master-port", "29561", "bench.py", "--gpus", "1", *ARGS],
                    env={"AIWC_BENCH_SHARDED": "1"})
    assert "concurrent shard streams" in sharded["lanes"]["how"]
    assert sharded["config"] == single["config"]
    assert sharded["report_check"] == single["report_check"]
