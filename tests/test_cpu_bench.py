"""bench.py's reference arm on the CPU: its input comes from the pure-numpy
generator (bit-identical to the Python twin of the device generator), it never
maps the product library, it prints the same `config` the GPU arm prints, and
`--gpus N` spawns N ranks itself (rank 0 alone prints)."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT
from oracle import oracle, synth_np
from paper_1805_04207_b200 import synth


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_numpy_generator_matches_python_twin(cfg):
    w = synth_np.LOCAL[cfg] * 5
    kind, payload = synth_np.trace(cfg, w, chunk_groups=2)
    tw = synth.python_trace(cfg, w)
    assert np.array_equal(kind, tw.kind)
    assert np.array_equal(payload, tw.payload.view(np.uint64))
    assert synth_np.n_events(cfg, w) == kind.shape[0]


@pytest.mark.parametrize("cfg", [2, 5])
def test_reference_sample_prefix_is_a_closed_trace(cfg):
    """A prefix of whole work-groups closed by kernel_end equals the whole trace of
    that many work-items (the groups do not depend on the trace length except
    through buffer bases, which the oracle's statistics are invariant to)."""
    import bench

    class A:
        ref_sample_wi = synth_np.LOCAL[cfg] * 2

    wi, kind, payload = bench.reference_sample(cfg, synth_np.LOCAL[cfg] * 16, A, 2)
    assert wi == synth_np.LOCAL[cfg] * 2
    assert kind[0] == synth_np.K_KB and kind[-1] == synth_np.K_KE
    oracle.build()
    r = oracle.run(kind, payload, kernel=synth_np.NAMES[cfg], invocation=0, n_opcodes=len(synth_np.OPCODES[cfg]))
    assert r["work_items"] == wi


def _run(cmd, env=None):
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600,
                         env={**os.environ, **(env or {})})
    assert out.returncode == 0, out.stderr[-3000:]
    return out


PROBE = ("import runpy, sys; sys.argv = ['bench.py'] + sys.argv[1:]; "
         "runpy.run_path('bench.py', run_name='__main__'); "
         "maps = open('/proc/self/maps').read(); "
         "print('PRODUCT_SO_MAPPED' if 'libaiwc_b200' in maps else 'PRODUCT_SO_ABSENT')")


def test_reference_arm_never_maps_the_product_library_and_reports_our_config():
    import bench

    out = _run([sys.executable, "-c", PROBE, "--impl", "reference", "--config", "2", "--work-items", "4096",
                "--steps", "1", "--warmup", "0"])
    lines = out.stdout.strip().splitlines()
    assert lines[-1] == "PRODUCT_SO_ABSENT"
    line = json.loads(lines[-2])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["config"] == bench.bench_config(2, 1, 4096, "weak")
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"


def test_gpus_flag_spawns_ranks_and_rank0_prints():
    out = _run([sys.executable, "bench.py", "--gpus", "2", "--impl", "reference", "--config", "1", "--work-items",
                "4096", "--steps", "1", "--warmup", "0", "--scaling", "strong"])
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["work_items"] == 4096
