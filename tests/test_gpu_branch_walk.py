"""Branch statistics: the sort-free walk (<= 64 sites, csrc/aiwc_branch.cu
bw_*_kernel) and the site-sort path against the C oracle, on random traces
built to stress stream boundaries: short and long work-groups, repeated group
ids (A B A: the third block's streams continue the first's, reference
metrics.py:145-152), sites that skip groups, periodic and random outcomes,
history lengths 1..16, and tiles / ranges forced down to 32 records so state
carries across every tile and range boundary (AIWC_BRANCH_TILE / _RANGE).  Bit-exact counts,
reals within 1e-9 (north_star)."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from branch_cases import CASES, HS, K_BRANCH, make_trace  # noqa: E402


RUNNER = r"""
import ctypes, json, sys
import numpy as np, torch
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
from branch_cases import CASES, HS, make_trace
from paper_1805_04207_b200 import _native
from paper_1805_04207_b200.metrics import ingest_columns, _copy_result
from paper_1805_04207_b200.trace import ColumnarTrace
ctxs = {H: _native.Context(0, history_len=H) for H in HS}
out = []
for case in CASES:
    k, p, w, lv = make_trace(*case)
    tr = ColumnarTrace(torch.from_numpy(k).cuda(), torch.from_numpy(p.view(np.int64)).cuda(), "bw", 0,
                       (w, 1, 1), (lv, 1, 1), ["br"], [])
    for H in HS:
        ctx = ctxs[H]
        ctx.check(ctx.lib.aiwc_reset(ctx.h))
        stream = ingest_columns(ctx, tr, False, False)
        res = _native.Result()
        ctx.check(ctx.lib.aiwc_finalize(ctx.h, ctypes.byref(res), ctypes.c_void_p(stream) if stream else None))
        r = _copy_result(res)
        out.append(dict(yokota=r.yokota, linear=r.linear, obs=r.branch_observations, excl=r.branch_excluded,
                        execs=r.branch_executions, b90=r.branch_90, sites=sorted(map(list, r.sites))))
print("JSON" + json.dumps(out))
"""


def _engine_reports(env):
    r = subprocess.run([sys.executable, "-c", RUNNER], cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env={**os.environ, **env})
    assert r.returncode == 0, r.stderr[-3000:]
    line = next(ln for ln in r.stdout.splitlines() if ln.startswith("JSON"))
    return json.loads(line[4:])


@pytest.fixture(scope="module")
def expected():
    from oracle import oracle
    oracle.build()
    out = []
    for case in CASES:
        k, p, w, lv = make_trace(*case)
        br = p[k == K_BRANCH] >> np.uint64(1)
        ids, cnt = np.unique(br, return_counts=True)
        sites = [[int(a), int(b)] for a, b in zip(ids, cnt)]
        for H in HS:
            out.append((oracle.run(k, p, kernel="bw", invocation=0, n_opcodes=1, history_len=H), sites))
    return out


def _r12(x):
    return round(x, 12) + 0.0


@pytest.mark.parametrize("env", [{}, {"AIWC_BRANCH_TILE": "32", "AIWC_BRANCH_RANGE": "1"},
                                 {"AIWC_BRANCH_TILE": "96", "AIWC_BRANCH_RANGE": "3"},
                                 {"AIWC_BRANCH_TILE": "1000", "AIWC_BRANCH_RANGE": "2"}, {"AIWC_BRANCH_SORT": "1"}],
                         ids=["walk", "tile32-range1", "tile96-range3", "tile1000-range2", "sort"])
def test_branch_paths_match_oracle(env, expected):
    got = _engine_reports(env)
    assert len(got) == len(expected)
    for i, (g, (want, sites)) in enumerate(zip(got, expected)):
        ctx = f"case {CASES[i // len(HS)]} H={HS[i % len(HS)]}"
        assert g["sites"] == sites, ctx
        assert g["b90"] == want["branch_90"], ctx
        assert g["execs"] == sum(c for _, c in sites), ctx
        if want["no_branches"] or want["warmup_excluded_fraction"] == 1.0:
            assert g["obs"] == 0, ctx
            continue
        assert _r12(g["excl"] / g["execs"]) == pytest.approx(want["warmup_excluded_fraction"], rel=1e-9, abs=1e-12), ctx
        assert _r12(g["yokota"]) == pytest.approx(want["yokota_entropy"], rel=1e-9, abs=1e-12), ctx
        assert _r12(g["linear"]) == pytest.approx(want["linear_entropy"], rel=1e-9, abs=1e-12), ctx
