"""Randomized differential stress test: valid columnar traces drawn from wide
parameter ranges -- large opcode dictionaries (> 256 ids, the non-DevState
counter path), widths outside the 1..16 fast bins, many branch sites (> 256,
the big site list), streams longer than the 16-bit history, sparse 64-bit
address spaces (sort path) and hot keys (u64 dense table), barriers with
resumes (lifetime IPT slots), empty work-items and groups -- through the CUDA
engine and through the oracle (pinned to the reference by
test_oracle_golden.py).  Counts must match exactly, entropies to 1e-9."""

import random

import numpy as np
import pytest

from conftest import assert_report_matches

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

K = dict(KB=0x20, KE=0xA0, WGB=0x40, WGE=0xC0, WIB=0x30, WIR=0xB0, WIE=0x10, BAR=0x90, INS=0x01, LD=0x02,
         ALD=0x82, ST=0x04, AST=0x84, BR=0x08)


def random_trace(rng: random.Random):
    """A valid stream: groups in order, work-items sequential until a barrier,
    every work-item of a group hitting the same number of barriers."""
    from paper_1805_04207_b200.trace import ColumnarTrace

    lv = rng.choice([1, 3, 16, 64])
    groups = rng.randint(1, 12)
    n_opc = rng.choice([3, 20, 300])
    n_bar = rng.choice([0, 0, 1, 3])
    addr_mode = rng.choice(["dense", "hot", "sparse64", "strided"])
    widths = rng.choice([[1], [1, 2, 4, 8, 16], [1, 3, 17, 255, 4096, 65535]])
    sites = rng.choice([3, 40, 600])
    kinds, pays = [K["KB"]], [0]

    def addr():
        if addr_mode == "dense":
            return 4096 + 4 * rng.randrange(1 << 14)
        if addr_mode == "hot":
            return 1 << 20 | 8 * rng.randrange(8)
        if addr_mode == "strided":
            return (rng.randrange(64) << 12) | 0x80
        return rng.getrandbits(64) & ~3

    def segment(lid):
        for _ in range(rng.randint(0, 30)):
            r = rng.random()
            if r < 0.5:
                kinds.append(K["INS"])
                pays.append(rng.randrange(n_opc) << 32 | rng.choice(widths))
            elif r < 0.8:
                kinds.append(rng.choice([K["LD"], K["ALD"], K["ST"], K["AST"]]))
                pays.append(addr())
            else:
                kinds.append(K["BR"])
                pays.append(rng.randrange(sites) << 1 | rng.randrange(2))

    for g in range(groups):
        kinds.append(K["WGB"]); pays.append(g)
        order = list(range(lv))
        active = rng.sample(order, rng.randint(0, lv))  # some groups run no work-item at all
        for lid in active:
            kinds.append(K["WIB"]); pays.append(lid)
            segment(lid)
            if n_bar:
                kinds.append(K["BAR"]); pays.append(0)
            else:
                kinds.append(K["WIE"]); pays.append(lid)
        for b in range(n_bar):
            for lid in active:
                kinds.append(K["WIR"]); pays.append(lid)
                segment(lid)
                if b + 1 < n_bar:
                    kinds.append(K["BAR"]); pays.append(0)
                else:
                    kinds.append(K["WIE"]); pays.append(lid)
        kinds.append(K["WGE"]); pays.append(g)
    kinds.append(K["KE"]); pays.append(0)
    return ColumnarTrace(np.array(kinds, np.uint8), np.array(pays, np.uint64), "stress", 0, (groups * lv, 1, 1),
                         (lv, 1, 1), [f"op{i}" for i in range(n_opc)], [])


@pytest.mark.parametrize("seed", range(60))
def test_random_traces_match_oracle(seed):
    from oracle import oracle

    from paper_1805_04207_b200 import consume, finalize, report_to_dict
    from paper_1805_04207_b200.metrics import validate_columnar

    oracle.build()
    rng = random.Random(1000 + seed)
    tr = random_trace(rng)
    assert validate_columnar(tr, 0) is None  # the generator's streams are valid
    want = oracle.run_trace(tr)
    host = report_to_dict(finalize(consume(tr, max_entries=1 << 40)))
    assert_report_matches(host, want)
    dev = type(tr)(torch.from_numpy(tr.kind).cuda(), torch.from_numpy(tr.payload.view(np.int64)).cuda(),
                   tr.kernel_name, 0, tr.global_size, tr.local_size, tr.opcodes, [], validated=True)
    assert_report_matches(report_to_dict(finalize(consume(dev, max_entries=1 << 40))), want)
