"""Wide address spans made of a few clustered buffers (far apart in the 64-bit
space, e.g. heap and stack) take the dense path through region compaction:
occupied 1 MB regions are squeezed together with their low 20 bits kept, which
preserves every address group of LSB-skip levels <= 10.  Reports must equal
the oracle's on the original addresses; traces touching too many regions keep
the sparse (sort) path, also checked."""

import numpy as np
import pytest

from conftest import assert_report_matches

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from test_gpu_hot_window import LD, ST, hot_trace  # noqa: E402

# remap the trace's buffers (hot / far / random / streaming bases of hot_trace) far apart
SPREADS = {
    "two_far": [1 << 40, 1 << 46],
    "three_far": [1 << 32, 0x7F0000000000, 0x5500000000],
    "byte_offsets": [(1 << 44) + 3, (1 << 45) + 1],   # misaligned: constant low bits differ
    "many_regions": None,                             # every access its own region: sparse path
}


def spread_trace(name: str, mode: str = "dense_mid"):
    tr = hot_trace(mode, seed=7, W=1 << 13)
    k, p = tr.kind.copy(), tr.payload.copy()
    mem = (k == LD) | (k == ST)
    a = p[mem]
    if SPREADS[name] is None:
        a = (a * np.uint64(0x9E3779B97F4A7C15)) & np.uint64((1 << 60) - 1) & ~np.uint64(3)
    else:
        bases = np.array(SPREADS[name], dtype=np.uint64)
        # buffer of each address by its original 1 MB region, moved to one of the bases
        reg = a >> np.uint64(20)
        ureg, inv = np.unique(reg, return_inverse=True)
        a = bases[inv % len(bases)] + (ureg[inv] - ureg.min()) * np.uint64(1 << 20) + (a & np.uint64((1 << 20) - 1))
    p[mem] = a
    return type(tr)(k, p, tr.kernel_name, 0, tr.global_size, tr.local_size, tr.opcodes, [], validated=True)


@pytest.mark.parametrize("name", sorted(SPREADS))
def test_clustered_spans_match_oracle(name):
    from oracle import oracle

    from paper_1805_04207_b200 import consume, finalize, report_to_dict

    oracle.build()
    tr = spread_trace(name)
    want = oracle.run_trace(tr)
    dev = type(tr)(torch.from_numpy(tr.kind).cuda(), torch.from_numpy(tr.payload.view(np.int64)).cuda(),
                   tr.kernel_name, 0, tr.global_size, tr.local_size, tr.opcodes, [], validated=True)
    acc = consume(dev, max_entries=1 << 40)
    assert_report_matches(report_to_dict(finalize(acc)), want)
    assert acc.result.used_dense_table == (SPREADS[name] is not None)
