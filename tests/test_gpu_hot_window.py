"""Dense-table paths at sizes where the hot-key window is eligible (>= 2^20
memory accesses, more than 1024 keys): traces mixing a contended block of
keys (unaligned, so it straddles two 1024-key blocks), random accesses over a
wide range and streaming accesses, with reads and writes, at densities that
select the u32 (count | flags) and the u64 (reads | writes) table, one or two
hot blocks, and byte / 4-byte / 8-byte address granularity.  Whatever block
the sampler elects (or none), the report must equal the oracle's: counts
exact, entropies to 1e-9."""

import numpy as np
import pytest

from conftest import assert_report_matches

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

KB, KE, WGB, WGE, WIB, WIE, INS, LD, ST = 0x20, 0xA0, 0x40, 0xC0, 0x30, 0x10, 0x01, 0x02, 0x04

# mode: (hot share, random share, random range, write share, element size, two hot blocks, streaming range)
# (ranges in elements; M = 1.31 M accesses)
MODES = {
    "scratch_u32": (0.35, 0.15, 1 << 21, 0.1, 4, False, 1 << 20),   # < 1 access per key: u32 + window
    "scratch_u64": (0.60, 0.05, 1 << 14, 0.2, 4, False, 1 << 15),   # > 4 accesses per key: u64 + window
    "dense_mid": (0.30, 0.20, 1 << 18, 0.3, 4, False, 1 << 18),     # 1..4 accesses per key: u32 + window
    "hot_writes": (0.30, 0.30, 1 << 21, 0.5, 4, False, 1 << 20),    # hot block written and read
    "two_hot": (0.40, 0.10, 1 << 19, 0.1, 8, True, 1 << 19),        # window takes one block, L2 the other
    "no_hot": (0.00, 0.60, 1 << 21, 0.2, 4, False, 1 << 20),        # nothing hot: no window
    "bytes_sparse": (0.05, 0.90, 1 << 26, 0.1, 1, False, 1 << 20),  # span too wide: compacted (sort) path
}


def hot_trace(mode: str, seed: int, W: int = 1 << 15, A: int = 40, LV: int = 64):
    from paper_1805_04207_b200.trace import ColumnarTrace

    p_hot, p_rand, rng_elems, p_wr, esz, two, seq_elems = MODES[mode]
    rng = np.random.default_rng(seed)
    G = W // LV
    gid = np.arange(W, dtype=np.uint64)[:, None]
    j = np.arange(A, dtype=np.uint64)[None, :]
    u = rng.random((W, A))
    # buffers 4096-aligned and close together (the dense table spans all of them)
    hot_base = 1 << 20
    far_base = hot_base + (1 << 14)
    rand_base = far_base + (1 << 16)
    seq_base = rand_base + ((esz * rng_elems + 4095) & ~4095)
    hot = hot_base + esz * (600 + rng.integers(0, 700, (W, A), dtype=np.uint64))
    if two:
        far = far_base + esz * rng.integers(0, 300, (W, A), dtype=np.uint64)
        hot = np.where(rng.random((W, A)) < 0.4, far, hot)
    rand = rand_base + esz * rng.integers(0, rng_elems, (W, A), dtype=np.uint64)
    seq = seq_base + esz * ((gid * np.uint64(A) + j) % np.uint64(seq_elems))
    addr = np.where(u < p_hot, hot, np.where(u < p_hot + p_rand, rand, seq)).astype(np.uint64)
    mk = np.where(rng.random((W, A)) < p_wr, ST, LD).astype(np.uint8)
    # work-item rows: WIB, (INS, MEM) x A, WIE
    per = 2 + 2 * A
    k = np.empty((W, per), np.uint8)
    p = np.empty((W, per), np.uint64)
    lid = (np.arange(W) % LV).astype(np.uint64)
    k[:, 0], p[:, 0] = WIB, lid
    k[:, -1], p[:, -1] = WIE, lid
    k[:, 1:-1:2], p[:, 1:-1:2] = INS, (np.where(mk == ST, 1, 0).astype(np.uint64) << np.uint64(32)) | np.uint64(1)
    k[:, 2:-1:2], p[:, 2:-1:2] = mk, addr
    # group rows: WGB, LV work-items, WGE
    k = k.reshape(G, LV * per)
    p = p.reshape(G, LV * per)
    g = np.arange(G, dtype=np.uint64)[:, None]
    k = np.hstack([np.full((G, 1), WGB, np.uint8), k, np.full((G, 1), WGE, np.uint8)]).reshape(-1)
    p = np.hstack([g, p, g]).reshape(-1)
    k = np.concatenate([[KB], k, [KE]]).astype(np.uint8)
    p = np.concatenate([[0], p, [0]]).astype(np.uint64)
    return ColumnarTrace(k, p, f"hot_{mode}", 0, (W, 1, 1), (LV, 1, 1), ["load", "store"], [])


@pytest.mark.parametrize("mode", sorted(MODES))
def test_hot_window_traces_match_oracle(mode):
    from oracle import oracle

    from paper_1805_04207_b200 import consume, finalize, report_to_dict
    from paper_1805_04207_b200.metrics import validate_columnar

    oracle.build()
    tr = hot_trace(mode, seed=len(mode))
    n_mem = int(np.count_nonzero((tr.kind == LD) | (tr.kind == ST)))
    assert n_mem >= 1 << 20  # large enough for the window sampler
    want = oracle.run_trace(tr)
    assert validate_columnar(tr, 0) is None
    dev = type(tr)(torch.from_numpy(tr.kind).cuda(), torch.from_numpy(tr.payload.view(np.int64)).cuda(),
                   tr.kernel_name, 0, tr.global_size, tr.local_size, tr.opcodes, [], validated=True)
    assert_report_matches(report_to_dict(finalize(consume(dev, max_entries=1 << 40))), want)
