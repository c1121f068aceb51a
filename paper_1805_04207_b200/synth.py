"""Synthetic BASELINE traces -- generated on the device.

``device_trace(cfg, work_items)`` fills CUDA columns with aiwc_synth_fill
(csrc/aiwc_synth.cu).  ``python_trace`` is the event-by-event Python twin of
the same formulas, used only to cross-check the device generator on small
sizes (tests) -- it is not on any product path.

    cfg 1  C1  sweep4 (reference kernel pkg/kernels/sweep4.aiwck, --buf a=iota), local 64
    cfg 2  C2  kmeans-like streaming, local 256                 (BASELINE configs[1]: 2^23 WI)
    cfg 3  C3  mixed global / shared-scratch / gather, local 256 (configs[2]: 2^26 WI)
    cfg 4  C4  branch-heavy CRC/coin/loop sites, local 256       (configs[3]: 2^20 WI)
    cfg 5  C5  barrier-heavy 4-stage, local 256                  (configs[4]: 2^24 WI)
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .trace import ColumnarTrace

FULL_WORK_ITEMS = {1: 262144, 2: 1 << 23, 3: 1 << 26, 4: 1 << 20, 5: 1 << 24}
NAMES = {1: "sweep4", 2: "kmeans_stream", 3: "mixed_global_local", 4: "branchy_crc", 5: "barrier_stages"}
OPCODES = {
    1: ["load"],
    2: ["load", "store", "fmul", "fadd"],
    3: ["load", "store", "fmul", "fadd"],
    4: ["load", "store", "xor", "br", "add"],
    5: ["load", "store", "barrier", "fmul", "fadd", "fma"],
}
LOCAL = {1: 64, 2: 256, 3: 256, 4: 256, 5: 256}
DEFAULT_SEED = 7


def info(cfg: int, work_items: int) -> _native.TraceInfo:
    lib = _native.load_library()
    ti = _native.TraceInfo()
    n = lib.aiwc_synth_size(cfg, work_items, ctypes.byref(ti))
    if n == 0:
        raise ValueError(f"bad synthetic config {cfg} / {work_items} work-items")
    return ti


def n_events(cfg: int, work_items: int) -> int:
    return int(info(cfg, work_items).n_events)


def shard_range(cfg: int, work_items: int, rank: int, world: int) -> tuple[int, int]:
    """(first event, event count) of rank's contiguous work-group shard.

    Layout (aiwc_synth.cu): KERNEL_BEGIN, then `groups` work-groups of equal
    length, then KERNEL_END; rank 0 also takes the kernel begin and the last
    rank the kernel end, so the shards tile the whole trace."""
    n = n_events(cfg, work_items)
    groups = work_items // LOCAL[cfg]
    per_group = (n - 2) // groups
    g_lo, g_hi = groups * rank // world, groups * (rank + 1) // world
    first = 0 if rank == 0 else 1 + g_lo * per_group
    end = n if rank == world - 1 else 1 + g_hi * per_group
    return first, end - first


def _columnar(cfg: int, work_items: int, kind, payload, ti, whole: bool = True) -> ColumnarTrace:
    lv = LOCAL[cfg]
    counts = (ti.n_instr, ti.n_reads, ti.n_writes, ti.n_branches, ti.n_groups, ti.any_barrier_or_resume) if whole else None
    return ColumnarTrace(kind, payload, NAMES[cfg], 0, (work_items, 1, 1), (lv, 1, 1), list(OPCODES[cfg]), [],
                         (ti.addr_min, ti.addr_max, ti.addr_and, ti.addr_or), validated=True, class_counts=counts)


def device_trace(cfg: int, work_items: int | None = None, seed: int = DEFAULT_SEED, device: int = 0,
                 first: int = 0, count: int | None = None):
    """Generate (a slice of) config `cfg` straight into CUDA memory."""
    import torch

    w = FULL_WORK_ITEMS[cfg] if work_items is None else work_items
    ti = info(cfg, w)
    n = int(ti.n_events) - first if count is None else count
    dev = torch.device("cuda", device)
    kind = torch.empty(n, dtype=torch.uint8, device=dev)
    payload = torch.empty(n, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    rc = _native.load_library().aiwc_synth_fill(cfg, w, seed, ctypes.c_void_p(kind.data_ptr()),
                                                ctypes.c_void_p(payload.data_ptr()), first, n,
                                                ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(f"aiwc_synth_fill failed ({rc})")
    return _columnar(cfg, w, kind, payload, ti, whole=(first == 0 and n == int(ti.n_events)))


# ---------------------------------------------------------------------------
# Python twin (tests only)
# ---------------------------------------------------------------------------
M64 = (1 << 64) - 1


def _mix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def _hash3(seed: int, a: int, b: int) -> int:
    return _mix64(seed ^ _mix64(((a * 0x9E3779B97F4A7C15) & M64) ^ ((b + 0x632BE59BD9B4E019) & M64)))


def _a4k(x: int) -> int:
    return (x + 4095) & ~4095


def python_trace(cfg: int, work_items: int, seed: int = DEFAULT_SEED) -> ColumnarTrace:
    W = work_items
    LV = LOCAL[cfg]
    A = 4096
    B = C = D = 0
    if cfg == 2:
        B = A + _a4k(4 * 8 * W)
    elif cfg == 3:
        B = A + _a4k(4 * 4 * W); C = B + 4096; D = C + 16 * W
    elif cfg == 5:
        B = A + _a4k(4 * 2 * W)
    ins = lambda op, w: (op << 32) | w  # noqa: E731
    kinds, pays = [0x20], [0]

    def body(gid, lid, stage):
        if cfg == 1:
            return [(0x01, ins(0, 1)), (0x02, A + 4 * gid)]
        if cfg == 2:
            out = []
            for it in range(8):
                out += [(0x01, ins(0, 1)), (0x02, A + 4 * (8 * gid + it)), (0x01, ins(2, 1))]
            out += [(0x01, ins(3, 4))] * 4 + [(0x01, ins(1, 1)), (0x04, B + 4 * gid)]
            return out
        if cfg == 3:
            out = []
            for it in range(10):
                if it < 4:
                    a = A + 4 * (4 * gid + it)
                elif it < 8:
                    a = B + 4 * ((4 * lid + it - 4) & 1023)
                else:
                    a = C + 4 * (_hash3(seed, gid, it) % (4 * W))
                out += [(0x01, ins(0, 1)), (0x02, a)]
            out += [(0x01, ins(1, 1)), (0x04, D + 4 * gid)]
            for j in range(8):
                out.append((0x01, ins(3 if j & 1 else 2, 1 if j & 2 else 4)))
            return out
        if cfg == 4:
            out = []
            crc = ((gid * 0x9E37) ^ 0xFFFF) & 0xFFFF
            for it in range(32):
                h = _hash3(seed, gid, it)
                bit = crc & 1
                crc = (crc >> 1) ^ (0xA001 if bit else 0)
                out += [(0x01, ins(2, 1)), (0x01, ins(0, 1)), (0x02, A + 4 * (h & 255)),
                        (0x01, ins(3, 1)), (0x08, (10 << 1) | bit),
                        (0x01, ins(3, 1)), (0x08, (12 << 1) | ((h >> 40) & 1)),
                        (0x01, ins(4, 1)), (0x01, ins(3, 1)), (0x08, (14 << 1) | (1 if it < 31 else 0))]
            return out
        # cfg 5: one stage
        out = []
        for q in range(2):
            out += [(0x01, ins(0, 1)), (0x02, A + 4 * ((2 * gid + q + 2 * stage) % (2 * W)))]
        for j in range(21):
            out.append((0x01, ins(3 + j % 3, 1 << (j % 3))))
        out += [(0x01, ins(1, 1)), (0x04, B + 4 * (stage * W + gid)), (0x01, ins(2, 1)), (0x90, 0)]
        return out

    for grp in range(W // LV):
        kinds.append(0x40); pays.append(grp)
        if cfg != 5:
            for lid in range(LV):
                gid = grp * LV + lid
                kinds.append(0x30); pays.append(lid)
                for k, p in body(gid, lid, 0):
                    kinds.append(k); pays.append(p)
                kinds.append(0x10); pays.append(lid)
        else:
            for stage in range(4):
                for lid in range(LV):
                    kinds.append(0x30 if stage == 0 else 0xB0); pays.append(lid)
                    for k, p in body(grp * LV + lid, lid, stage):
                        kinds.append(k); pays.append(p)
            for lid in range(LV):
                kinds += [0xB0, 0x10]; pays += [lid, lid]
        kinds.append(0xC0); pays.append(grp)
    kinds.append(0xA0); pays.append(0)
    kind = np.array(kinds, dtype=np.uint8)
    payload = np.array(pays, dtype=np.uint64)
    mem = (kind & 0x06) != 0
    stats = None
    if mem.any():
        a = payload[mem]
        stats = (int(a.min()), int(a.max()), 0, (1 << 64) - 4)
    return ColumnarTrace(kind, payload, NAMES[cfg], 0, (W, 1, 1), (LV, 1, 1), list(OPCODES[cfg]), [], stats,
                         validated=True)
