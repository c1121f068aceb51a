"""TEST INFRASTRUCTURE ONLY -- pure-numpy generator of the synthetic BASELINE
configs C1..C5, bit-identical to the device generator
(paper_1805_04207_b200/csrc/aiwc_synth.cu) and to its event-by-event Python
twin (paper_1805_04207_b200/synth.py:python_trace).

It exists so that bench.py's reference arm and cpu_baseline leg build their
input WITHOUT loading the product library (libaiwc_b200.so): the reference arm
must run on the host cores alone.  Nothing here imports the product package.

Geometry (per work-group, constant across groups): wg_begin, LV work-item
bodies (C5: 4 stages of LV segments, then LV resume/end pairs), wg_end; the
whole trace is kernel_begin, the groups in order, kernel_end.  Payloads are
affine in the global work-item id except C3's gathers and C4's hashed bits,
which use the same splitmix64 hash as the device generator.
"""

from __future__ import annotations

import numpy as np

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
PER_WI_BODY = {1: 2, 2: 30, 3: 30, 4: 320, 5: 29}
DEFAULT_SEED = 7

K_INSTR, K_LOAD, K_STORE, K_BRANCH, K_BARRIER = 0x01, 0x02, 0x04, 0x08, 0x90
K_WI_END, K_WI_BEGIN, K_WI_RESUME, K_WG_BEGIN, K_WG_END, K_KB, K_KE = 0x10, 0x30, 0xB0, 0x40, 0xC0, 0x20, 0xA0

_U = np.uint64


def _a4k(x: int) -> int:
    return (x + 4095) & ~4095


def bases(cfg: int, W: int):
    A = 4096
    B = C = D = 0
    if cfg == 2:
        B = A + _a4k(4 * 8 * W)
    elif cfg == 3:
        B = A + _a4k(4 * 4 * W); C = B + 4096; D = C + 16 * W
    elif cfg == 5:
        B = A + _a4k(4 * 2 * W)
    return A, B, C, D


def per_group(cfg: int) -> int:
    lv = LOCAL[cfg]
    if cfg == 5:
        return 2 + lv * 122
    return 2 + lv * (PER_WI_BODY[cfg] + 2)


def n_events(cfg: int, W: int) -> int:
    return 2 + (W // LOCAL[cfg]) * per_group(cfg)


def _mix64(x):
    x = x + _U(0x9E3779B97F4A7C15)
    x = (x ^ (x >> _U(30))) * _U(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> _U(27))) * _U(0x94D049BB133111EB)
    return x ^ (x >> _U(31))


def _hash3(seed: int, a, b: int):
    return _mix64(_U(seed) ^ _mix64((a * _U(0x9E3779B97F4A7C15)) ^ _U((b + 0x632BE59BD9B4E019) & ((1 << 64) - 1))))


def _ins(op: int, w: int) -> int:
    return (op << 32) | w


def _body(cfg, W, seed, gid, lid, stage=0):
    """(kinds[P], payload[G*LV, P]) of one work-item body for every gid."""
    A, B, C, D = bases(cfg, W)
    n = gid.shape[0]
    if cfg == 1:
        k = [K_INSTR, K_LOAD]
        p = np.empty((n, 2), _U)
        p[:, 0] = _ins(0, 1)
        p[:, 1] = _U(A) + _U(4) * gid
        return k, p
    if cfg == 2:
        k, cols = [], []
        for it in range(8):
            k += [K_INSTR, K_LOAD, K_INSTR]
            cols += [_ins(0, 1), _U(A) + _U(4) * (_U(8) * gid + _U(it)), _ins(2, 1)]
        k += [K_INSTR] * 4 + [K_INSTR, K_STORE]
        cols += [_ins(3, 4)] * 4 + [_ins(1, 1), _U(B) + _U(4) * gid]
    elif cfg == 3:
        k, cols = [], []
        for it in range(10):
            if it < 4:
                a = _U(A) + _U(4) * (_U(4) * gid + _U(it))
            elif it < 8:
                a = _U(B) + _U(4) * ((_U(4) * lid + _U(it - 4)) & _U(1023))
            else:
                a = _U(C) + _U(4) * (_hash3(seed, gid, it) % _U(4 * W))
            k += [K_INSTR, K_LOAD]
            cols += [_ins(0, 1), a]
        k += [K_INSTR, K_STORE]
        cols += [_ins(1, 1), _U(D) + _U(4) * gid]
        for j in range(8):
            k.append(K_INSTR)
            cols.append(_ins(3 if j & 1 else 2, 1 if j & 2 else 4))
    elif cfg == 4:
        k, cols = [], []
        crc = ((gid * _U(0x9E37)) ^ _U(0xFFFF)) & _U(0xFFFF)
        for it in range(32):
            h = _hash3(seed, gid, it)
            bit = crc & _U(1)
            crc = (crc >> _U(1)) ^ np.where(bit != 0, _U(0xA001), _U(0))
            k += [K_INSTR, K_INSTR, K_LOAD, K_INSTR, K_BRANCH, K_INSTR, K_BRANCH, K_INSTR, K_INSTR, K_BRANCH]
            cols += [_ins(2, 1), _ins(0, 1), _U(A) + _U(4) * (h & _U(255)), _ins(3, 1), _U(10 << 1) | bit,
                     _ins(3, 1), _U(12 << 1) | ((h >> _U(40)) & _U(1)), _ins(4, 1), _ins(3, 1),
                     (14 << 1) | (1 if it < 31 else 0)]
    else:  # cfg 5, one stage
        k, cols = [], []
        for q in range(2):
            k += [K_INSTR, K_LOAD]
            cols += [_ins(0, 1), _U(A) + _U(4) * ((_U(2) * gid + _U(q + 2 * stage)) % _U(2 * W))]
        for j in range(21):
            k.append(K_INSTR)
            cols.append(_ins(3 + j % 3, 1 << (j % 3)))
        k += [K_INSTR, K_STORE, K_INSTR, K_BARRIER]
        cols += [_ins(1, 1), _U(B) + _U(4) * (_U(stage * W) + gid), _ins(2, 1), 0]
    p = np.empty((n, len(cols)), _U)
    for j, c in enumerate(cols):
        p[:, j] = c
    return k, p


def group_range(cfg: int, W: int, g_lo: int, g_hi: int, seed: int = DEFAULT_SEED):
    """kind u8 / payload u64 of work-groups [g_lo, g_hi) (no kernel begin / end)."""
    lv = LOCAL[cfg]
    G = g_hi - g_lo
    pg = per_group(cfg)
    kind = np.empty((G, pg), np.uint8)
    pay = np.empty((G, pg), _U)
    grp = np.arange(g_lo, g_hi, dtype=_U)
    lid = np.tile(np.arange(lv, dtype=_U), G)
    gid = np.repeat(grp * _U(lv), lv) + lid
    kind[:, 0] = K_WG_BEGIN; pay[:, 0] = grp
    kind[:, -1] = K_WG_END; pay[:, -1] = grp
    with np.errstate(over="ignore"):
        if cfg != 5:
            P = PER_WI_BODY[cfg] + 2
            kb, pb = _body(cfg, W, seed, gid, lid)
            k3 = kind[:, 1:-1].reshape(G, lv, P)
            p3 = pay[:, 1:-1].reshape(G, lv, P)
            k3[:, :, 0] = K_WI_BEGIN; p3[:, :, 0] = lid.reshape(G, lv)
            k3[:, :, -1] = K_WI_END; p3[:, :, -1] = lid.reshape(G, lv)
            k3[:, :, 1:-1] = np.array(kb, np.uint8)
            p3[:, :, 1:-1] = pb.reshape(G, lv, P - 2)
        else:
            ph = lv * 30
            for stage in range(4):
                kb, pb = _body(cfg, W, seed, gid, lid, stage)
                k3 = kind[:, 1 + stage * ph:1 + (stage + 1) * ph].reshape(G, lv, 30)
                p3 = pay[:, 1 + stage * ph:1 + (stage + 1) * ph].reshape(G, lv, 30)
                k3[:, :, 0] = K_WI_BEGIN if stage == 0 else K_WI_RESUME
                p3[:, :, 0] = lid.reshape(G, lv)
                k3[:, :, 1:] = np.array(kb, np.uint8)
                p3[:, :, 1:] = pb.reshape(G, lv, 29)
            k3 = kind[:, 1 + 4 * ph:-1].reshape(G, lv, 2)
            p3 = pay[:, 1 + 4 * ph:-1].reshape(G, lv, 2)
            k3[:, :, 0] = K_WI_RESUME; k3[:, :, 1] = K_WI_END
            p3[:, :, 0] = lid.reshape(G, lv); p3[:, :, 1] = lid.reshape(G, lv)
    return kind.reshape(-1), pay.reshape(-1)


def trace(cfg: int, W: int, seed: int = DEFAULT_SEED, chunk_groups: int = 4096):
    """The whole config-`cfg` trace of W work-items as (kind u8[N], payload u64[N])."""
    lv = LOCAL[cfg]
    if W <= 0 or W % lv:
        raise ValueError(f"work-items {W} not a multiple of local size {lv}")
    groups = W // lv
    n = n_events(cfg, W)
    pg = per_group(cfg)
    kind = np.empty(n, np.uint8)
    pay = np.empty(n, _U)
    kind[0], pay[0] = K_KB, 0
    kind[-1], pay[-1] = K_KE, 0
    for g0 in range(0, groups, chunk_groups):
        g1 = min(groups, g0 + chunk_groups)
        k, p = group_range(cfg, W, g0, g1, seed)
        kind[1 + g0 * pg:1 + g1 * pg] = k
        pay[1 + g0 * pg:1 + g1 * pg] = p
    return kind, pay
