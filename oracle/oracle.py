"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the C oracle (aiwc_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module.  It turns the oracle's exact integers
into report fields with the reference's own host-side expressions
(``pkg/src/aiwc/metrics.py:287-386``, ``report.py:25-27``), independently of
the product package.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")


class _Params(ctypes.Structure):
    _fields_ = [("n_opcodes", ctypes.c_uint32), ("history_len", ctypes.c_uint32),
                ("entry_cap", ctypes.c_uint64), ("keep_raw", ctypes.c_uint32), ("pad", ctypes.c_uint32)]


_u64p = ctypes.POINTER(ctypes.c_uint64)


class _Raw(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in ("n_itb", "n_ipt", "n_opc", "n_sites", "table_size", "n_rd", "n_wr")] + [
        (n, _u64p) for n in ("itb", "ipt", "opc", "width_first", "site_ids", "site_exec", "taken_tab", "total_tab",
                             "rd_addr", "rd_cnt", "wr_addr", "wr_cnt")]


class _Dist(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in ("n", "min", "max", "sum", "mid_lo", "mid_hi")]


class _Result(ctypes.Structure):
    _fields_ = [
        ("status", ctypes.c_int), ("entries_at_fail", ctypes.c_uint64),
        ("total_instructions", ctypes.c_uint64), ("work_items", ctypes.c_uint64),
        ("barriers", ctypes.c_uint64), ("opcode_cov", ctypes.c_uint64),
        ("itb", _Dist), ("ipt", _Dist),
        ("n_widths", ctypes.c_uint64),
        ("width_vals", ctypes.POINTER(ctypes.c_uint64)), ("width_counts", ctypes.POINTER(ctypes.c_uint64)),
        ("footprint", ctypes.c_uint64), ("footprint90", ctypes.c_uint64),
        ("unique_reads", ctypes.c_uint64), ("unique_writes", ctypes.c_uint64),
        ("total_reads", ctypes.c_uint64), ("total_writes", ctypes.c_uint64),
        ("gmae", ctypes.c_double), ("lmae", ctypes.c_double * 10),
        ("n_sites", ctypes.c_uint64), ("branch90", ctypes.c_uint64), ("executions", ctypes.c_uint64),
        ("excluded", ctypes.c_uint64), ("observations", ctypes.c_uint64),
        ("yokota", ctypes.c_double), ("linear", ctypes.c_double),
        ("raw", _Raw),
    ]


def accumulator(kind: np.ndarray, payload: np.ndarray, n_opcodes: int, history_len: int = 16) -> dict:
    """The reference accumulator of one (shard of a) trace as numpy arrays:
    ITB / IPT samples, opcode counts, widths with first event index, pooled
    branch pattern tables, site executions, read / write address counts."""
    lib = _load()
    kind = np.ascontiguousarray(kind, dtype=np.uint8)
    payload = np.ascontiguousarray(payload, dtype=np.uint64)
    prm = _Params(n_opcodes, history_len, 0, 1, 0)
    res = _Result()
    if lib.oracle_run(kind.ctypes.data, payload.ctypes.data, kind.shape[0], ctypes.byref(prm), ctypes.byref(res)):
        raise MemoryError("oracle allocation failed")
    try:
        if res.status:
            raise ValueError("malformed columnar trace")
        w = res.raw

        def a(p, n):
            return np.ctypeslib.as_array(p, shape=(n,)).copy() if n else np.zeros(0, np.uint64)

        return {
            "itb": a(w.itb, w.n_itb), "ipt": a(w.ipt, w.n_ipt), "opc": a(w.opc, w.n_opc),
            "widths": [(res.width_vals[i], res.width_counts[i], w.width_first[i]) for i in range(res.n_widths)],
            "sites": dict(zip(a(w.site_ids, w.n_sites).tolist(), a(w.site_exec, w.n_sites).tolist())),
            "taken": a(w.taken_tab, w.table_size), "total": a(w.total_tab, w.table_size),
            "rd": (a(w.rd_addr, w.n_rd), a(w.rd_cnt, w.n_rd)), "wr": (a(w.wr_addr, w.n_wr), a(w.wr_cnt, w.n_wr)),
            "total_instructions": res.total_instructions, "work_items": res.work_items, "barriers": res.barriers,
            "executions": res.executions,
        }
    finally:
        lib.oracle_free(ctypes.byref(res))


SOURCES = ("aiwc_oracle.c", "aiwc_oracle_mt.c")
DEPS = SOURCES + ("aiwc_oracle.h", "oracle_util.h")


def build() -> str:
    """Compile liboracle.so from the C restatement (plain gcc)."""
    newest = max(os.path.getmtime(os.path.join(HERE, f)) for f in DEPS)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        tmp = f"{LIB}.{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", tmp, *[os.path.join(HERE, f) for f in SOURCES],
                               "-lm", "-lpthread"])
        os.replace(tmp, LIB)  # atomic: concurrent test processes never load a half-written library
    return LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        lib = ctypes.CDLL(LIB)
        lib.oracle_run.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                   ctypes.POINTER(_Params), ctypes.POINTER(_Result)]
        lib.oracle_run.restype = ctypes.c_int
        lib.oracle_run_mt.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                      ctypes.POINTER(_Params), ctypes.c_uint32, ctypes.POINTER(_Result)]
        lib.oracle_run_mt.restype = ctypes.c_int
        lib.oracle_free.argtypes = [ctypes.POINTER(_Result)]
        _lib = lib
    return _lib


class OracleTooLarge(Exception):
    def __init__(self, entries, cap):
        self.entries, self.cap = entries, cap
        super().__init__(f"{entries} > {cap}")


def _r12(x: float) -> float:
    return float(f"{x:.12g}")


def _median(d) -> float:
    # summarize_distribution (metrics.py:216-220)
    if d.n % 2:
        return float(d.mid_hi)
    return (d.mid_lo + d.mid_hi) / 2.0


def run(kind: np.ndarray, payload: np.ndarray, *, kernel: str, invocation: int, n_opcodes: int,
        entry_cap: int = 0, history_len: int = 16, threads: int = 1) -> dict:
    """Full report dict (AiwcReport fields, no derived keys) for one columnar trace.
    threads > 1 runs the work-group-sharded driver (aiwc_oracle_mt.c; uncapped only)."""
    lib = _load()
    kind = np.ascontiguousarray(kind, dtype=np.uint8)
    payload = np.ascontiguousarray(payload, dtype=np.uint64)
    prm = _Params(n_opcodes, history_len, entry_cap, 0, 0)
    res = _Result()
    if threads > 1:
        if entry_cap:
            raise ValueError("the multi-threaded oracle runs uncapped")
        rc = lib.oracle_run_mt(kind.ctypes.data, payload.ctypes.data, kind.shape[0], ctypes.byref(prm), threads,
                               ctypes.byref(res))
    else:
        rc = lib.oracle_run(kind.ctypes.data, payload.ctypes.data, kind.shape[0], ctypes.byref(prm),
                            ctypes.byref(res))
    if rc != 0:
        raise MemoryError("oracle allocation failed")
    try:
        if res.status == 1:
            raise OracleTooLarge(res.entries_at_fail, entry_cap)
        if res.status == 2:
            raise ValueError("malformed columnar trace")
        widths = [(res.width_vals[i], res.width_counts[i]) for i in range(res.n_widths)]
    finally:
        lib.oracle_free(ctypes.byref(res))
    total = res.total_instructions
    itb, ipt = res.itb, res.ipt
    # SIMD statistics with the reference's expressions over insertion order (metrics.py:298-306)
    width_total = sum(c for _, c in widths)
    if width_total:
        simd_sum = sum(w * c for w, c in widths)
        simd_mean = simd_sum / width_total
        simd_var = sum(c * (w - simd_mean) ** 2 for w, c in widths) / width_total
        simd_max = max(w for w, _ in widths)
        simd_sd = math.sqrt(simd_var)
    else:
        simd_sum, simd_mean, simd_sd, simd_max = 0, 0.0, 0.0, 0
    ur, uw, tr, tw = res.unique_reads, res.unique_writes, res.total_reads, res.total_writes
    if res.footprint:
        gmae = _r12(res.gmae)
        lmae = [_r12(v) for v in res.lmae]
    else:
        gmae, lmae = 0.0, [0.0] * 10
    executions = res.executions
    if executions == 0:
        yok, lin, warm = 0.0, 0.0, 0.0
    elif res.observations == 0:
        yok, lin, warm = 0.0, 0.0, 1.0
    else:
        yok, lin, warm = _r12(res.yokota), _r12(res.linear), _r12(res.excluded / executions)
    return {
        "kernel": kernel,
        "invocations": [invocation],
        "opcode": res.opcode_cov,
        "total_instruction_count": total,
        "work_items": res.work_items,
        "total_barriers_hit": res.barriers,
        "min_itb": itb.min if itb.n else 0,
        "max_itb": itb.max if itb.n else 0,
        "median_itb": _r12(_median(itb)) if itb.n else 0.0,
        "min_ipt": ipt.min if ipt.n else 0,
        "max_ipt": ipt.max if ipt.n else 0,
        "median_ipt": _r12(_median(ipt)) if ipt.n else 0.0,
        "max_simd_width": simd_max,
        "mean_simd_width": _r12(simd_mean),
        "sd_simd_width": _r12(simd_sd),
        "total_memory_footprint": res.footprint,
        "footprint_90": res.footprint90,
        "unique_reads": ur,
        "unique_writes": uw,
        "unique_rw_ratio": None if uw == 0 else _r12(ur / uw),
        "total_reads": tr,
        "total_writes": tw,
        "reread_ratio": 0.0 if tr == 0 else _r12(ur / tr),
        "rewrite_ratio": 0.0 if tw == 0 else _r12(uw / tw),
        "gmae": gmae,
        "lmae": lmae,
        "total_unique_branch_instructions": res.n_sites,
        "branch_90": res.branch90,
        "yokota_entropy": yok,
        "linear_entropy": lin,
        "mean_itb": _r12(itb.sum / itb.n) if itb.n else 0.0,
        "simd_width_sum": simd_sum,
        "no_branches": executions == 0,
        "warmup_excluded_fraction": warm,
        "no_reads": tr == 0,
        "no_writes": tw == 0,
        "lmae_per_invocation": [{"invocation": invocation, "lmae": list(lmae)}],
    }


def run_trace(tr, **kw) -> dict:
    """`run` on a paper_1805_04207_b200.trace.ColumnarTrace (host arrays)."""
    t = tr.to_numpy()
    return run(t.kind, t.payload, kernel=t.kernel_name, invocation=t.invocation,
               n_opcodes=len(t.opcodes), **kw)


def timed(kind, payload, n_opcodes: int) -> float:
    """Seconds for one oracle pass (cpu_baseline helper)."""
    t0 = time.perf_counter()
    run(kind, payload, kernel="k", invocation=0, n_opcodes=n_opcodes)
    return time.perf_counter() - t0
