"""ctypes binding of libaiwc_b200.so (include/aiwc_b200.h).

There is no fallback: if the library is missing or no CUDA device is present,
every entry point raises ``DeviceError``.  Return codes map 1:1 onto the
reference's exceptions (``pkg/src/aiwc/errors.py``).
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import AiwcError, DeviceError, InvalidStream, TraceTooLarge, UnsupportedTrace

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AIWC_LIB") or os.path.join(HERE, "libaiwc_b200.so")  # AIWC_LIB: measurement builds

OK, ERR_INVALID_STREAM, ERR_TOO_LARGE, ERR_INCONSISTENT, ERR_UNSUPPORTED, ERR_ARGUMENT, ERR_CUDA, ERR_NCCL = range(8)
OPT_NO_CONSERVATION = 1  # Python's finalize() runs the reference's conservation checks itself

u8p = ctypes.POINTER(ctypes.c_uint8)
u64p = ctypes.POINTER(ctypes.c_uint64)


class Opts(ctypes.Structure):
    _fields_ = [("history_len", ctypes.c_uint32), ("flags", ctypes.c_uint32),
                ("entry_cap", ctypes.c_uint64), ("dense_budget_bytes", ctypes.c_uint64)]


class TraceInfo(ctypes.Structure):
    _fields_ = [("n_events", ctypes.c_uint64), ("local_volume", ctypes.c_uint32), ("n_opcodes", ctypes.c_uint32),
                ("has_addr_stats", ctypes.c_uint32), ("has_counts", ctypes.c_uint32),
                ("addr_min", ctypes.c_uint64), ("addr_max", ctypes.c_uint64),
                ("addr_and", ctypes.c_uint64), ("addr_or", ctypes.c_uint64),
                ("n_instr", ctypes.c_uint64), ("n_reads", ctypes.c_uint64), ("n_writes", ctypes.c_uint64),
                ("n_branches", ctypes.c_uint64), ("n_groups", ctypes.c_uint64),
                ("any_barrier_or_resume", ctypes.c_uint32), ("check_stream", ctypes.c_uint32),
                ("first_event", ctypes.c_uint64), ("export_state", ctypes.c_uint32), ("reserved2", ctypes.c_uint32)]


class Dist(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in ("n", "min", "max", "sum", "mid_lo", "mid_hi")]


class Result(ctypes.Structure):
    _fields_ = [
        ("n_events", ctypes.c_uint64),
        ("total_instructions", ctypes.c_uint64), ("work_items", ctypes.c_uint64), ("barriers_hit", ctypes.c_uint64),
        ("opcode_coverage", ctypes.c_uint64),
        ("itb", Dist), ("ipt", Dist),
        ("total_reads", ctypes.c_uint64), ("total_writes", ctypes.c_uint64),
        ("unique_reads", ctypes.c_uint64), ("unique_writes", ctypes.c_uint64),
        ("footprint", ctypes.c_uint64), ("footprint_90", ctypes.c_uint64),
        ("gmae", ctypes.c_double), ("lmae", ctypes.c_double * 10),
        ("branch_executions", ctypes.c_uint64), ("branch_observations", ctypes.c_uint64),
        ("branch_excluded", ctypes.c_uint64), ("n_sites", ctypes.c_uint64), ("branch_90", ctypes.c_uint64),
        ("yokota", ctypes.c_double), ("linear", ctypes.c_double),
        ("entries", ctypes.c_uint64),
        ("n_opcodes", ctypes.c_uint32), ("opcode_counts", u64p),
        ("n_widths", ctypes.c_uint32), ("width_values", u64p), ("width_counts", u64p),
        ("n_site_list", ctypes.c_uint32), ("site_ids", u64p), ("site_counts", u64p),
        ("used_dense_table", ctypes.c_uint32), ("kernels_launched", ctypes.c_uint32),
        ("d2h_bytes", ctypes.c_uint64), ("phase_ms", ctypes.c_double * 8), ("binned_accesses", ctypes.c_uint64),
        ("stream_checked", ctypes.c_uint32), ("reserved", ctypes.c_uint32),
    ]


OPT_TIMING = 2
OPT_SHARD = 4
OPT_VALIDATE_REPLAY = 8
PHASES = ("pass1", "ingest", "memory", "branch", "ingest_total", "finalize_total")


class ShardTables(ctypes.Structure):
    _fields_ = [("itb_hist", u64p), ("ipt_hist", u64p), ("n_itb_ovf", ctypes.c_uint64), ("n_ipt_ovf", ctypes.c_uint64),
                ("itb_ovf", u64p), ("ipt_ovf", u64p), ("branch_table_size", ctypes.c_uint32),
                ("branch_table", u64p), ("width_first", u64p), ("addr_stats", ctypes.c_uint64 * 4),
                ("rd_dev", ctypes.c_void_p), ("wr_dev", ctypes.c_void_p)]


class MemoryPart(ctypes.Structure):
    _fields_ = [("unique_reads", ctypes.c_uint64), ("unique_writes", ctypes.c_uint64), ("footprint", ctypes.c_uint64),
                ("level_sum", ctypes.c_double * 11), ("cnt_hist0", u64p), ("n_big", ctypes.c_uint64),
                ("big", u64p), ("kernels_launched", ctypes.c_uint32)]


class ShardStats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in ("addr_min", "addr_max", "addr_and", "addr_or", "n_accesses",
                                             "dense_budget_bytes", "n_branches")]


class State(ctypes.Structure):
    _fields_ = [("exported", ctypes.c_uint32), ("branch_table_size", ctypes.c_uint32), ("n_runs", ctypes.c_uint64),
                ("runs_dev", ctypes.c_void_p), ("base", ctypes.c_uint64), ("low_const", ctypes.c_uint64),
                ("k", ctypes.c_uint32), ("pad", ctypes.c_uint32), ("addr_stats", ctypes.c_uint64 * 4),
                ("itb_hist", u64p), ("ipt_hist", u64p), ("n_itb_ovf", ctypes.c_uint64), ("n_ipt_ovf", ctypes.c_uint64),
                ("itb_ovf", u64p), ("ipt_ovf", u64p), ("branch_table", u64p), ("width_first", u64p)]


class RunsPart(ctypes.Structure):
    _fields_ = [("runs_dev", ctypes.c_void_p), ("n_runs", ctypes.c_uint64), ("base", ctypes.c_uint64),
                ("low_const", ctypes.c_uint64), ("k", ctypes.c_uint32), ("pad", ctypes.c_uint32)]


class Violation(ctypes.Structure):
    _fields_ = [("event_index", ctypes.c_int64), ("rule", ctypes.c_char * 48), ("detail", ctypes.c_char * 256),
                ("detail_code", ctypes.c_uint32), ("metric_kind", ctypes.c_uint32), ("group_key", ctypes.c_uint64),
                ("local_id", ctypes.c_uint64), ("n_counts", ctypes.c_uint32), ("pad", ctypes.c_uint32),
                ("counts", ctypes.c_uint64 * 64)]


V_UNFINISHED, V_DIVERGENCE = 10, 11  # AIWC_V_* codes whose text names a group


class Error(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("event_index", ctypes.c_int64), ("rule", ctypes.c_char * 48),
                ("entries", ctypes.c_uint64), ("cap", ctypes.c_uint64), ("message", ctypes.c_char * 256)]


class SimLaunch(ctypes.Structure):
    _fields_ = [("code", ctypes.c_void_p), ("imm", ctypes.c_void_p), ("buf_base", ctypes.c_void_p),
                ("buf_len", ctypes.c_void_p), ("mem_dev", ctypes.c_void_p), ("n_instr", ctypes.c_uint32),
                ("n_imm", ctypes.c_uint32), ("n_regs", ctypes.c_uint32), ("max_width", ctypes.c_uint32),
                ("n_buffers", ctypes.c_uint32), ("flags", ctypes.c_uint32), ("global_size", ctypes.c_uint64 * 3),
                ("local_size", ctypes.c_uint64 * 3), ("step_limit", ctypes.c_uint64)]


class SimResult(ctypes.Structure):
    _fields_ = [("n_events", ctypes.c_uint64), ("prefix_events", ctypes.c_uint64), ("n_instr", ctypes.c_uint64),
                ("n_reads", ctypes.c_uint64), ("n_writes", ctypes.c_uint64), ("n_branches", ctypes.c_uint64),
                ("n_groups", ctypes.c_uint64), ("n_barriers", ctypes.c_uint64), ("error", ctypes.c_int32),
                ("line", ctypes.c_int32), ("wi", ctypes.c_uint64), ("wi2", ctypes.c_uint64), ("index", ctypes.c_int64),
                ("buffer", ctypes.c_uint32), ("reg", ctypes.c_uint32), ("lanes", ctypes.c_uint32),
                ("width", ctypes.c_uint32), ("sequential", ctypes.c_uint32), ("n_round", ctypes.c_uint32)]


SIM_OK, SIM_OUT_OF_BOUNDS, SIM_WIDTH, SIM_NONE_LEN, SIM_NONE_INDEX, SIM_DIVERGENCE, SIM_STEP_LIMIT, SIM_UNSUPPORTED = range(8)
SIM_FORCE_SEQUENTIAL, SIM_FORCE_GROUP = 1, 2
SIM_SCHEDULE_FLAGS = {"auto": 0, "group": SIM_FORCE_GROUP, "sequential": SIM_FORCE_SEQUENTIAL}

EXPORTS = ("aiwc_abi_version", "aiwc_ctx_create", "aiwc_ctx_destroy", "aiwc_reset", "aiwc_ingest",
           "aiwc_ingest_host", "aiwc_finalize", "aiwc_last_error", "aiwc_synth_size", "aiwc_synth_fill",
           "aiwc_shard_tables_get", "aiwc_partition_addresses", "aiwc_memory_partial", "aiwc_validate",
           "aiwc_sim_create", "aiwc_sim_destroy", "aiwc_sim_last_error", "aiwc_sim_plan", "aiwc_sim_emit",
           "aiwc_partition_runs", "aiwc_memory_partial_runs", "aiwc_shard_prepare", "aiwc_shard_ingest",
           "aiwc_shard_chunks", "aiwc_shard_pack", "aiwc_shard_owned", "aiwc_nccl_unique_id", "aiwc_ctx_set_comm",
           "aiwc_state_export", "aiwc_memory_merge")

_lib = None
_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load libaiwc_b200.so and declare signatures (no device needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise DeviceError(f"native engine {path} is not built (run __graft_entry__.build())")
        lib = ctypes.CDLL(path)
        vp = ctypes.c_void_p
        lib.aiwc_abi_version.restype = ctypes.c_int
        lib.aiwc_ctx_create.argtypes = [ctypes.POINTER(vp), ctypes.c_int, ctypes.POINTER(Opts)]
        lib.aiwc_ctx_destroy.argtypes = [vp]
        lib.aiwc_ctx_destroy.restype = None
        lib.aiwc_reset.argtypes = [vp]
        lib.aiwc_ingest.argtypes = [vp, vp, vp, ctypes.POINTER(TraceInfo), vp]
        lib.aiwc_ingest_host.argtypes = [vp, vp, vp, ctypes.POINTER(TraceInfo), vp]
        lib.aiwc_finalize.argtypes = [vp, ctypes.POINTER(Result), vp]
        lib.aiwc_last_error.argtypes = [vp, ctypes.POINTER(Error)]
        lib.aiwc_synth_size.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.POINTER(TraceInfo)]
        lib.aiwc_synth_size.restype = ctypes.c_uint64
        lib.aiwc_synth_fill.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, vp, vp, ctypes.c_uint64,
                                        ctypes.c_uint64, vp]
        lib.aiwc_shard_tables_get.argtypes = [vp, ctypes.POINTER(ShardTables)]
        lib.aiwc_partition_runs.argtypes = [vp, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32,
                                            ctypes.POINTER(u64p), u64p, vp]
        lib.aiwc_memory_partial_runs.argtypes = [vp, vp, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64,
                                                 ctypes.c_uint64, ctypes.c_uint64, ctypes.POINTER(MemoryPart), vp]
        lib.aiwc_partition_addresses.argtypes = [vp, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32,
                                                 ctypes.POINTER(u64p), ctypes.POINTER(u64p), u64p, vp]
        lib.aiwc_memory_partial.argtypes = [vp, vp, ctypes.c_uint64, vp, ctypes.c_uint64, ctypes.c_uint64,
                                            ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                            ctypes.POINTER(MemoryPart), vp]
        lib.aiwc_shard_prepare.argtypes = [vp, vp, vp, ctypes.POINTER(TraceInfo), ctypes.POINTER(ShardStats), vp]
        lib.aiwc_shard_ingest.argtypes = [vp, ctypes.POINTER(ShardStats), ctypes.POINTER(ctypes.c_uint32), vp]
        lib.aiwc_shard_chunks.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(ctypes.c_uint64)]
        lib.aiwc_shard_pack.argtypes = [vp, vp, ctypes.c_uint32, ctypes.c_uint32, ctypes.POINTER(vp), u64p, vp]
        lib.aiwc_shard_owned.argtypes = [vp, vp, ctypes.c_uint64, vp, ctypes.c_uint32, ctypes.c_uint32,
                                         ctypes.c_uint64, ctypes.POINTER(MemoryPart), vp]
        lib.aiwc_nccl_unique_id.argtypes = [vp]
        lib.aiwc_state_export.argtypes = [vp, ctypes.POINTER(State)]
        lib.aiwc_memory_merge.argtypes = [vp, ctypes.POINTER(RunsPart), ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint64),
                                          ctypes.c_uint64, ctypes.POINTER(MemoryPart), vp]
        lib.aiwc_ctx_set_comm.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int]
        i64x3 = ctypes.c_int64 * 3
        lib.aiwc_validate.argtypes = [vp, vp, vp, ctypes.POINTER(TraceInfo), i64x3, i64x3, ctypes.POINTER(Violation), vp]
        lib.aiwc_sim_create.restype = vp
        lib.aiwc_sim_create.argtypes = []
        lib.aiwc_sim_destroy.argtypes = [vp]
        lib.aiwc_sim_destroy.restype = None
        lib.aiwc_sim_last_error.argtypes = [vp]
        lib.aiwc_sim_last_error.restype = ctypes.c_char_p
        lib.aiwc_sim_plan.argtypes = [vp, ctypes.POINTER(SimLaunch), ctypes.POINTER(SimResult), vp]
        lib.aiwc_sim_emit.argtypes = [vp, vp, vp, ctypes.c_uint64, vp]
        for name in ("aiwc_sim_plan", "aiwc_sim_emit", "aiwc_ctx_create", "aiwc_reset", "aiwc_ingest", "aiwc_ingest_host", "aiwc_finalize",
                     "aiwc_last_error", "aiwc_synth_fill", "aiwc_shard_tables_get", "aiwc_partition_addresses",
                     "aiwc_memory_partial", "aiwc_validate", "aiwc_partition_runs", "aiwc_memory_partial_runs",
                     "aiwc_shard_prepare", "aiwc_shard_ingest", "aiwc_shard_chunks", "aiwc_shard_pack",
                     "aiwc_shard_owned", "aiwc_nccl_unique_id", "aiwc_ctx_set_comm", "aiwc_state_export",
                     "aiwc_memory_merge"):
            getattr(lib, name).restype = ctypes.c_int
        if lib.aiwc_abi_version() != 2:
            raise DeviceError("libaiwc_b200.so ABI version mismatch")
        _lib = lib
        return lib


class Context:
    """One aiwc_ctx (one accumulator at a time) on one CUDA device."""

    def __init__(self, device: int = 0, *, entry_cap: int = 0, history_len: int = 16,
                 flags: int = OPT_NO_CONSERVATION, dense_budget_bytes: int = 0):
        self.lib = load_library()
        self.device = device
        self.entry_cap = entry_cap
        opts = Opts(history_len, flags, entry_cap, dense_budget_bytes)
        h = ctypes.c_void_p()
        rc = self.lib.aiwc_ctx_create(ctypes.byref(h), device, ctypes.byref(opts))
        self.h = h
        if rc != OK:
            msg = self._message() if h.value else f"aiwc_ctx_create failed with code {rc}"
            self.close()
            raise DeviceError(msg)

    def _message(self) -> str:
        e = Error()
        self.lib.aiwc_last_error(self.h, ctypes.byref(e))
        return e.message.decode(errors="replace")

    def check(self, rc: int) -> None:
        if rc == OK:
            return
        e = Error()
        self.lib.aiwc_last_error(self.h, ctypes.byref(e))
        msg = e.message.decode(errors="replace")
        if rc == ERR_TOO_LARGE:
            raise TraceTooLarge(e.entries, e.cap)
        if rc == ERR_INVALID_STREAM:
            raise InvalidStream(e.event_index, e.rule.decode(), msg)
        if rc == ERR_INCONSISTENT:
            raise AiwcError(msg)
        if rc == ERR_UNSUPPORTED:
            raise UnsupportedTrace(msg)
        if rc == ERR_ARGUMENT:
            raise AiwcError(msg)
        raise DeviceError(msg)

    def close(self) -> None:
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.aiwc_ctx_destroy(self.h)
        self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
