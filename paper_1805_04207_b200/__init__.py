"""B200-native AIWC metric path (arXiv:1805.04207).

Drop-in for the reference package's trace -> feature-vector path: the same
TraceEvent vocabulary, ``consume`` / ``finalize`` / ``merge_accumulators``,
``AiwcReport`` schema and exceptions, computed by hand-written sm_100a CUDA
kernels in ``libaiwc_b200.so`` behind a C ABI (include/aiwc_b200.h).  The
reference's in-process trace producer (the `.aiwck` NDRange simulator) runs on
the device too: ``simulate_trace`` hands ``consume`` a device-resident trace.
"""

from .errors import (
    AiwcError, DeviceError, EmptyHistogram, EmptySample, IncompatibleReports, InvalidSkip, InvalidStream,
    MalformedEvent, NoBranches, SchemaError, TraceTooLarge, UnsupportedTrace,
    BarrierDivergence, ConfigError, MissingTerminator, OutOfBoundsAccess, ParseError, SimulationError,
    StepLimitExceeded, UndefinedLabel, UseBeforeDef,
)
from .metrics import (
    DistStats, KernelAccumulator, consume, default_entry_cap, finalize, lmae_profile, merge_accumulators,
    summarize_distribution,
)
from .report import (
    AiwcReport, DerivedMetrics, derive, emit_report, load_report, report_from_dict, report_to_dict, round12,
)
from .trace import (
    Barrier, Branch, ColumnarTrace, Instruction, KernelBegin, KernelEnd, Memory, TraceEvent, ValidationReport,
    Violation, WorkGroupBegin, WorkGroupEnd, WorkItemBegin, WorkItemEnd, WorkItemId, WorkItemResume, validate_stream,
)
from .entropy import BranchStats, branch_entropy, coverage_count, local_entropy, shannon_entropy
from .tracefile import (
    consume_file, decode_event, encode_event, iter_trace, load_trace, read_columnar, read_trace, write_columnar,
    write_trace,
)
from .ir import KernelProgram, parse_kernel
from .sim import NDRangeConfig, assign_bases, simulate, simulate_events, simulate_trace

__version__ = "0.1.0"

__all__ = [
    "BranchStats", "ValidationReport", "Violation", "branch_entropy", "consume_file", "coverage_count",
    "decode_event", "encode_event", "iter_trace", "load_trace", "local_entropy", "read_trace", "shannon_entropy",
    "validate_stream", "write_trace", "read_columnar", "write_columnar",
    "AiwcError", "AiwcReport", "Barrier", "Branch", "ColumnarTrace", "DerivedMetrics", "DeviceError", "DistStats",
    "EmptyHistogram", "EmptySample", "IncompatibleReports", "Instruction", "InvalidSkip", "InvalidStream",
    "KernelAccumulator", "KernelBegin", "KernelEnd", "MalformedEvent", "Memory", "NoBranches", "SchemaError",
    "TraceEvent", "TraceTooLarge", "UnsupportedTrace", "WorkGroupBegin", "WorkGroupEnd", "WorkItemBegin",
    "WorkItemEnd", "WorkItemId", "WorkItemResume", "consume", "default_entry_cap", "derive", "emit_report",
    "finalize", "lmae_profile", "load_report", "merge_accumulators", "report_from_dict", "report_to_dict",
    "round12", "summarize_distribution",
    "BarrierDivergence", "ConfigError", "KernelProgram", "MissingTerminator", "NDRangeConfig", "OutOfBoundsAccess",
    "ParseError", "SimulationError", "StepLimitExceeded", "UndefinedLabel", "UseBeforeDef", "assign_bases",
    "parse_kernel", "simulate", "simulate_events", "simulate_trace",
]
