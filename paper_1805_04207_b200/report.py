"""The ``aiwc-report/1`` artifact: field schema, rounding, derived metrics, bytes.

The field names and their order ARE the reference's public schema
(``pkg/src/aiwc/report.py:30-77``; key order frozen by
``pkg/tests/test_report.py:84-90``), and every real goes through the same
12-significant-digit rounding (``report.py:25-27``) so JSON output is
byte-comparable with the reference.  Kiviat suite normalisation is out of
scope.
"""

from __future__ import annotations

import csv
import io
import json
from dataclasses import dataclass, field, fields

from .errors import SchemaError

REPORT_SCHEMA = "aiwc-report/1"


def round12(x: float) -> float:
    """Round to 12 significant digits, the serialization precision (ref report.py:25)."""
    return float(f"{x:.12g}")


@dataclass
class AiwcReport:
    kernel: str
    invocations: list[int]
    opcode: int
    total_instruction_count: int
    work_items: int
    total_barriers_hit: int
    min_itb: int
    max_itb: int
    median_itb: float
    min_ipt: int
    max_ipt: int
    median_ipt: float
    max_simd_width: int
    mean_simd_width: float
    sd_simd_width: float
    total_memory_footprint: int
    footprint_90: int
    unique_reads: int
    unique_writes: int
    unique_rw_ratio: float | None
    total_reads: int
    total_writes: int
    reread_ratio: float
    rewrite_ratio: float
    gmae: float
    lmae: list[float]
    total_unique_branch_instructions: int
    branch_90: int
    yokota_entropy: float
    linear_entropy: float
    mean_itb: float
    simd_width_sum: int
    no_branches: bool
    warmup_excluded_fraction: float
    no_reads: bool
    no_writes: bool
    lmae_per_invocation: list[dict] = field(default_factory=list)


@dataclass
class DerivedMetrics:
    granularity: float
    barriers_per_instruction: float
    instructions_per_operand: float
    load_imbalance: int


DERIVED_KEYS = ("granularity", "barriers_per_instruction", "instructions_per_operand", "load_imbalance")


def _inverse(x) -> float:
    return 1.0 / x if x > 0 else 0.0


def derive(report: AiwcReport) -> DerivedMetrics:
    """Inverted parallelism metrics (ref report.py:88-103); degenerate inputs give 0.0."""
    return DerivedMetrics(
        granularity=round12(_inverse(report.work_items)),
        barriers_per_instruction=round12(_inverse(report.mean_itb)),
        instructions_per_operand=round12(_inverse(report.simd_width_sum)),
        load_imbalance=report.max_ipt - report.min_ipt,
    )


def report_to_dict(report: AiwcReport, derived: DerivedMetrics | None = None) -> dict:
    d = derived if derived is not None else derive(report)
    out: dict = {"schema": REPORT_SCHEMA}
    out.update((f.name, getattr(report, f.name)) for f in fields(AiwcReport))
    out.update((k, getattr(d, k)) for k in DERIVED_KEYS)
    return out


def report_from_dict(obj: dict) -> AiwcReport:
    if not isinstance(obj, dict):
        raise SchemaError("report must be a JSON object")
    if obj.get("schema") != REPORT_SCHEMA:
        raise SchemaError(f"expected schema {REPORT_SCHEMA!r}, got {obj.get('schema')!r}")
    missing = [f.name for f in fields(AiwcReport) if f.name not in obj]
    if missing:
        raise SchemaError(f"report is missing field {missing[0]!r}")
    return AiwcReport(**{f.name: obj[f.name] for f in fields(AiwcReport)})


CSV_COLUMNS = (
    ["kernel", "invocations", "opcode", "total_instruction_count",
     "work_items", "total_barriers_hit", "min_itb", "max_itb", "median_itb",
     "min_ipt", "max_ipt", "median_ipt", "max_simd_width", "mean_simd_width", "sd_simd_width",
     "total_memory_footprint", "footprint_90", "unique_reads", "unique_writes", "unique_rw_ratio",
     "total_reads", "total_writes", "reread_ratio", "rewrite_ratio", "gmae"]
    + [f"lmae_skip{n}" for n in range(1, 11)]
    + ["total_unique_branch_instructions", "branch_90", "yokota_entropy", "linear_entropy",
       "mean_itb", "simd_width_sum"]
    + list(DERIVED_KEYS)
    + ["no_branches", "warmup_excluded_fraction", "no_reads", "no_writes"]
)


def _cell(v) -> str:
    if v is None:
        return ""
    if isinstance(v, bool):
        return "true" if v else "false"
    return str(v)


def emit_report(report: AiwcReport, derived: DerivedMetrics | None = None, format: str = "json") -> bytes:
    """JSON (indent 2, fixed key order) or one-row CSV bytes (ref report.py:165-182)."""
    flat = report_to_dict(report, derived)
    if format == "json":
        return (json.dumps(flat, indent=2, ensure_ascii=False) + "\n").encode("utf-8")
    if format == "csv":
        flat["invocations"] = ";".join(str(i) for i in report.invocations)
        for n in range(1, 11):
            flat[f"lmae_skip{n}"] = report.lmae[n - 1]
        buf = io.StringIO()
        w = csv.writer(buf, lineterminator="\n")
        w.writerow(CSV_COLUMNS)
        w.writerow([_cell(flat[c]) for c in CSV_COLUMNS])
        return buf.getvalue().encode("utf-8")
    raise ValueError(f"unknown report format {format!r}")


def load_report(fp) -> AiwcReport:
    try:
        obj = json.load(fp)
    except ValueError as exc:
        raise SchemaError(f"bad report JSON: {exc}") from None
    return report_from_dict(obj)
