"""TraceEvent iterable -> ColumnarTrace, via the native ``_walker`` extension.

The walker also runs the reference's StreamChecker rules
(``pkg/src/aiwc/trace.py:289-424``) and stops at the first violation.
"""

from __future__ import annotations

import importlib

import numpy as np

from .errors import DeviceError, UnsupportedTrace
from .trace import ColumnarTrace

_mod = None


def _walker():
    global _mod
    if _mod is None:
        try:
            _mod = importlib.import_module("paper_1805_04207_b200._walker")
        except ImportError as exc:  # no silent Python fallback
            raise DeviceError(f"native walker is not built (run __graft_entry__.build()): {exc}") from None
        _mod.init(UnsupportedTrace)
    return _mod


def encode_events(events) -> tuple[ColumnarTrace | None, tuple | None]:
    """Columns for the stream (up to its first violation) and that violation or None."""
    out = _walker().encode(events)
    violation = out["violation"]
    if not out["have_header"]:
        return None, violation
    kind = np.frombuffer(out["kind"], dtype=np.uint8)
    payload = np.frombuffer(out["payload"], dtype=np.uint64)
    tr = ColumnarTrace(kind, payload, out["kernel_name"], out["invocation"], tuple(out["global_size"]),
                       tuple(out["local_size"]), list(out["opcodes"]), [tuple(g) for g in out["extra_groups"]],
                       out["addr_stats"], validated=violation is None,
                       class_counts=tuple(out["counts"]) if violation is None else None)
    return tr, violation
