""".aiwctrace files: the reference's line format and a columnar fast path.

The format and the object-level API are the reference's
(``pkg/src/aiwc/trace.py:100-256``): one compact JSON object per line in a
fixed key order, ``#`` comment lines, ``MalformedEvent(reason, line_no)`` for
lines that do not decode.  ``load_trace`` / ``consume_file`` read a file
straight into the columnar layout instead of building one Python object per
event: canonical lines (what ``write_trace`` emits) are parsed by the native
walker, every other line by ``decode_event`` below -- so escapes, key order,
whitespace and the rejection rules and messages stay the reference's -- and
the stream is validated on the way like ``consume``'s StreamChecker.  Errors
come out in stream order as the reference's lazy ``consume(iter_trace(fp))``
would raise them (cli.py:130-152).

``write_columnar`` / ``read_columnar`` are the binary columnar on-disk form the
survey pairs with the parser: the two columns as they sit in device memory
behind a small JSON header, memory-mapped on load (no parsing; the columns are
untrusted and the engine checks the stream invariants inside its pass).
``consume_file`` recognises them by their magic.
"""

from __future__ import annotations

import json
import os
from typing import IO, Iterable, Iterator

import numpy as np

from .errors import InvalidStream, MalformedEvent, TraceTooLarge
from .trace import (
    Barrier, Branch, ColumnarTrace, Instruction, KernelBegin, KernelEnd, Memory, TraceEvent, Vec3, WorkGroupBegin,
    WorkGroupEnd, WorkItemBegin, WorkItemEnd, WorkItemId, WorkItemResume,
)

MEMORY_OPS = ("load", "store", "atomic_load", "atomic_store")
_ADDR_MAX = (1 << 64) - 1


# ---------------------------------------------------------------------------
# object-level API (trace.py:100-256)
# ---------------------------------------------------------------------------
def encode_event(event: TraceEvent) -> str:
    """The canonical single-line record of one event (trace.py:100-138)."""
    t = type(event).__name__
    if t == "Instruction":
        obj = {"ev": "instr", "opcode": event.opcode, "width": event.width}
    elif t == "Memory":
        obj = {"ev": "mem", "op": event.op, "addr": event.addr}
    elif t == "Branch":
        obj = {"ev": "branch", "site": event.site, "taken": event.taken}
    elif t == "Barrier":
        obj = {"ev": "barrier"}
    elif t in ("WorkItemBegin", "WorkItemResume", "WorkItemEnd"):
        tag = {"WorkItemBegin": "wi_begin", "WorkItemResume": "wi_resume", "WorkItemEnd": "wi_end"}[t]
        wi = event.work_item
        obj = {"ev": tag, "global": list(wi.global_id), "local": list(wi.local_id), "group": list(wi.group_id)}
    elif t == "WorkGroupBegin":
        obj = {"ev": "wg_begin", "group": list(event.group_id)}
    elif t == "WorkGroupEnd":
        obj = {"ev": "wg_end", "group": list(event.group_id)}
    elif t == "KernelBegin":
        obj = {"ev": "kernel_begin", "kernel": event.kernel_name, "invocation": event.invocation,
               "global_size": list(event.global_size), "local_size": list(event.local_size)}
    elif t == "KernelEnd":
        obj = {"ev": "kernel_end"}
    else:
        raise TypeError(f"not a trace event: {event!r}")
    return json.dumps(obj, separators=(",", ":"), ensure_ascii=False)


def _need(obj: dict, keys: tuple, line_no: int | None) -> None:
    got = set(obj)
    want = set(keys) | {"ev"}
    missing = want - got
    if missing:
        raise MalformedEvent(f"missing field {sorted(missing)[0]!r}", line_no)
    extra = got - want
    if extra:
        raise MalformedEvent(f"unknown field {sorted(extra)[0]!r}", line_no)


def _uint(obj: dict, key: str, line_no: int | None, maximum: int | None = None) -> int:
    v = obj[key]
    if isinstance(v, bool) or not isinstance(v, int) or v < 0:
        raise MalformedEvent(f"field {key!r} must be a non-negative integer", line_no)
    if maximum is not None and v > maximum:
        raise MalformedEvent(f"field {key!r} out of range", line_no)
    return v


def _vec3(obj: dict, key: str, line_no: int | None) -> Vec3:
    v = obj[key]
    if not isinstance(v, list) or len(v) != 3 or any(isinstance(x, bool) or not isinstance(x, int) or x < 0 for x in v):
        raise MalformedEvent(f"field {key!r} must be a 3-vector of non-negative integers", line_no)
    return (v[0], v[1], v[2])


def _work_item(obj: dict, line_no: int | None) -> WorkItemId:
    _need(obj, ("global", "local", "group"), line_no)
    return WorkItemId(_vec3(obj, "global", line_no), _vec3(obj, "local", line_no), _vec3(obj, "group", line_no))


def decode_event(line: str, line_no: int | None = None) -> TraceEvent:
    """Decode one trace line (trace.py:177-244), same rules and messages."""
    try:
        obj = json.loads(line)
    except ValueError as exc:
        raise MalformedEvent(f"bad record syntax: {exc}", line_no) from None
    if not isinstance(obj, dict):
        raise MalformedEvent("record is not an object", line_no)
    tag = obj.get("ev")
    if not isinstance(tag, str):
        raise MalformedEvent("missing or non-string 'ev' tag", line_no)
    if tag == "instr":
        _need(obj, ("opcode", "width"), line_no)
        opcode = obj["opcode"]
        if not isinstance(opcode, str) or not opcode:
            raise MalformedEvent("field 'opcode' must be a non-empty string", line_no)
        width = _uint(obj, "width", line_no)
        if width == 0:
            raise MalformedEvent("field 'width' must be >= 1", line_no)
        return Instruction(opcode, width)
    if tag == "mem":
        _need(obj, ("op", "addr"), line_no)
        op = obj["op"]
        if op not in MEMORY_OPS:
            raise MalformedEvent(f"unknown memory op {op!r}", line_no)
        return Memory(op, _uint(obj, "addr", line_no, _ADDR_MAX))
    if tag == "branch":
        _need(obj, ("site", "taken"), line_no)
        taken = obj["taken"]
        if not isinstance(taken, bool):
            raise MalformedEvent("field 'taken' must be a boolean", line_no)
        return Branch(_uint(obj, "site", line_no), taken)
    if tag == "barrier":
        _need(obj, (), line_no)
        return Barrier()
    if tag == "wi_begin":
        return WorkItemBegin(_work_item(obj, line_no))
    if tag == "wi_resume":
        return WorkItemResume(_work_item(obj, line_no))
    if tag == "wi_end":
        return WorkItemEnd(_work_item(obj, line_no))
    if tag == "wg_begin":
        _need(obj, ("group",), line_no)
        return WorkGroupBegin(_vec3(obj, "group", line_no))
    if tag == "wg_end":
        _need(obj, ("group",), line_no)
        return WorkGroupEnd(_vec3(obj, "group", line_no))
    if tag == "kernel_begin":
        _need(obj, ("kernel", "invocation", "global_size", "local_size"), line_no)
        name = obj["kernel"]
        if not isinstance(name, str) or not name:
            raise MalformedEvent("field 'kernel' must be a non-empty string", line_no)
        gsz = _vec3(obj, "global_size", line_no)
        lsz = _vec3(obj, "local_size", line_no)
        if any(x < 1 for x in gsz) or any(x < 1 for x in lsz):
            raise MalformedEvent("launch sizes must be positive", line_no)
        return KernelBegin(name, _uint(obj, "invocation", line_no), gsz, lsz)
    if tag == "kernel_end":
        _need(obj, (), line_no)
        return KernelEnd()
    raise MalformedEvent(f"unknown event tag {tag!r}", line_no)


def write_trace(events: Iterable[TraceEvent], fp: IO[str]) -> None:
    """Write events as `.aiwctrace` lines to a text stream (trace.py:246-250)."""
    for event in events:
        fp.write(encode_event(event))
        fp.write("\n")


def _decode_line(line: str, line_no: int) -> TraceEvent:
    # iter_trace's per-line rules for a non-comment line (trace.py:252-256)
    if not line.strip():
        raise MalformedEvent("blank line", line_no)
    return decode_event(line, line_no)


def iter_trace(fp: IO[str]) -> Iterator[TraceEvent]:
    """Events from a `.aiwctrace` text stream, skipping comments (trace.py:252-256)."""
    for line_no, raw in enumerate(fp, start=1):
        line = raw.rstrip("\n")
        if line.startswith("#"):
            continue
        yield _decode_line(line, line_no)


def read_trace(fp: IO[str]) -> list[TraceEvent]:
    return list(iter_trace(fp))


# ---------------------------------------------------------------------------
# columnar fast path
# ---------------------------------------------------------------------------
def _encode_file(path: str) -> dict:
    from .walker import _walker

    with open(path, "rb") as fp:
        data = fp.read()
    if b"\r" in data:
        # universal-newline files split lines on '\r' too: read them as text, like the reference
        with open(path, "r", encoding="utf-8") as fp:
            out = _walker().encode(_tracked(fp, holder := {}))
        out["last_line"] = holder.get("last", -1)
        return out
    return _walker().encode_lines(data, _decode_line)


def _tracked(fp, holder):
    for line_no, raw in enumerate(fp, start=1):
        line = raw.rstrip("\n")
        if line.startswith("#"):
            continue
        holder["last"] = line_no
        yield _decode_line(line, line_no)


def load_trace(path: str) -> tuple[ColumnarTrace | None, tuple | None, BaseException | None, int]:
    """(columns up to the first problem, first violation or None, pending line
    error or None, last line read) for an `.aiwctrace` file."""
    out = _encode_file(path)
    err = out.get("error")
    tr = None
    if out["have_header"]:
        tr = ColumnarTrace(np.frombuffer(out["kind"], dtype=np.uint8), np.frombuffer(out["payload"], dtype=np.uint64),
                           out["kernel_name"], out["invocation"], tuple(out["global_size"]), tuple(out["local_size"]),
                           list(out["opcodes"]), [tuple(g) for g in out["extra_groups"]], out["addr_stats"],
                           validated=out["violation"] is None and err is None,
                           class_counts=tuple(out["counts"]) if out["violation"] is None and err is None else None)
    return tr, out["violation"], err, out["last_line"]


def fast_trace(path: str, threads: int | None = None) -> ColumnarTrace | None:
    """An all-canonical `.aiwctrace` file parsed on all host threads into untrusted
    columns (the engine checks the stream invariants on the device), or None when
    the file needs the sequential walker (comments, other line forms, '\r', or a
    per-event error the columns cannot carry)."""
    from .walker import _walker

    with open(path, "rb") as fp:
        data = fp.read()
    if b"\r" in data:
        return None
    out = _walker().encode_lines_fast(data, threads or max(1, os.cpu_count() or 1))
    if out is None:
        return None
    return ColumnarTrace(np.frombuffer(out["kind"], dtype=np.uint8), np.frombuffer(out["payload"], dtype=np.uint64),
                         out["kernel_name"], out["invocation"], tuple(out["global_size"]), tuple(out["local_size"]),
                         list(out["opcodes"]), [tuple(g) for g in out["extra_groups"]], out["addr_stats"],
                         validated=False, class_counts=tuple(out["counts"]))


COLUMNAR_MAGIC = b"AIWCCOL1"
_COL_ALIGN = 64


def write_columnar(tr: ColumnarTrace, path: str) -> None:
    """The binary columnar file of one trace: magic, u64 header length, a JSON
    header (launch, opcode dictionary, extra groups, declared statistics), then the
    kind bytes and the little-endian u64 payloads, each 64-byte aligned."""
    t = tr.to_numpy()
    kind = np.ascontiguousarray(t.kind, dtype=np.uint8)
    payload = np.ascontiguousarray(t.payload).view(np.uint64)
    if kind.shape != payload.shape:
        raise ValueError("kind and payload columns differ in length")
    head = json.dumps({"n_events": int(kind.shape[0]), "kernel_name": t.kernel_name, "invocation": int(t.invocation),
                       "global_size": [int(x) for x in t.global_size], "local_size": [int(x) for x in t.local_size],
                       "opcodes": list(t.opcodes), "extra_groups": [[int(x) for x in g] for g in t.extra_groups],
                       "addr_stats": [int(x) for x in t.addr_stats] if t.addr_stats is not None else None,
                       "class_counts": [int(x) for x in t.class_counts] if t.class_counts is not None else None},
                      separators=(",", ":")).encode("utf-8")

    def pad(n: int) -> bytes:
        return b"\0" * ((-n) % _COL_ALIGN)

    with open(path, "wb") as fp:
        pre = COLUMNAR_MAGIC + len(head).to_bytes(8, "little") + head
        fp.write(pre + pad(len(pre)))
        fp.write(kind.tobytes())
        fp.write(pad(kind.nbytes))
        fp.write(payload.astype("<u8", copy=False).tobytes())


def is_columnar_file(path: str) -> bool:
    with open(path, "rb") as fp:
        return fp.read(len(COLUMNAR_MAGIC)) == COLUMNAR_MAGIC


def read_columnar(path: str) -> ColumnarTrace:
    """A binary columnar file as an untrusted ColumnarTrace over memory-mapped columns
    (copy-on-write maps: the file is never written)."""
    size = os.path.getsize(path)
    with open(path, "rb") as fp:
        pre = fp.read(len(COLUMNAR_MAGIC) + 8)
        if len(pre) < len(COLUMNAR_MAGIC) + 8 or pre[:len(COLUMNAR_MAGIC)] != COLUMNAR_MAGIC:
            raise ValueError(f"{path}: not a columnar trace file")
        hlen = int.from_bytes(pre[len(COLUMNAR_MAGIC):], "little")
        if hlen > size:
            raise ValueError(f"{path}: truncated columnar header")
        try:
            h = json.loads(fp.read(hlen).decode("utf-8"))
        except (UnicodeDecodeError, json.JSONDecodeError) as exc:
            raise ValueError(f"{path}: bad columnar header ({exc})") from None
    n = int(h["n_events"])
    k_off = len(pre) + hlen
    k_off += (-k_off) % _COL_ALIGN
    p_off = k_off + n
    p_off += (-p_off) % _COL_ALIGN
    if n < 0 or p_off + 8 * n > size:
        raise ValueError(f"{path}: truncated columnar file ({size} bytes, {n} events declared)")
    kind = np.memmap(path, dtype=np.uint8, mode="c", offset=k_off, shape=(n,)) if n else np.zeros(0, np.uint8)
    payload = np.memmap(path, dtype="<u8", mode="c", offset=p_off, shape=(n,)) if n else np.zeros(0, np.uint64)
    return ColumnarTrace(kind, payload, h["kernel_name"], int(h["invocation"]), tuple(h["global_size"]),
                         tuple(h["local_size"]), list(h["opcodes"]), [tuple(g) for g in h["extra_groups"]],
                         tuple(h["addr_stats"]) if h.get("addr_stats") is not None else None, validated=False,
                         class_counts=tuple(h["class_counts"]) if h.get("class_counts") is not None else None)


def consume_file(path: str, *, max_entries: int | None = None, device: int | None = None):
    """``consume(iter_trace(open(path)))`` without per-event Python objects.

    Raises what the reference's lazy pipeline raises first in stream order:
    TraceTooLarge when the entry cap is crossed before the first problem,
    else the MalformedEvent of a bad line or the InvalidStream of the first
    violation (cli.py:130-152 adds the line number to the latter's message;
    it is returned here as ``exc.line_no``).
    """
    from .metrics import KernelAccumulator, consume, default_entry_cap, run_engine

    cap = default_entry_cap() if max_entries is None else max_entries
    if is_columnar_file(path):  # binary columns: no parsing, checked inside the engine's pass
        return consume(read_columnar(path), max_entries=cap, device=device)
    fast = fast_trace(path)
    if fast is not None:
        # canonical files: parsed in parallel, checked on the device; an invalid stream is
        # re-read by the sequential walker, whose exception carries the line number
        try:
            return consume(fast, max_entries=cap, device=device)
        except InvalidStream:
            pass
    tr, violation, err, last_line = load_trace(path)
    if violation is not None or err is not None:
        if tr is not None and tr.n_events:
            res = run_engine(tr, device)
            if res.entries > cap:
                raise TraceTooLarge(cap + 1, cap)
        if err is not None:
            raise err
        index, rule, detail = violation
        exc = InvalidStream(index, rule, detail)
        exc.line_no = last_line
        raise exc
    res = run_engine(tr, device)
    if res.entries > cap:
        raise TraceTooLarge(cap + 1, cap)
    return KernelAccumulator(kernel_name=tr.kernel_name, invocations=[tr.invocation],
                             launches=[(tr.invocation, tuple(tr.global_size), tuple(tr.local_size))], result=res,
                             opcodes=list(tr.opcodes), trace=tr)
