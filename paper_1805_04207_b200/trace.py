"""Trace event vocabulary and the canonical columnar layout.

Event classes mirror the reference's ``TraceEvent`` union field-for-field
(``pkg/src/aiwc/trace.py:31-99``) so existing producers keep working; the
native walker also accepts the reference's own classes (dispatch is by class
name and tuple position).

The throughput representation is columnar: one ``kind`` byte
and one ``payload`` u64 per event, resident in HBM.  Kind codes are chosen so
every class the ingest scan needs is a single bit test (SWAR-countable four
events per 32-bit word):

    bit0 instr   bit1 read   bit2 write   bit3 branch
    bit4 work-item boundary (segment open/close)   bit5 open (with bit4)
    bit6 work-group   bit7 variant (atomic mem / resume / barrier / end)

Payload per kind: instr ``opcode_id << 32 | width``; branch
``site << 1 | taken``; mem ``addr``; wi_* ``local linear id``; wg_* ``group
key``; everything else 0.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import NamedTuple, Union

import numpy as np

Vec3 = tuple[int, int, int]

MEMORY_OPS = ("load", "store", "atomic_load", "atomic_store")
READ_OPS = frozenset(("load", "atomic_load"))
WRITE_OPS = frozenset(("store", "atomic_store"))


class KernelBegin(NamedTuple):
    kernel_name: str
    invocation: int
    global_size: Vec3
    local_size: Vec3


class KernelEnd(NamedTuple):
    pass


class WorkGroupBegin(NamedTuple):
    group_id: Vec3


class WorkGroupEnd(NamedTuple):
    group_id: Vec3


class WorkItemId(NamedTuple):
    global_id: Vec3
    local_id: Vec3
    group_id: Vec3


class WorkItemBegin(NamedTuple):
    work_item: WorkItemId


class WorkItemResume(NamedTuple):
    work_item: WorkItemId


class WorkItemEnd(NamedTuple):
    work_item: WorkItemId


class Instruction(NamedTuple):
    opcode: str
    width: int


class Branch(NamedTuple):
    site: int
    taken: bool


class Memory(NamedTuple):
    op: str
    addr: int


class Barrier(NamedTuple):
    pass


TraceEvent = Union[
    KernelBegin, KernelEnd, WorkGroupBegin, WorkGroupEnd, WorkItemBegin,
    WorkItemResume, WorkItemEnd, Instruction, Branch, Memory, Barrier,
]

# --- columnar kind codes (must match include/aiwc_b200.h) -------------------
K_PAD = 0x00
K_INSTR = 0x01
K_LOAD = 0x02
K_ATOMIC_LOAD = 0x82
K_STORE = 0x04
K_ATOMIC_STORE = 0x84
K_BRANCH = 0x08
K_WI_END = 0x10
K_BARRIER = 0x90
K_WI_BEGIN = 0x30
K_WI_RESUME = 0xB0
K_WG_BEGIN = 0x40
K_WG_END = 0xC0
K_KERNEL_BEGIN = 0x20
K_KERNEL_END = 0xA0

MEM_KIND = {"load": K_LOAD, "atomic_load": K_ATOMIC_LOAD, "store": K_STORE, "atomic_store": K_ATOMIC_STORE}
MEM_OP_OF_KIND = {v: k for k, v in MEM_KIND.items()}

# Rule identifiers (ref trace.py:278-286).
RULE_KERNEL_BEGIN = "kernel_begin.first"
RULE_KERNEL_END = "kernel_end.last"
RULE_WG_NESTING = "wg.nesting"
RULE_WI_NESTING = "wi.nesting"
RULE_WI_ID = "wi.id_arithmetic"
RULE_OUTSIDE_SEGMENT = "event.outside_segment"
RULE_RESUME = "wi.resume_without_barrier"
RULE_BARRIER_DIVERGENCE = "barrier.divergence"
RULE_UNFINISHED = "wi.unfinished"

RULES = (
    RULE_KERNEL_BEGIN, RULE_KERNEL_END, RULE_WG_NESTING, RULE_WI_NESTING, RULE_WI_ID,
    RULE_OUTSIDE_SEGMENT, RULE_RESUME, RULE_BARRIER_DIVERGENCE, RULE_UNFINISHED,
)


def group_grid(global_size: Vec3, local_size: Vec3) -> Vec3:
    """Groups per dimension used for linear group keys (ceil division)."""
    return tuple(-(-int(g) // int(l)) for g, l in zip(global_size, local_size))  # type: ignore[return-value]


def local_volume(local_size: Vec3) -> int:
    return int(local_size[0]) * int(local_size[1]) * int(local_size[2])


@dataclass
class ColumnarTrace:
    """One kernel invocation's trace in the canonical columnar layout.

    ``kind``/``payload`` may be numpy arrays (host) or torch tensors (host or
    CUDA).  ``extra_groups`` lists group ids outside the launch grid, whose
    keys start at ``prod(group_grid)``.  ``addr_stats`` = (min, max, and, or)
    over every memory address, when the producer knows it (Parquet-style
    column statistics); the engine verifies it and uses it to size the dense
    address table up front.
    """

    kind: object
    payload: object
    kernel_name: str
    invocation: int
    global_size: Vec3
    local_size: Vec3
    opcodes: list[str] = field(default_factory=list)
    extra_groups: list[Vec3] = field(default_factory=list)
    addr_stats: tuple[int, int, int, int] | None = None
    # True when the producer guarantees a valid stream (native walker, .aiwctrace
    # loader, synthetic generators, merges of such); consume() validates the rest
    validated: bool = False
    # (instructions, reads, writes, branches, work-groups, any barrier/resume) when the
    # producer knows them: the engine then ingests in one pass (verified on the device)
    class_counts: tuple | None = None

    @property
    def n_events(self) -> int:
        return int(self.kind.shape[0])

    @property
    def local_volume(self) -> int:
        return local_volume(self.local_size)

    @property
    def grid(self) -> Vec3:
        return group_grid(self.global_size, self.local_size)

    def group_of_key(self, key: int) -> Vec3:
        g = self.grid
        base = g[0] * g[1] * g[2]
        if key >= base:
            return tuple(self.extra_groups[key - base])  # type: ignore[return-value]
        return (key % g[0], (key // g[0]) % g[1], key // (g[0] * g[1]))

    def local_of_id(self, lid: int) -> Vec3:
        l0, l1, _ = self.local_size
        return (lid % l0, (lid // l0) % l1, lid // (l0 * l1))

    def to_numpy(self) -> "ColumnarTrace":
        def host(a):
            if isinstance(a, np.ndarray):
                return a
            return a.cpu().numpy()
        return ColumnarTrace(host(self.kind), host(self.payload), self.kernel_name, self.invocation,
                             tuple(self.global_size), tuple(self.local_size), list(self.opcodes),
                             list(self.extra_groups), self.addr_stats, self.validated, self.class_counts)

    def iter_events(self):
        """Decode back to TraceEvent objects (debugging / CPU baselines)."""
        kt = self.to_numpy()
        kinds = kt.kind.tolist()
        pays = kt.payload.astype(np.uint64).tolist()
        lsz = tuple(self.local_size)
        cur_group: Vec3 | None = None
        for k, p in zip(kinds, pays):
            if k == K_INSTR:
                yield Instruction(self.opcodes[p >> 32], p & 0xFFFFFFFF)
            elif k in MEM_OP_OF_KIND:
                yield Memory(MEM_OP_OF_KIND[k], p)
            elif k == K_BRANCH:
                yield Branch(p >> 1, bool(p & 1))
            elif k == K_BARRIER:
                yield Barrier()
            elif k in (K_WI_BEGIN, K_WI_RESUME, K_WI_END):
                lid = self.local_of_id(p)
                grp = cur_group if cur_group is not None else (0, 0, 0)
                gid = tuple(grp[d] * lsz[d] + lid[d] for d in range(3))
                wi = WorkItemId(gid, lid, grp)
                yield {K_WI_BEGIN: WorkItemBegin, K_WI_RESUME: WorkItemResume, K_WI_END: WorkItemEnd}[k](wi)
            elif k == K_WG_BEGIN:
                cur_group = self.group_of_key(p)
                yield WorkGroupBegin(cur_group)
            elif k == K_WG_END:
                yield WorkGroupEnd(self.group_of_key(p))
            elif k == K_KERNEL_BEGIN:
                yield KernelBegin(self.kernel_name, self.invocation, tuple(self.global_size), tuple(self.local_size))
            elif k == K_KERNEL_END:
                yield KernelEnd()
            else:
                raise ValueError(f"bad kind code {k:#x}")


# ---------------------------------------------------------------------------
# stream validation (trace.py:263-275, 427-437): every violation, natively
# ---------------------------------------------------------------------------
class Violation(NamedTuple):
    event_index: int
    rule: str
    detail: str


class ValidationReport(NamedTuple):
    violations: list

    @property
    def ok(self) -> bool:
        return not self.violations


def validate_stream(events) -> ValidationReport:
    """Check a stream against every trace invariant; violations are data, not
    failures (the reference's StreamChecker rules, run by the native walker)."""
    from .walker import _walker

    return ValidationReport([Violation(*v) for v in _walker().validate(events)])
