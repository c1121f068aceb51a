"""NDRange producer: `.aiwck` programs executed on the device into the columnar layout.

Mirrors the reference's in-process trace producer (``pkg/src/aiwc/sim.py``):
``NDRangeConfig`` (launch geometry + named buffers, ``validate`` with the same
ConfigError texts), ``assign_bases`` (disjoint 4096-aligned buffer bases in
parameter order), ``simulate_events`` / ``simulate`` (the TraceEvent stream,
lazily raising the reference's faults after the events that precede them) and,
new, ``simulate_trace`` -- the device-resident ``ColumnarTrace`` that
``consume`` folds without materialising any event object (SURVEY.md §8f
item 4; ``cli.py:106-118``).

Semantics are the reference's (sim.py:1-12, 171-344): work-groups in
lexicographic order, work-items one at a time in lexicographic local order
until a barrier or return, 64-bit lanes, 4-byte elements, width-w accesses
touching ``base + 4*(i + lane)``, every store visible to every later load.  The
engine (``csrc/aiwc_sim.cu``) interprets each work-item on its own thread and
proves that no work-item read another's earlier store; when one did, the
launch re-runs in the exact sequential schedule on the device.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field
from typing import Iterator

import numpy as np

from . import _native
from .errors import (
    BarrierDivergence, ConfigError, DeviceError, OutOfBoundsAccess, SimulationError, StepLimitExceeded,
    UnsupportedTrace,
)
from .ir import KernelProgram, compile_program
from .trace import K_INSTR, ColumnarTrace

ELEMENT_BYTES = 4
BUFFER_ALIGN = 4096
DEFAULT_STEP_LIMIT = 10 ** 8
_MASK = (1 << 64) - 1


@dataclass
class NDRangeConfig:
    """Launch geometry plus named buffer contents (sim.py:88-130)."""

    global_size: tuple
    local_size: tuple
    buffers: dict = field(default_factory=dict)
    bases: dict | None = None

    def validate(self) -> None:
        for what, size in (("global_size", self.global_size), ("local_size", self.local_size)):
            if len(size) != 3 or any(not isinstance(x, int) or x < 1 for x in size):
                raise ConfigError(f"{what} must be three positive integers")
        for d in range(3):
            if self.global_size[d] % self.local_size[d]:
                raise ConfigError(f"local_size[{d}]={self.local_size[d]} does not divide "
                                  f"global_size[{d}]={self.global_size[d]}")
        if self.bases is None:
            return
        spans = []
        for name, values in self.buffers.items():
            if name not in self.bases:
                raise ConfigError(f"no base address for buffer {name!r}")
            lo = self.bases[name]
            hi = lo + ELEMENT_BYTES * len(values)
            if lo < 0 or hi > 1 << 64:
                raise ConfigError(f"buffer {name!r} does not fit in the 64-bit address space")
            spans.append((lo, hi, name))
        spans.sort()
        for (_, end_a, a), (start_b, _, b) in zip(spans, spans[1:]):
            if start_b < end_a:
                raise ConfigError(f"buffers {a!r} and {b!r} overlap")

    @property
    def work_item_count(self) -> int:
        return self.global_size[0] * self.global_size[1] * self.global_size[2]


def assign_bases(params: tuple, buffers: dict) -> dict:
    """Disjoint BUFFER_ALIGN-aligned bases in parameter order (sim.py:132-141)."""
    out, at = {}, BUFFER_ALIGN
    for name in params:
        out[name] = at
        span = ELEMENT_BYTES * max(len(buffers.get(name, ())), 1)
        at += -(-span // BUFFER_ALIGN) * BUFFER_ALIGN
    return out


def _as_u64(values) -> np.ndarray:
    """Buffer contents as u64 lanes: integer / bool arrays keep their bits (fast
    path); anything else is reduced element-wise with ``v & (2^64 - 1)`` like
    the reference (sim.py:186), which also rejects non-integers the same way."""
    arr = values if isinstance(values, np.ndarray) else np.asarray(values)
    if arr.ndim == 1 and arr.dtype.kind in "iub":
        return np.ascontiguousarray(arr.astype(np.int64, copy=False)).view(np.uint64)
    return np.asarray([v & _MASK for v in values], dtype=np.uint64)


def _prepare(program: KernelProgram, cfg: NDRangeConfig):
    cfg.validate()
    missing = [p for p in program.params if p not in cfg.buffers]
    if missing:
        raise ConfigError(f"kernel parameter {missing[0]!r} has no buffer")
    bases = cfg.bases if cfg.bases is not None else assign_bases(program.params, cfg.buffers)
    return bases


_POOL: dict = {}
_POOL_LOCK = threading.Lock()


def _acquire(lib, device: int) -> ctypes.c_void_p:
    """A producer handle for `device`; handles keep their device scratch between
    launches, so repeated launches do not re-allocate."""
    with _POOL_LOCK:
        free = _POOL.setdefault(device, [])
        if free:
            return free.pop()
    h = ctypes.c_void_p(lib.aiwc_sim_create())
    if not h.value:
        raise DeviceError("aiwc_sim_create failed")
    return h


def _release(device: int, h: ctypes.c_void_p) -> None:
    with _POOL_LOCK:
        _POOL.setdefault(device, []).append(h)


class _Launch:
    """One planned launch on the device: counts, layout, first fault."""

    def __init__(self, program: KernelProgram, cfg: NDRangeConfig, bases: dict, step_limit: int, device: int,
                 schedule: str = "auto"):
        import torch

        self.program, self.cfg, self.step_limit = program, cfg, step_limit
        self.cp = compile_program(program)
        self.lib = _native.load_library()
        self.dev = torch.device("cuda", device)
        params = program.params
        bufs = [cfg.buffers[p] for p in params]
        if bufs and all(isinstance(b, torch.Tensor) and b.is_cuda for b in bufs):
            # device-resident buffers: concatenated on the device, no host round trip
            self.mem = torch.cat([b.to(self.dev).reshape(-1).to(torch.int64) for b in bufs] +
                                 [torch.zeros(1, dtype=torch.int64, device=self.dev)])
        else:
            vals = [_as_u64(b if not isinstance(b, torch.Tensor) else b.cpu().numpy()) for b in bufs]
            mem = np.concatenate(vals) if vals else np.zeros(0, np.uint64)
            self.mem = torch.from_numpy(mem.view(np.int64) if mem.size else np.zeros(1, np.int64)).to(self.dev)
        self.code = np.ascontiguousarray(self.cp.code, dtype=np.int32)
        self.imm = np.ascontiguousarray(self.cp.imm, dtype=np.uint64)
        self.bbase = np.array([bases[p] & _MASK for p in params] or [0], dtype=np.uint64)
        self.blen = np.array([len(cfg.buffers[p]) for p in params] or [0], dtype=np.uint64)
        L = _native.SimLaunch()
        L.code = self.code.ctypes.data
        L.imm = self.imm.ctypes.data
        L.buf_base = self.bbase.ctypes.data
        L.buf_len = self.blen.ctypes.data
        L.mem_dev = self.mem.data_ptr()
        L.n_instr, L.n_imm = len(self.code), len(self.imm)
        L.n_regs, L.max_width, L.n_buffers = self.cp.n_regs, self.cp.max_width, len(params)
        if schedule not in _native.SIM_SCHEDULE_FLAGS:
            raise ValueError(f"schedule must be one of {sorted(_native.SIM_SCHEDULE_FLAGS)}")
        L.flags = _native.SIM_SCHEDULE_FLAGS[schedule]
        for d in range(3):
            L.global_size[d], L.local_size[d] = cfg.global_size[d], cfg.local_size[d]
        L.step_limit = max(0, min(int(step_limit), (1 << 62)))
        self.device = device
        self.h = _acquire(self.lib, device)
        self.res = _native.SimResult()
        with torch.cuda.device(self.dev):
            self.stream = torch.cuda.current_stream(self.dev).cuda_stream
            rc = self.lib.aiwc_sim_plan(self.h, ctypes.byref(L), ctypes.byref(self.res), ctypes.c_void_p(self.stream))
        self._check(rc)

    def _check(self, rc: int) -> None:
        if rc == _native.OK:
            return
        msg = (self.lib.aiwc_sim_last_error(self.h) or b"").decode(errors="replace")
        if rc == _native.ERR_UNSUPPORTED:
            raise UnsupportedTrace(msg)
        raise DeviceError(msg or f"aiwc_sim_plan failed with code {rc}")

    @property
    def schedule(self) -> str:
        """The schedule the device used: speculative / group / sequential."""
        return {0: "speculative", 1: "sequential", 2: "group"}[int(self.res.sequential)]

    def emit(self):
        import torch

        n = int(self.res.n_events)
        kind = torch.empty(n + 16, dtype=torch.uint8, device=self.dev)[:n]
        pay = torch.empty(n + 2, dtype=torch.int64, device=self.dev)[:n]
        with torch.cuda.device(self.dev):
            self._check(self.lib.aiwc_sim_emit(self.h, ctypes.c_void_p(kind.data_ptr()), ctypes.c_void_p(pay.data_ptr()),
                                               n, ctypes.c_void_p(self.stream)))
        cfg = self.cfg
        r = self.res
        counts = (int(r.n_instr), int(r.n_reads), int(r.n_writes), int(r.n_branches), int(r.n_groups),
                  int(r.n_barriers > 0))
        return ColumnarTrace(kind, pay, self.program.name, 0, tuple(cfg.global_size), tuple(cfg.local_size),
                             list(self.cp.opcodes), [], None, validated=True,
                             class_counts=counts if r.error == _native.SIM_OK else None)

    # ---- the reference's exceptions (sim.py:205-344) ----
    def _ids(self, w: int):
        lsz = self.cfg.local_size
        ng = tuple(self.cfg.global_size[d] // lsz[d] for d in range(3))
        vol = lsz[0] * lsz[1] * lsz[2]
        g, l = divmod(w, vol)
        grp = (g // (ng[1] * ng[2]), (g // ng[2]) % ng[1], g % ng[2])
        lid = (l // (lsz[1] * lsz[2]), (l // lsz[2]) % lsz[1], l % lsz[2])
        return grp, tuple(grp[d] * lsz[d] + lid[d] for d in range(3))

    def exception(self) -> BaseException | None:
        r = self.res
        e = r.error
        if e == _native.SIM_OK:
            return None
        if e == _native.SIM_OUT_OF_BOUNDS:
            return OutOfBoundsAccess(self.program.params[r.buffer], int(r.index), int(r.line))
        if e == _native.SIM_WIDTH:
            return SimulationError(f"line {r.line}: register r{r.reg} holds {r.lanes} lanes, "
                                   f"but the instruction has width {r.width}", int(r.line))
        if e == _native.SIM_NONE_LEN:
            return TypeError("object of type 'NoneType' has no len()")
        if e == _native.SIM_NONE_INDEX:
            return TypeError("'NoneType' object is not subscriptable")
        if e == _native.SIM_STEP_LIMIT:
            return StepLimitExceeded(self.step_limit)
        if e == _native.SIM_DIVERGENCE:
            grp, culprit = self._ids(int(r.wi))
            _, waiting = self._ids(int(r.wi2))
            line = int(r.line) if r.line >= 0 else None
            at = f"after branching at line {line}" if line is not None else "without branching"
            return BarrierDivergence(f"barrier divergence in group {grp}: work-item {culprit} finished {at} "
                                     f"while work-item {waiting} waits at a barrier", line)
        return UnsupportedTrace("the launch exceeds the device producer's limits "
                                f"(vector width above {_native_max_width()} or more than 2^32 work-items)")

    def close(self) -> None:
        if getattr(self, "h", None) is not None and self.h.value:
            _release(self.device, self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _native_max_width() -> int:
    from .ir import MAX_SIM_WIDTH

    return MAX_SIM_WIDTH


def _device(device: int | None) -> int:
    if device is not None:
        return device
    from .metrics import _default_device

    return _default_device()


def simulate_trace(program: KernelProgram, cfg: NDRangeConfig, *, step_limit: int = DEFAULT_STEP_LIMIT,
                   invocation: int = 0, device: int | None = None, schedule: str = "auto") -> ColumnarTrace:
    """The launch's trace as a device-resident ColumnarTrace (validated, class
    totals declared), or the reference's fault for it.  ``schedule`` forces the
    group or sequential device schedule (default: the cheapest exact one)."""
    bases = _prepare(program, cfg)
    launch = _Launch(program, cfg, bases, step_limit, _device(device), schedule)
    try:
        exc = launch.exception()
        if exc is not None:
            raise exc
        tr = launch.emit()
        tr.invocation = invocation
        return tr
    finally:
        launch.close()


def _events_then_raise(launch: _Launch, invocation: int) -> Iterator:
    try:
        exc = launch.exception()
        tr = launch.emit()
        tr.invocation = invocation
        n = int(launch.res.n_events)
        if exc is not None:
            n = int(launch.res.prefix_events)
            if n == (1 << 64) - 1:
                # speculative step limit: the (limit+1)-th instruction charge raises before its event
                import torch

                is_instr = (tr.kind == K_INSTR).to(torch.int64).cumsum(0)
                n = int(torch.searchsorted(is_instr, max(0, int(launch.step_limit)) + 1).item())
        host = ColumnarTrace(tr.kind[:n].cpu().numpy(), tr.payload[:n].cpu().numpy().view(np.uint64), tr.kernel_name,
                             invocation, tr.global_size, tr.local_size, tr.opcodes)
    finally:
        launch.close()
    yield from host.iter_events()
    if exc is not None:
        raise exc


def simulate_events(program: KernelProgram, cfg: NDRangeConfig, *, step_limit: int = DEFAULT_STEP_LIMIT,
                    invocation: int = 0, device: int | None = None, schedule: str = "auto") -> Iterator:
    """Stream the trace of one kernel invocation (sim.py:347-356): ConfigError
    at call time, faults after the events that precede them."""
    bases = _prepare(program, cfg)
    dev = _device(device)

    def run():
        launch = _Launch(program, cfg, bases, step_limit, dev, schedule)
        yield from _events_then_raise(launch, invocation)

    return run()


def simulate(program: KernelProgram, cfg: NDRangeConfig, *, step_limit: int = DEFAULT_STEP_LIMIT,
             invocation: int = 0, device: int | None = None, schedule: str = "auto") -> list:
    """Materialised variant of simulate_events (sim.py:359-372)."""
    return list(simulate_events(program, cfg, step_limit=step_limit, invocation=invocation, device=device,
                                schedule=schedule))
