"""Golden NDRange-producer vectors from the REFERENCE (build container only).

    python tests/golden/make_sim.py

Runs the reference's parser (pkg/src/aiwc/ir.py), simulator
(pkg/src/aiwc/sim.py) and buffer specs (pkg/src/aiwc/buffers.py) and records:
  * parse outcomes (program repr, or error class / line / message) for valid
    and invalid kernel sources;
  * simulation outcomes for its kernels, its test programs, semantic edge
    cases and seeded random programs (work-item-private and shared memory,
    barriers, loops, vector widths, faults, divergence, step limits): event
    count + sha256 of the canonical lines (and the lines for short traces),
    or the fault's class / message and the events yielded before it;
  * buffer spec outputs.
Writes tests/golden/sim.json.
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys

REF = "/root/reference/pkg"
sys.path[:0] = [os.path.join(REF, "src")]
OUT = os.path.dirname(os.path.abspath(__file__))

from aiwc import buffers, ir, sim  # noqa: E402
from aiwc.trace import encode_event  # noqa: E402

KERNELS = os.path.join(REF, "kernels")


def digest(lines):
    return hashlib.sha256("\n".join(lines).encode()).hexdigest()


def run_case(name, source, gsz, lsz, bufs, step_limit=sim.DEFAULT_STEP_LIMIT, bases=None, invocation=0):
    """bufs: name -> list of ints (already expanded)."""
    prog = ir.parse_kernel(source)
    cfg = sim.NDRangeConfig(tuple(gsz), tuple(lsz), {k: list(v) for k, v in bufs.items()}, bases)
    lines, err = [], None
    try:
        for ev in sim.simulate_events(prog, cfg, step_limit=step_limit, invocation=invocation):
            lines.append(encode_event(ev))
    except Exception as exc:  # noqa: BLE001 -- the fault is the expected outcome
        err = {"type": type(exc).__name__, "message": str(exc), "line": getattr(exc, "line", None)}
    case = {"name": name, "source": source, "global": list(gsz), "local": list(lsz), "buffers": bufs,
            "step_limit": step_limit, "bases": bases, "invocation": invocation,
            "n_events": len(lines), "sha256": digest(lines), "error": err}
    if len(lines) <= 400:
        case["lines"] = lines
    return case


# ---------------------------------------------------------------------------
# random programs
# ---------------------------------------------------------------------------
BIN = ["add", "sub", "mul", "div", "rem", "mod", "and", "or", "xor", "shl", "shr", "min", "max", "eq", "ne",
       "lt", "le", "gt", "ge", "fadd", "fmul"]
UN = ["mov", "not", "neg", "abs"]
TRI = ["mad", "select"]


class Gen:
    def __init__(self, rng, mode, la, lb):
        self.rng, self.mode, self.la, self.lb = rng, mode, la, lb
        self.blocks = []  # (label, [lines])
        self.cur = None
        self.nlab = 0

    def label(self, stem):
        self.nlab += 1
        return f"{stem}{self.nlab}"

    def open(self, label):
        self.cur = (label, [])
        self.blocks.append(self.cur)

    def emit(self, line):
        self.cur[1].append("  " + line)

    def opnd(self):
        r = self.rng.random()
        if r < 0.6:
            return f"r{self.rng.randrange(8)}"
        if r < 0.8:
            return self.rng.choice(["gid0", "lid0", "grp0", "gsz0", "lsz0", "gid1", "lid2"])
        return str(self.rng.choice([0, 1, 2, 3, 5, 7, 63, 64, -1, -7, 1 << 40, -(1 << 63), (1 << 64) - 1]))

    def scalar_stmt(self):
        rng = self.rng
        d = f"r{rng.randrange(8)}"
        k = rng.random()
        if k < 0.55:
            self.emit(f"{rng.choice(BIN)} {d}, {self.opnd()}, {self.opnd()}")
        elif k < 0.7:
            self.emit(f"{rng.choice(UN)} {d}, {self.opnd()}")
        else:
            self.emit(f"{rng.choice(TRI)} {d}, {self.opnd()}, {self.opnd()}, {self.opnd()}")

    def index(self, reg, length, width):
        # an in-bounds index from arbitrary data: rem by a positive modulus is non-negative
        self.emit(f"rem {reg}, {self.opnd()}, {max(length - width + 1, 1)}")

    def mem_stmt(self):
        rng = self.rng
        w = rng.choice([1, 1, 1, 2, 4])
        suf = f".x{w}" if w > 1 else ""
        dst = "r10" if w == 4 else ("r11" if w == 2 else f"r{rng.randrange(8)}")
        if rng.random() < 0.5:  # load
            buf = rng.choice(["a", "b"]) if self.mode == "shared" else "b"
            length = self.la if buf == "a" else self.lb
            self.index("r8", length, w)
            op = rng.choice(["load", "load", "aload"])
            self.emit(f"{op}{suf} {dst}, buf[{buf}][r8]")
        else:  # store
            op = rng.choice(["store", "store", "astore"])
            src = dst if rng.random() < 0.5 else f"r{rng.randrange(8)}"
            if self.mode == "shared":
                self.index("r9", self.la, w)
                self.emit(f"{op}{suf} buf[a][r9], {src}")
            else:  # a private 8-element slot per work-item: a[8*gid0 + k]
                self.emit(f"mul r9, gid0, 8")
                self.emit(f"add r9, r9, {rng.randrange(8 - w + 1)}")
                self.emit(f"{op}{suf} buf[a][r9], {src}")
            if self.mode == "private" and rng.random() < 0.5:  # read back my own store
                self.emit(f"load{suf} {dst}, buf[a][r9]")

    def vec_stmt(self):
        rng = self.rng
        op = rng.choice(["add", "mul", "xor", "max", "select"])
        if op == "select":
            self.emit(f"select.x4 r10, r10, r10, {self.opnd()}")
        else:
            self.emit(f"{op}.x4 r10, r10, {rng.choice(['r10', self.opnd()])}")

    def straight(self, n):
        for _ in range(n):
            k = self.rng.random()
            if k < 0.45:
                self.scalar_stmt()
            elif k < 0.85:
                self.mem_stmt()
            else:
                self.vec_stmt()

    def diamond(self, depth, barrier_inside=False):
        t, e, j = self.label("then"), self.label("else"), self.label("join")
        self.emit(f"and r12, {self.opnd()}, 1")
        self.emit(f"br r12, {t}, {e}")
        self.open(t)
        self.body(depth + 1, 2)
        if barrier_inside:
            self.emit("barrier")
        self.emit(f"jmp {j}")
        self.open(e)
        self.body(depth + 1, 2)
        self.emit(f"jmp {j}")
        self.open(j)

    def loop(self, depth):
        lp, af = self.label("loop"), self.label("after")
        n = self.rng.randint(1, 4)
        c, t = f"r{16 + 2 * depth}", f"r{17 + 2 * depth}"  # one counter per nesting depth
        self.emit(f"mov {c}, 0")
        self.emit(f"jmp {lp}")
        self.open(lp)
        self.body(depth + 1, 2)
        self.emit(f"add {c}, {c}, 1")
        self.emit(f"lt {t}, {c}, {n}")
        self.emit(f"br {t}, {lp}, {af}")
        self.open(af)

    def body(self, depth, parts):
        for _ in range(parts):
            k = self.rng.random()
            if depth < 2 and k < 0.2:
                self.diamond(depth)
            elif depth < 2 and k < 0.35:
                self.loop(depth)
            else:
                self.straight(self.rng.randint(1, 5))

    def program(self, barriers, fault):
        self.open("entry")
        for r in range(8):
            self.emit(f"mov r{r}, {self.rng.choice(['gid0', 'lid0', 'grp0', '3', '-5', 'gid1', 'lid2'])}")
        self.emit("mov.x4 r10, gid0")
        self.emit("mov.x2 r11, lid0")
        self.emit("mov r12, 0")
        self.emit("mov r13, 0")
        self.emit("mov r14, 0")
        for i in range(barriers + 1):
            self.body(0, self.rng.randint(1, 3))
            if i < barriers:
                self.emit("barrier")
        if fault == "oob":
            self.emit(f"load r0, buf[b][{self.opnd()}]")
        elif fault == "width":
            self.emit("add.x4 r10, r10, r11")
        elif fault == "none":
            t, j = self.label("maybe"), self.label("join")
            self.emit("and r12, gid0, 3")
            self.emit(f"br r12, {t}, {j}")
            self.open(t)
            self.emit("mov r15, 1")
            self.emit(f"jmp {j}")
            self.open(j)
            self.emit("add r0, r15, 1")
        elif fault == "divergence":
            self.diamond(0, barrier_inside=True)
        self.emit("ret")
        out = ["kernel rnd(a, b)"]
        for lab, body in self.blocks:
            out.append(f"{lab}:")
            out.extend(body)
        return "\n".join(out) + "\n"


def random_cases(n_cases):
    cases = []
    for seed in range(n_cases):
        rng = random.Random(7000 + seed)
        mode = rng.choice(["private", "private", "shared"])
        shape = rng.choice([((16, 1, 1), (4, 1, 1)), ((32, 1, 1), (8, 1, 1)), ((8, 4, 1), (2, 2, 1)),
                            ((4, 2, 3), (2, 1, 3)), ((64, 1, 1), (64, 1, 1)), ((12, 1, 1), (1, 1, 1))])
        gsz, lsz = shape
        n = gsz[0] * gsz[1] * gsz[2]
        la = 8 * n if mode == "private" else rng.choice([8, 64, 3 * n])
        lb = rng.choice([5, 16, 100])
        fault = rng.choice([None] * 6 + ["oob", "width", "none", "divergence", "steps"])
        g = Gen(rng, mode, la, lb)
        src = g.program(rng.choice([0, 0, 1, 2]), fault)
        bufs = {"a": buffers.make_buffer(rng.choice(["iota", "zeros", "bernoulli:0.5"]), la, seed),
                "b": buffers.make_buffer(rng.choice(["iota", "bernoulli:0.3", "const:-9"]), lb, seed)}
        limit = rng.randint(50, 2000) if fault == "steps" else 300_000
        cases.append(run_case(f"random{seed}_{mode}_{fault}", src, gsz, lsz, bufs, limit))
    return cases


# ---------------------------------------------------------------------------
# fixed cases
# ---------------------------------------------------------------------------
def kernel(name):
    with open(os.path.join(KERNELS, name), encoding="utf-8") as fp:
        return fp.read()


STRAIGHT = ("kernel straight(a)\nentry:\n  mov r0, gid0\n  add r1, r0, 1\n  mul r2, r1, r1\n  load r3, buf[a][r0]\n"
            "  add r3, r3, r2\n  store buf[a][r0], r3\n  ret\n")
LOOP = ("kernel loop()\nentry:\n  mov r0, 0\n  mov r1, 0\n  jmp head\nhead:\n  add r1, r1, gid0\n  add r0, r0, 1\n"
        "  lt r2, r0, 5\n  br r2, head, done\ndone:\n  ret\n")
DATA_BRANCH = ("kernel databranch(flags)\nentry:\n  load r0, buf[flags][gid0]\n  br r0, yes, no\nyes:\n  add r1, r0, 1\n"
               "  jmp out\nno:\n  mov r1, 0\n  jmp out\nout:\n  ret\n")
REJOIN = "kernel k(a)\nentry:\n  store buf[a][lid0], 1\n  barrier\n  load r0, buf[a][lid0]\n  ret\n"
DIVERGE = ("kernel div(x)\nentry:\n  eq r0, lid0, 0\n  br r0, skip, wait\nwait:\n  barrier\n  jmp out\nskip:\n"
           "  jmp out\nout:\n  ret\n")
SEMANTICS = """kernel sem(a)
entry:
  mov r0, -7
  div r1, r0, 2
  rem r2, r0, 2
  mod r3, 7, -2
  div r4, -9223372036854775808, -1
  rem r5, -9223372036854775808, -1
  div r6, 5, 0
  shl r7, 1, 65
  shr r8, -1, 60
  min r9, -1, 1
  max r10, -1, 1
  abs r11, -9223372036854775808
  neg r12, -9223372036854775808
  not r13, 0
  lt r14, -1, 0
  ge r15, -1, 0
  mad r16, 3, 4, 5
  select r17, 0, 11, 22
  fmul r18, 99999999999999999999, 3
  mov.x3 r19, r0
  sub.x3 r19, r19, r1
  store.x3 buf[a][0], r19
  store buf[a][3], r1
  store buf[a][4], r2
  store buf[a][5], r3
  store buf[a][6], r4
  store buf[a][7], r5
  store buf[a][8], r6
  store buf[a][9], r7
  store buf[a][10], r8
  store buf[a][11], r9
  store buf[a][12], r10
  store buf[a][13], r11
  store buf[a][14], r12
  store buf[a][15], r13
  load.x16 r20, buf[a][0]
  add.x16 r20, r20, r14
  store.x16 buf[a][16], r20
  load.x16 r21, buf[a][16]
  xor.x16 r21, r21, r20
  eq r22, r21, 0
  br r22, good, bad
good:
  store buf[a][32], r15
  jmp fin
bad:
  store buf[a][33], r16
  jmp fin
fin:
  store buf[a][34], r17
  store buf[a][35], r18
  ret
"""


def fixed_cases():
    c = []
    c.append(run_case("straight", STRAIGHT, (16, 1, 1), (4, 1, 1), {"a": list(range(16))}))
    c.append(run_case("loop", LOOP, (16, 1, 1), (4, 1, 1), {}))
    c.append(run_case("databranch", DATA_BRANCH, (24, 1, 1), (4, 1, 1), {"flags": [int(i % 3 == 0) for i in range(24)]}))
    c.append(run_case("rejoin", REJOIN, (3, 1, 1), (3, 1, 1), {"a": [0] * 3}))
    c.append(run_case("diverge", DIVERGE, (4, 1, 1), (2, 1, 1), {"x": [0] * 4}))
    c.append(run_case("semantics", SEMANTICS, (2, 1, 1), (1, 1, 1), {"a": [0] * 40}))
    c.append(run_case("semantics_seq", SEMANTICS, (1, 1, 1), (1, 1, 1), {"a": [0] * 40}))
    c.append(run_case("oob", "kernel k(a)\nentry:\n  load r0, buf[a][9]\n  ret\n", (1, 1, 1), (1, 1, 1), {"a": [0] * 4}))
    c.append(run_case("oob_negative", "kernel k(a)\nentry:\n  store buf[a][-1], 3\n  ret\n", (2, 1, 1), (1, 1, 1),
                      {"a": [0] * 4}))
    c.append(run_case("oob_second_item", "kernel k(a)\nentry:\n  load r0, buf[a][gid0]\n  ret\n", (5, 1, 1), (5, 1, 1),
                      {"a": [0] * 3}))
    c.append(run_case("step_limit", "kernel k()\nentry:\n  jmp entry\n", (1, 1, 1), (1, 1, 1), {}, step_limit=1000))
    c.append(run_case("step_limit_many", LOOP, (64, 1, 1), (8, 1, 1), {}, step_limit=500))
    c.append(run_case("step_limit_exact", LOOP, (4, 1, 1), (2, 1, 1), {}, step_limit=4 * 17))
    c.append(run_case("step_limit_zero", LOOP, (1, 1, 1), (1, 1, 1), {}, step_limit=0))
    c.append(run_case("width_mismatch", "kernel k()\nentry:\n  mov.x2 r0, 3\n  mov.x4 r1, 5\n  add.x4 r2, r0, r1\n  ret\n",
                      (1, 1, 1), (1, 1, 1), {}))
    c.append(run_case("store_width_mismatch", "kernel k(a)\nentry:\n  mov.x2 r0, 3\n  store.x4 buf[a][0], r0\n  ret\n",
                      (1, 1, 1), (1, 1, 1), {"a": [0] * 8}))
    c.append(run_case("none_register", "kernel k()\nentry:\n  eq r0, gid0, 1\n  br r0, a, b\na:\n  mov r1, 1\n  jmp b\nb:\n"
                      "  add r2, r1, 1\n  ret\n", (2, 1, 1), (2, 1, 1), {}))
    c.append(run_case("none_index", "kernel k(a)\nentry:\n  eq r0, gid0, 1\n  br r0, x, y\nx:\n  mov r1, 0\n  jmp y\ny:\n"
                      "  load r2, buf[a][r1]\n  ret\n", (2, 1, 1), (1, 1, 1), {"a": [1, 2]}))
    c.append(run_case("bases", STRAIGHT, (4, 1, 1), (2, 1, 1), {"a": [5, 6, 7, 8]}, bases={"a": 1 << 40}))
    c.append(run_case("invocation", STRAIGHT, (4, 1, 1), (2, 1, 1), {"a": [5, 6, 7, 8]}, invocation=7))
    seg = ["  mul r0, lid0, 1", "  load r1, buf[a][r0]", "  add r1, r1, 1", "  store buf[a][r0], r1"]
    seg += ["  add r2, r1, %d" % k for k in range(20)] + ["  barrier"]
    c.append(run_case("stage24", "kernel stage(a)\nentry:\n" + "\n".join(seg * 8) + "\n  ret\n", (4, 1, 1), (4, 1, 1),
                      {"a": [0] * 8}))
    n = 256
    c.append(run_case("sweep4", kernel("sweep4.aiwck"), (n, 1, 1), (64, 1, 1), {"a": list(range(n))}))
    c.append(run_case("sweep64", kernel("sweep64.aiwck"), (n, 1, 1), (64, 1, 1), {"a": list(range(16 * n))}))
    c.append(run_case("sweep64_oob", kernel("sweep64.aiwck"), (n, 1, 1), (64, 1, 1), {"a": list(range(n))}))
    c.append(run_case("bfs_flags", kernel("bfs_flags.aiwck"), (n, 1, 1), (16, 1, 1),
                      {"flags": buffers.make_buffer("bernoulli:0.5:seed=3", n), "out": [0] * n}))
    c.append(run_case("wavefront", kernel("wavefront.aiwck"), (64, 1, 1), (16, 1, 1), {"a": list(range(80))}))
    c.append(run_case("wavefront_2d", kernel("wavefront.aiwck"), (8, 4, 2), (4, 2, 1), {"a": [1] * 80}))
    c.append(run_case("divergent", kernel("divergent.aiwck"), (8, 1, 1), (4, 1, 1), {"x": [0] * 8}))
    c.append(run_case("grid3d", "kernel g(a)\nentry:\n  mad r0, gid1, gsz0, gid0\n  mad r0, gid2, 100, r0\n"
                      "  store buf[a][r0], grp2\n  ret\n", (4, 3, 2), (2, 3, 1), {"a": [0] * 400}))
    # cross-work-item dependence without barriers (sequential mode), and a neighbour read after a barrier
    c.append(run_case("chain", "kernel c(a)\nentry:\n  load r0, buf[a][gid0]\n  add r1, gid0, 1\n  add r0, r0, 1\n"
                      "  store buf[a][r1], r0\n  and r2, r0, 1\n  br r2, x, y\nx:\n  jmp y\ny:\n  ret\n", (32, 1, 1), (8, 1, 1),
                      {"a": [0] * 33}))
    c.append(run_case("neighbour", "kernel nb(a)\nentry:\n  store buf[a][gid0], gid0\n  barrier\n  add r0, gid0, 1\n"
                      "  rem r0, r0, lsz0\n  load r1, buf[a][r0]\n  br r1, x, y\nx:\n  jmp y\ny:\n  ret\n",
                      (16, 1, 1), (4, 1, 1), {"a": [0] * 16}))
    return c


# ---------------------------------------------------------------------------
# parser
# ---------------------------------------------------------------------------
PARSE_SOURCES = [
    STRAIGHT, LOOP, DATA_BRANCH, SEMANTICS, DIVERGE,
    "", "; only a comment\n\n", "kernel k()\n", "kernel k(\nentry:\n  ret\n", "kernel 9k()\nentry:\n  ret\n",
    "kernel k(a, 1b)\nentry:\n  ret\n", "kernel k(a, a)\nentry:\n  ret\n", "kernel k()\n  ret\n",
    "kernel k()\nentry:\n  ret\nentry:\n  ret\n", "kernel k()\nentry:\n  ret\n  ret\n",
    "kernel k()\nentry:\n  add r0, 1, 2\n", "kernel k()\nentry:\n  jmp nowhere\n",
    "kernel k()\nentry:\n  add r0, r1, 2\n  ret\n", "kernel k()\nentry:\n  add.x0 r0, 1, 2\n  ret\n",
    "kernel k()\nentry:\n  ret.x2\n", "kernel k()\nentry:\n  ret r0\n", "kernel k()\nentry:\n  barrier 1\n  ret\n",
    "kernel k()\nentry:\n  jmp a, b\n", "kernel k()\nentry:\n  jmp 9\n", "kernel k()\nentry:\n  br 1, a\n",
    "kernel k()\nentry:\n  br 1, a, 2b\n", "kernel k()\nentry:\n  br q, a, b\n",
    "kernel k(a)\nentry:\n  load r0\n  ret\n", "kernel k(a)\nentry:\n  load 3, buf[a][0]\n  ret\n",
    "kernel k(a)\nentry:\n  load r0, buf[b][0]\n  ret\n", "kernel k(a)\nentry:\n  load r0, a[0]\n  ret\n",
    "kernel k(a)\nentry:\n  store buf[a][0]\n  ret\n", "kernel k(a)\nentry:\n  store buf[a][0], x\n  ret\n",
    "kernel k()\nentry:\n  frobnicate r0, 1\n  ret\n", "kernel k()\nentry:\n  fadd r0, 1\n  ret\n",
    "kernel k()\nentry:\n  add 1, 1, 2\n  ret\n", "kernel k()\nentry:\n  add r4096, 1, 2\n  ret\n",
    "kernel k()\nentry:\n  add r0, 1, , 2\n  ret\n", "kernel k(a)\nentry:\n  load r0, buf[a]][0]\n  ret\n",
    "kernel k(a)\nentry:\n  load r0, buf[a][[0]\n  ret\n", "kernel k()\nentry:\n  add r0, 1,\n  ret\n",
    "kernel k()\nentry:\n  mov r0, 1 ; comment\n  fmov r1, r0\n  ret   ; done\n",
    "  ; lead\nkernel   k  ( a , b )\nentry:\n  aload.x2 r0, buf[b][ gid0 ]\n  astore.x2 buf[a][lid1], r0\n  ret\n",
    "kernel k()\nentry:\n  br 1, x, y\nx:\n  jmp y\ny:\n  ret\nz:\n",
    "kernel k()\nentry:\n  mov r5, 1\n  br r5, a, b\na:\n  add r0, r7, 1\n  ret\nb:\n  mov r7, 2\n  jmp a\n",
    "kernel k()\nentry:\n  mov r0, 99999999999999999999999\n  ret\n", "kernel k()\nentry:\n  mov\tr0, 1\n  ret\n",
    "kernel k()\nentry:\n  select r0, 1, 2\n  ret\n", "kernel k()\nentry:\n  mad.x3 r0, 1, 2, 3\n  ret\n",
]


def parse_outcome(src):
    try:
        p = ir.parse_kernel(src)
    except Exception as exc:  # noqa: BLE001
        return {"error": type(exc).__name__, "line": getattr(exc, "line", None), "message": str(exc)}
    return {"program": repr(p)}


BUFFER_SPECS = ["zeros", "iota", "const:42", "const:0x10", "const:-1", "bernoulli:0.5", "bernoulli:0.5:seed=9",
                "iota:len=5", "zeros:len=0", "bernoulli:0.25:len=20:seed=4", "const:7:len=3", "zeros:1", "iota:2",
                "const", "bernoulli", "bernoulli:1.5", "nope", "iota:len=-1", "file:"]


def buffer_outcome(spec):
    try:
        return {"values": buffers.make_buffer(spec, 12, 5)}
    except Exception as exc:  # noqa: BLE001
        return {"error": type(exc).__name__, "message": str(exc)}


def main():
    cases = fixed_cases() + random_cases(120)
    parse = [{"source": s, **parse_outcome(s)} for s in PARSE_SOURCES]
    specs = [{"spec": s, **buffer_outcome(s)} for s in BUFFER_SPECS]
    with open(os.path.join(OUT, "sim.json"), "w") as fp:
        json.dump({"cases": cases, "parse": parse, "buffers": specs}, fp, separators=(",", ":"))
    errs = {}
    for c in cases:
        k = c["error"]["type"] if c["error"] else "ok"
        errs[k] = errs.get(k, 0) + 1
    print(len(cases), "sim cases", errs, "events", sum(c["n_events"] for c in cases))


if __name__ == "__main__":
    main()
