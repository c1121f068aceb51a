"""Device stream validation of columnar traces (aiwc_validate) against the
collect-all StreamChecker restatement (validate_stream, itself pinned to the
reference by test_validation.py) on the same decoded events: golden traces
mutated at random in the columnar layout (events dropped, duplicated, swapped,
local ids / group keys / kinds changed) must give the same first violation --
index, rule and detail text -- and consume() must raise it as InvalidStream."""

import random

import numpy as np
import pytest

from conftest import golden_cases

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

STRUCT = [0x10, 0x90, 0x30, 0xB0, 0x40, 0xC0, 0x20, 0xA0]


def _traces():
    return [(c["name"], t) for c, t in golden_cases() if t is not None and "error" not in c and t.n_events < 20000]


def _mutate(tr, rng):
    from paper_1805_04207_b200.trace import ColumnarTrace

    k = np.array(tr.kind, dtype=np.uint8).copy()
    p = np.array(tr.payload, dtype=np.uint64).copy()
    for _ in range(rng.randint(1, 3)):
        n = len(k)
        i = rng.randrange(n)
        op = rng.choice(["drop", "dup", "swap", "lid", "key", "kind"])
        if op == "drop":
            k, p = np.delete(k, i), np.delete(p, i)
        elif op == "dup":
            k, p = np.insert(k, i, k[i]), np.insert(p, i, p[i])
        elif op == "swap" and i + 1 < n:
            k[[i, i + 1]] = k[[i + 1, i]]
            p[[i, i + 1]] = p[[i + 1, i]]
        elif op == "lid":
            j = np.flatnonzero((k == 0x30) | (k == 0xB0) | (k == 0x10))
            if j.size:
                q = rng.choice(j.tolist())
                p[q] = np.uint64(rng.randrange(int(np.prod(tr.local_size)) + 2))
        elif op == "key":
            j = np.flatnonzero((k == 0x40) | (k == 0xC0))
            if j.size:
                q = rng.choice(j.tolist())
                grid = int(np.prod([-(-tr.global_size[d] // tr.local_size[d]) for d in range(3)]))
                p[q] = np.uint64(rng.randrange(grid + len(tr.extra_groups)))
        elif op == "kind":  # a representable event of another kind (payload in its range)
            k[i] = rng.choice(STRUCT + [0x01])
            if k[i] == 0x01:
                p[i] = np.uint64(0 << 32 | 1)
            elif k[i] in (0x40, 0xC0):
                grid = int(np.prod([-(-tr.global_size[d] // tr.local_size[d]) for d in range(3)]))
                p[i] = np.uint64(rng.randrange(grid + len(tr.extra_groups)))
            elif k[i] in (0x10, 0x30, 0xB0):
                p[i] = np.uint64(rng.randrange(int(np.prod(tr.local_size))))
            else:
                p[i] = np.uint64(0)
    return ColumnarTrace(k, p, tr.kernel_name, tr.invocation, tr.global_size, tr.local_size, tr.opcodes,
                         tr.extra_groups)


def _expected(tr):
    from paper_1805_04207_b200.trace import validate_stream

    v = validate_stream(tr.iter_events()).violations
    return tuple(v[0]) if v else None


@pytest.mark.parametrize("seed", range(40))
def test_device_first_violation_matches_checker(seed):
    from paper_1805_04207_b200.metrics import validate_columnar

    _run_seed(seed, validate_columnar)


@pytest.mark.parametrize("seed", range(10))
def test_replay_checker_matches_checker(seed):
    """The per-work-group replay kernel (the fallback for huge id spaces), forced."""
    from paper_1805_04207_b200 import _native
    from paper_1805_04207_b200.metrics import trace_info, _device_columns

    ctx = _native.Context(0, flags=_native.OPT_NO_CONSERVATION | _native.OPT_VALIDATE_REPLAY)

    def replay(tr, device):
        import ctypes

        d = _device_columns(tr, device)
        out = _native.Violation()
        i64 = ctypes.c_int64 * 3
        rc = ctx.lib.aiwc_validate(ctx.h, ctypes.c_void_p(d.kind.data_ptr()), ctypes.c_void_p(d.payload.data_ptr()),
                                   ctypes.byref(trace_info(d)), i64(*tr.global_size), i64(*tr.local_size),
                                   ctypes.byref(out), None)
        if rc == _native.OK:
            return None
        assert rc == _native.ERR_INVALID_STREAM
        det = out.detail.decode()
        if out.detail_code in (_native.V_UNFINISHED, _native.V_DIVERGENCE):
            det = None  # text with group tuples is compared through validate_columnar
        return (out.event_index, out.rule.decode(), det)

    def cmp(tr, device):
        got = replay(tr, device)
        return got

    _run_seed(seed, cmp, detail_optional=True)
    ctx.close()


def _run_seed(seed, fn, detail_optional=False):
    rng = random.Random(seed)
    traces = _traces()
    checked = 0
    for _ in range(40):
        name, tr = rng.choice(traces)
        if len(tr.opcodes) == 0:
            continue
        mt = _mutate(tr, rng)
        want = _expected(mt)
        got = fn(mt, 0)
        if detail_optional and got is not None and want is not None and got[2] is None:
            want = want[:2] + (None,)
        assert got == want, (name, seed, got, want)
        checked += 1
    assert checked


def test_valid_golden_traces_pass():
    from paper_1805_04207_b200.metrics import validate_columnar

    for name, tr in _traces():
        assert validate_columnar(tr, 0) is None, name


def test_consume_raises_for_untrusted_columns():
    from paper_1805_04207_b200 import InvalidStream, consume
    from paper_1805_04207_b200.trace import ColumnarTrace

    name, tr = [x for x in _traces() if x[0] == "wavefront_big"][0]
    k = np.array(tr.kind).copy()
    p = np.array(tr.payload).copy()
    i = int(np.flatnonzero(k == 0x10)[3])  # drop a wi_end: the group ends with an unfinished work-item
    bad = ColumnarTrace(np.delete(k, i), np.delete(p, i), tr.kernel_name, tr.invocation, tr.global_size, tr.local_size,
                        tr.opcodes, tr.extra_groups)
    want = _expected(bad)
    with pytest.raises(InvalidStream) as ei:
        consume(bad, max_entries=1 << 40)
    assert (ei.value.event_index, ei.value.rule) == want[:2]
    assert str(ei.value).endswith(f"({want[2]})")


@pytest.mark.parametrize("seed", range(25))
def test_in_pass_check_is_complete(seed):
    """consume()'s in-pass StreamChecker (untrusted columns, checked inside the
    ingest): it never certifies an invalid stream and certifies every valid one."""
    from paper_1805_04207_b200 import AiwcError, UnsupportedTrace
    from paper_1805_04207_b200.metrics import _device_columns, run_engine

    rng = random.Random(5000 + seed)
    traces = _traces()
    certified_valid = 0
    for _ in range(60):
        name, tr = rng.choice(traces)
        if len(tr.opcodes) == 0:
            continue
        mt = _mutate(tr, rng) if rng.random() < 0.8 else tr
        want = _expected(mt)
        try:
            certified = run_engine(_device_columns(mt, 0), 0, check=True).stream_checked
        except (AiwcError, UnsupportedTrace):
            certified = False
        if want is not None:
            assert not certified, (name, seed, want)
        else:
            assert certified, (name, seed)
            certified_valid += 1
    assert certified_valid


def _mutate_bres(tr, rng):
    """One targeted change to the barrier / resume structure."""
    from paper_1805_04207_b200.trace import ColumnarTrace

    k = np.array(tr.kind, dtype=np.uint8).copy()
    p = np.array(tr.payload, dtype=np.uint64).copy()
    bar, res = np.flatnonzero(k == 0x90), np.flatnonzero(k == 0xB0)
    lv = int(np.prod(tr.local_size))
    op = rng.choice(["drop_bar", "drop_res", "dup_bar", "res_lid", "swap_res", "bar_to_end", "end_to_bar"])
    if op == "drop_bar" and bar.size:
        i = rng.choice(bar.tolist()); k, p = np.delete(k, i), np.delete(p, i)
    elif op == "drop_res" and res.size:  # with its segment up to the next close
        i = rng.choice(res.tolist())
        j = i + 1
        while j < len(k) and k[j] not in (0x90, 0x10):
            j += 1
        k, p = np.delete(k, range(i, j + 1)), np.delete(p, range(i, j + 1))
    elif op == "dup_bar" and bar.size:
        i = rng.choice(bar.tolist()); k, p = np.insert(k, i, k[i]), np.insert(p, i, p[i])
    elif op == "res_lid" and res.size:
        i = rng.choice(res.tolist()); p[i] = np.uint64(rng.randrange(lv + 1))
    elif op == "swap_res" and res.size > 1:
        a, b = rng.sample(res.tolist(), 2); p[[a, b]] = p[[b, a]]
    elif op == "bar_to_end" and bar.size:  # the closing barrier becomes the work-item's end
        i = rng.choice(bar.tolist())
        j = i - 1
        while j >= 0 and k[j] not in (0x30, 0xB0):
            j -= 1
        if j >= 0:
            k[i], p[i] = 0x10, p[j]
    elif op == "end_to_bar":
        e = np.flatnonzero(k == 0x10)
        if e.size:
            i = rng.choice(e.tolist()); k[i], p[i] = 0x90, 0
    return ColumnarTrace(k, p, tr.kernel_name, tr.invocation, tr.global_size, tr.local_size, tr.opcodes,
                         tr.extra_groups)


@pytest.mark.parametrize("seed", range(20))
def test_in_pass_check_barrier_rules(seed):
    """Barrier / resume traces: the per-work-item rules inside the pass (begin first,
    end last, one end, equal barrier counts) against the checker restatement."""
    from paper_1805_04207_b200 import AiwcError, UnsupportedTrace
    from paper_1805_04207_b200.metrics import _device_columns, run_engine

    rng = random.Random(9000 + seed)
    traces = [(n, t) for n, t in _traces() if len(t.opcodes) and np.isin(np.asarray(t.kind), [0x90, 0xB0]).any()]
    assert traces
    seen = {True: 0, False: 0}
    for _ in range(40):
        name, tr = rng.choice(traces)
        mt = _mutate_bres(tr, rng) if rng.random() < 0.85 else tr
        want = _expected(mt)
        try:
            certified = run_engine(_device_columns(mt, 0), 0, check=True).stream_checked
        except (AiwcError, UnsupportedTrace):
            certified = False
        assert certified == (want is None), (name, seed, want)
        seen[want is None] += 1
    assert seen[True] and seen[False]
