"""The exported entropy helpers against the reference's own values
(tests/golden/entropy.json, made by make_entropy.py): 1e-9 relative for reals,
exact for counts, same exception class and message."""

import json
import math
import os

import pytest

from conftest import GOLDEN

with open(os.path.join(GOLDEN, "entropy.json"), encoding="utf-8") as _fp:
    GOLD = json.load(_fp)


def _check(fn, args, want):
    import paper_1805_04207_b200.errors as errors

    if "error" in want:
        cls = getattr(errors, want["error"], None) or ValueError
        with pytest.raises(cls) as ei:
            fn(*args)
        assert str(ei.value) == want["message"]
        return
    got = fn(*args)
    exp = want["value"]
    if isinstance(exp, list):
        assert len(got) == len(exp)
        for g, e in zip(got, exp):
            assert (g == e) if isinstance(e, int) else math.isclose(g, e, rel_tol=1e-9, abs_tol=1e-15)
    elif isinstance(exp, int):
        assert got == exp
    else:
        assert math.isclose(got, exp, rel_tol=1e-9, abs_tol=1e-15) and math.copysign(1, got) == math.copysign(1, exp)


@pytest.mark.parametrize("i", range(len(GOLD["hist"])))
def test_histogram_helpers(i):
    from paper_1805_04207_b200 import entropy as E

    row = GOLD["hist"][i]
    h = {k: v for k, v in row["items"]}
    _check(E.shannon_entropy, (h,), row["shannon"])
    _check(E.coverage_count, (h,), row["coverage"])
    _check(E.coverage_count, (h, 0.5), row["coverage_half"])
    for s, want in zip((1, 3, 10), row["local"]):
        _check(E.local_entropy, (h, s), want)
    _check(E.local_entropy, (h, 11), row["local_bad"])


@pytest.mark.parametrize("i", range(len(GOLD["branch"])))
def test_branch_entropy(i):
    from paper_1805_04207_b200 import entropy as E

    row = GOLD["branch"][i]
    _check(E.branch_entropy, ({k: v for k, v in row["records"]}, row["history_len"]), row["result"])
