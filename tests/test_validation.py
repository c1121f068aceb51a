"""validate_stream (every violation, the reference's StreamChecker state rules)
against the reference's own reports (tests/golden/validation.json, made by
make_validation.py), and consistency of its first violation with the
consume() walker's InvalidStream."""

import json
import os

import pytest

from conftest import GOLDEN

with open(os.path.join(GOLDEN, "validation.json"), encoding="utf-8") as _fp:
    CASES = json.load(_fp)


@pytest.mark.parametrize("case", CASES, ids=lambda c: c["name"])
def test_validate_stream_matches_reference(case):
    from test_cpu_api import events_from_json

    from paper_1805_04207_b200.trace import validate_stream
    from paper_1805_04207_b200.walker import encode_events

    events = events_from_json(case["events"])
    rep = validate_stream(iter(events))
    assert [list(v) for v in rep.violations] == case["violations"]
    assert rep.ok == (not case["violations"])
    _, first = encode_events(iter(events))
    if case["violations"]:
        assert first is not None and list(first) == case["violations"][0]
    else:
        assert first is None
