"""Golden .aiwctrace line-decoding cases from the REFERENCE (build container only).

    python tests/golden/make_tracefile.py

Feeds hand-written lines (canonical, re-formatted and malformed) to the
reference's decode_event (pkg/src/aiwc/trace.py:177-244) and records the
decoded event (as its canonical encode_event line) or the MalformedEvent text.
"""

from __future__ import annotations

import json
import os
import sys

REF = "/root/reference/pkg"
sys.path[:0] = [os.path.join(REF, "src")]

from aiwc.errors import MalformedEvent  # noqa: E402
from aiwc.trace import decode_event, encode_event  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

LINES = [
    '{"ev":"instr","opcode":"add","width":1}',
    '{"ev":"instr","opcode":"fma","width":16}',
    '{ "ev" : "instr" , "opcode" : "add" , "width" : 4 }',
    '{"width":2,"opcode":"mul","ev":"instr"}',
    '{"ev":"instr","opcode":"a\\"b","width":1}',
    '{"ev":"instr","opcode":"\\u00e9t\\u00e9","width":1}',
    '{"ev":"instr","opcode":"été","width":3}',
    '{"ev":"instr","opcode":"add","width":0}',
    '{"ev":"instr","opcode":"","width":1}',
    '{"ev":"instr","opcode":"add","width":-1}',
    '{"ev":"instr","opcode":"add","width":true}',
    '{"ev":"instr","opcode":"add","width":1.0}',
    '{"ev":"instr","opcode":"add","width":4096.0}',
    '{"ev":"instr","opcode":7,"width":1}',
    '{"ev":"instr","opcode":"add"}',
    '{"ev":"instr","opcode":"add","width":1,"x":0}',
    '{"ev":"mem","op":"load","addr":4096}',
    '{"ev":"mem","op":"atomic_store","addr":18446744073709551615}',
    '{"ev":"mem","op":"store","addr":18446744073709551616}',
    '{"ev":"mem","op":"fetch","addr":8}',
    '{"ev":"mem","op":"load","addr":012}',
    '{"ev":"branch","site":9,"taken":true}',
    '{"ev":"branch","site":9,"taken":1}',
    '{"ev":"branch","site":4294967296,"taken":false}',
    '{"ev":"barrier"}',
    '{"ev":"barrier","x":1}',
    '{"ev":"wi_begin","global":[1,0,0],"local":[1,0,0],"group":[0,0,0]}',
    '{"ev":"wi_end","global":[1,0],"local":[1,0,0],"group":[0,0,0]}',
    '{"ev":"wi_resume","global":[1,0,0],"local":[1,0,0]}',
    '{"ev":"wg_begin","group":[0,0,0]}',
    '{"ev":"wg_end","group":[0,-1,0]}',
    '{"ev":"kernel_begin","kernel":"k","invocation":0,"global_size":[4,1,1],"local_size":[2,1,1]}',
    '{"ev":"kernel_begin","kernel":"k","invocation":0,"global_size":[4,1,1],"local_size":[0,1,1]}',
    '{"ev":"kernel_begin","kernel":"","invocation":0,"global_size":[4,1,1],"local_size":[2,1,1]}',
    '{"ev":"kernel_end"}',
    '{"ev":"kernel_stop"}',
    '{"ev":3}',
    '[1,2,3]',
    '{"ev":"instr","opcode":"add","width":1',
    'not json',
    '{"ev":"instr","opcode":"add","width":1}   ',
    '﻿{"ev":"kernel_end"}',
]


def main():
    out = []
    for i, line in enumerate(LINES, start=1):
        try:
            ev = decode_event(line, i)
            out.append({"line": line, "event": encode_event(ev)})
        except MalformedEvent as exc:
            out.append({"line": line, "error": str(exc)})
    with open(os.path.join(OUT, "tracefile_lines.json"), "w", encoding="utf-8") as fp:
        json.dump(out, fp, indent=1, ensure_ascii=False)
    print(f"{len(out)} lines")


if __name__ == "__main__":
    main()
