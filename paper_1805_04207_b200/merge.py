"""Column concatenation for ``merge_accumulators`` (ref metrics.py:235-270).

Merging invocation accumulators is defined by the reference as "equivalent to
having consumed one concatenated stream", with each part's branch streams kept
separate.  Concatenating the parts' columns reproduces that exactly once
(a) opcode ids are re-keyed into one dictionary and (b) every part's group
keys are shifted into a disjoint range, so no (site, group) history can run
across a part boundary.  Columns stay where they are (numpy on the host, torch
on the GPU); only the instr / wg payloads are rewritten.
"""

from __future__ import annotations

import numpy as np

from .trace import K_INSTR, K_WG_BEGIN, K_WG_END, ColumnarTrace


def _xp(a):
    if type(a).__module__.startswith("torch"):
        import torch

        return torch
    return np


def concat_traces(parts: list[ColumnarTrace]) -> ColumnarTrace:
    xp = _xp(parts[0].kind)
    opcodes: dict[str, int] = {}
    kinds, pays = [], []
    key_base = 0
    lv = max(p.local_volume for p in parts)
    stats = [p.addr_stats for p in parts]
    for p in parts:
        remap = [opcodes.setdefault(o, len(opcodes)) for o in p.opcodes]
        k, pay = p.kind, p.payload
        if xp is np:
            k = np.asarray(k, dtype=np.uint8)
            pay = np.asarray(pay).view(np.uint64).copy()
            is_i = k == K_INSTR
            if remap and len(remap) and is_i.any():
                table = np.asarray(remap, dtype=np.uint64)
                op = (pay[is_i] >> np.uint64(32)).astype(np.int64)
                pay[is_i] = (table[op] << np.uint64(32)) | (pay[is_i] & np.uint64(0xFFFFFFFF))
            is_g = (k == K_WG_BEGIN) | (k == K_WG_END)
            pay[is_g] += np.uint64(key_base)
        else:
            import torch

            pay = pay.clone().view(torch.int64)
            is_i = k == K_INSTR
            if remap:
                table = torch.tensor(remap, dtype=torch.int64, device=pay.device)
                op = pay[is_i] >> 32
                pay[is_i] = (table[op] << 32) | (pay[is_i] & 0xFFFFFFFF)
            is_g = (k == K_WG_BEGIN) | (k == K_WG_END)
            pay[is_g] += key_base
        g = p.grid
        key_base += g[0] * g[1] * g[2] + len(p.extra_groups)
        kinds.append(k)
        pays.append(pay)
    if key_base >= 1 << 31:
        raise ValueError("merged trace has more than 2^31 group keys")
    if xp is np:
        kind = np.concatenate(kinds)
        payload = np.concatenate(pays)
    else:
        import torch

        kind = torch.cat(kinds)
        payload = torch.cat(pays)
    addr_stats = None
    if all(s is not None for s in stats):
        addr_stats = (min(s[0] for s in stats), max(s[1] for s in stats),
                      np.bitwise_and.reduce([np.uint64(s[2]) for s in stats]).item(),
                      np.bitwise_or.reduce([np.uint64(s[3]) for s in stats]).item())
    first = parts[0]
    # group keys are already disjoint; a 1-D grid with key_base groups decodes them
    return ColumnarTrace(kind, payload, first.kernel_name, first.invocation, (key_base * lv, 1, 1), (lv, 1, 1),
                         [o for o, _ in sorted(opcodes.items(), key=lambda kv: kv[1])], [], addr_stats,
                         validated=all(p.validated for p in parts),
                         class_counts=(tuple(sum(p.class_counts[i] for p in parts) for i in range(5)) +
                                       (int(any(p.class_counts[5] for p in parts)),)
                                       if all(p.class_counts is not None for p in parts) else None))
