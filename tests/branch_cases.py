"""Random branch-heavy columnar traces for tests/test_gpu_branch_walk.py."""

import numpy as np

K_INSTR, K_BRANCH, K_WI_END, K_WI_BEGIN, K_WG_BEGIN, K_WG_END, K_KB, K_KE = 0x01, 0x08, 0x10, 0x30, 0x40, 0xC0, 0x20, 0xA0

# (seed, sites, groups, work-items per group, branches per work-item, repeat group ids)
CASES = [
    (1, 1, 3, 4, 40, False),
    (2, 3, 40, 8, 30, False),
    (3, 5, 7, 2, 300, True),
    (4, 17, 64, 4, 25, True),
    (5, 64, 20, 8, 60, False),
    (6, 65, 20, 8, 60, False),    # one past the walk's site table: the sort path
    (7, 200, 10, 4, 100, True),   # sort path
    (8, 2, 500, 1, 7, True),      # many tiny streams (most shorter than the history)
]


def make_trace(seed, n_sites, groups, lv, per_wi, repeat):
    """Columnar kind/payload of a 1-D launch of `groups` x `lv` work-items."""
    rng = np.random.default_rng(seed)
    site_ids = rng.choice(1 << 20, size=n_sites, replace=False).astype(np.uint64)
    order = list(range(groups))
    if repeat:  # revisit some group ids later in the trace
        order += [int(g) for g in rng.choice(groups, size=max(1, groups // 3))]
    kind, pay = [K_KB], [0]
    for g in order:
        kind.append(K_WG_BEGIN); pay.append(g)
        # each group uses a random subset of the sites, with a per-site period
        use = site_ids[rng.random(n_sites) < 0.7] if n_sites > 1 else site_ids
        if len(use) == 0:
            use = site_ids[:1]
        period = rng.integers(1, 9, size=len(use))
        for lid in range(lv):
            kind.append(K_WI_BEGIN); pay.append(lid)
            s = rng.integers(0, len(use), size=per_wi)
            noisy = rng.random(per_wi) < 0.2
            for j in range(per_wi):
                k = int(s[j])
                taken = (j % int(period[k]) == 0) ^ bool(noisy[j] and rng.random() < 0.5)
                kind += [K_INSTR, K_BRANCH]
                pay += [(0 << 32) | 1, (int(use[k]) << 1) | int(taken)]
            kind.append(K_WI_END); pay.append(lid)
        kind.append(K_WG_END); pay.append(g)
    kind.append(K_KE); pay.append(0)
    return np.asarray(kind, np.uint8), np.asarray(pay, np.uint64), groups * lv, lv

HS = (1, 5, 11, 16)  # history lengths
