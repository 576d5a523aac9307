"""Algorithmic bytes of the extend-add launches of a config (one launch per tree
level and child slot): 24 B per child update entry (read the entry, read and
write its target) + 4 B of position map per child row, matched to ncu's
grid sizes (warp per child column, 8 warps per CTA).

usage: python tools/extend_add_bytes.py c5 [grid ...]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1502_07405_b200 as P  # noqa: E402
from paper_1502_07405_b200.problems import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
op = P.ordered_grid(cfg.kind, cfg.k, cfg.nd_leaf)
t = op.t
nu = (t.upd_ptr[1:] - t.upd_ptr[:-1]).astype(np.int64)
rows = {}
for lv in range(int(t.level.max()), -1, -1):
    ids = np.nonzero(t.level == lv)[0]
    for slot, ch in ((0, t.child0), (1, t.child1)):
        c = ch[ids]
        c = c[c >= 0]
        if c.size == 0:
            continue
        ncols = int(nu[c].sum())
        grid = (ncols * 32 + 255) // 256
        rows[grid] = (lv, slot, len(c), ncols, int((24 * nu[c] ** 2 + 4 * nu[c]).sum()))
want = [int(g) for g in sys.argv[2:]]
for g, (lv, slot, nc, ncols, b) in sorted(rows.items(), key=lambda kv: -kv[1][4]):
    if want and g not in want:
        continue
    print("level %2d slot %d: %6d children, %8d columns, grid %7d, algorithmic %.3f GB" %
          (lv, slot, nc, ncols, g, b / 1e9))
