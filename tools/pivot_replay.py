"""Pivot-order stability of the Gram-route IDs across adaptive rounds.

Reads the records written by HSSMF_DUMP_PIVOTS=<file> (hss.cu dump_pivots)
and simulates the replay scheme: the ID of round t+1 guesses its next pivots
from round t's order (already chosen pivots skipped), verifies b guesses at a
time and keeps the matching prefix plus the true pivot found at the first
mismatch. Reports, per node size class, the sequential pivot steps against
the number of verify attempts (each attempt advances >= 1 step).

usage: python tools/pivot_replay.py gpurun_out/piv.bin [--block 48]
"""
import argparse
from collections import defaultdict

import numpy as np


def read(path):
    a = np.fromfile(path, dtype=np.int32)
    recs, i = [], 0
    while i + 9 <= a.size:
        inst, m, node, rnd, d, side, mt, rank, cert = (int(v) for v in a[i:i + 9])
        k = min(rank, mt)
        piv = a[i + 9:i + 9 + k].copy()
        i += 9 + k
        nrm = None
        if side & 0x100:  # pivot norms follow (float64)
            nrm = a[i:i + 2 * k].copy().view(np.float64)
            i += 2 * k
            side &= 0xff
        recs.append(dict(inst=inst, m=m, node=node, round=rnd, d=d, side=side, mt=mt,
                         rank=rank, cert=cert, piv=piv, nrm=nrm))
    return recs


def simulate(prev, cur, b):
    """attempts needed for cur's pivot sequence with guesses from prev"""
    chosen = set()
    order = [int(p) for p in prev]
    gi = 0  # pointer into order (skipping chosen)
    j, att, n = 0, 0, len(cur)
    while j < n:
        att += 1
        # b guesses: next entries of order not chosen yet
        g, q = [], gi
        while len(g) < b and q < len(order):
            if order[q] not in chosen:
                g.append(order[q])
            q += 1
        a = 0
        while a < len(g) and j + a < n and g[a] == cur[j + a]:
            a += 1
        step = a + 1 if j + a < n else a
        for s in range(step):
            chosen.add(int(cur[j + s]))
        j += max(step, 1)
        while gi < len(order) and order[gi] in chosen:
            gi += 1
    return att


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("path")
    ap.add_argument("--block", type=int, default=48)
    a = ap.parse_args()
    recs = read(a.path)
    by = defaultdict(list)
    for r in recs:
        by[(r["inst"], r["node"], r["side"])].append(r)
    cls = defaultdict(lambda: [0, 0, 0, 0])  # steps, attempts, first-round steps, ids
    prefix = []
    for key, rs in by.items():
        rs.sort(key=lambda r: r["round"])
        for q, r in enumerate(rs):
            c = "%d+" % (1000 * (r["mt"] // 1000)) if r["mt"] < 4000 else "4000+"
            k = len(r["piv"])
            cls[c][0] += k
            cls[c][3] += 1
            if q == 0:
                cls[c][1] += k
                cls[c][2] += k
                continue
            prev = rs[q - 1]["piv"]
            cls[c][1] += simulate(prev, r["piv"], a.block)
            lp = 0
            while lp < min(len(prev), k) and prev[lp] == r["piv"][lp]:
                lp += 1
            prefix.append((r["mt"], k, lp))
    print("records", len(recs), "node-sides", len(by))
    print("%8s %8s %12s %12s %10s" % ("class", "ids", "steps", "attempts", "ratio"))
    for c in sorted(cls):
        s, t, f, n = cls[c]
        print("%8s %8d %12d %12d %10.2f" % (c, n, s, t, s / max(t, 1)))
    if prefix:
        p = np.array(prefix)
        print("identical leading prefix / rank (median over rounds > 1): %.3f"
              % np.median(p[:, 2] / np.maximum(p[:, 1], 1)))


if __name__ == "__main__":
    main()
