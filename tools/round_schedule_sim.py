"""Simulation of a round schedule that skips presumably failing IDs, on the
per-round pivot norms of a real run (HSSMF_DUMP_PIVOTS records with norms).

Policy: a node is tried at its first eligible round and, while it fails, again
c x (rounds to go) later, the rounds to go extrapolated from the last two failing
attempts' end-of-ID ratios rho = (pivot norm at the cap) / threshold (log rho is
close to linear in the round). A certification that follows skipped rounds is
checked downwards in chunks until a failing round is met. Counts the IDs and
pivot steps of that schedule against the reference's one ID per node and round.

usage: python tools/round_schedule_sim.py piv.bin [--eps 1e-4 --p 10 --chunk 2]
"""
import argparse
import os
import sys
from collections import defaultdict

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from pivot_replay import read  # noqa: E402


def simulate(by, c, chunk, eps, p):
    ref_steps = steps = ref_att = att = moved = 0
    for key, rs in by.items():
        rs = sorted(rs, key=lambda r: r["round"])
        if not rs[-1]["cert"]:
            continue
        info = {r["round"]: r for r in rs}
        t0, tc = rs[0]["round"], rs[-1]["round"]
        ref_att += len(rs)
        ref_steps += sum(r["rank"] for r in rs)
        t, hist, tlo = t0, [], t0 - 1
        while True:
            if t >= tc:  # certifies (with the certifying attempt's rank); downward checks
                att += 1
                steps += rs[-1]["rank"]
                hi = t
                while hi - 1 > tlo:
                    lo = max(tlo + 1, hi - chunk)
                    for tr in range(hi - 1, lo - 1, -1):
                        att += 1
                        steps += info[min(tr, tc)]["rank"] if tr >= t0 else 0
                    if lo <= tc - 1:
                        break
                    hi = lo
                moved += t > tc
                break
            r = info[t]
            att += 1
            steps += r["rank"]
            tlo = t
            hist.append((t, r["nrm"][-1] / r["nrm"][0] / eps))
            g = 1.0
            if len(hist) >= 2:
                (ta, ra), (tb, rb) = hist[-2], hist[-1]
                if ra > rb > 1:
                    g = np.log(rb) / (np.log(ra / rb) / (tb - ta))
            t += max(1, int(np.floor(c * g)))
    return ref_att, att, ref_steps, steps, moved


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("path")
    ap.add_argument("--eps", type=float, default=1e-4)
    ap.add_argument("--p", type=int, default=10)
    ap.add_argument("--chunk", type=int, default=2)
    a = ap.parse_args()
    recs = [r for r in read(a.path) if r["side"] == 0 and r["nrm"] is not None]
    by = defaultdict(list)
    for r in recs:
        by[(r["inst"], r["m"], r["node"])].append(r)
    print("%5s %10s %10s %12s %12s %8s" % ("c", "ref IDs", "IDs", "ref steps", "steps", "moved"))
    for c in (0.7, 0.8, 0.9, 1.0, 1.1):
        print("%5.1f %10d %10d %12d %12d %8d" % ((c,) + simulate(by, c, a.chunk, a.eps, a.p)))


if __name__ == "__main__":
    main()
