"""Per-node adaptive-round history of the Gram-route IDs (HSSMF_DUMP_PIVOTS
records): first attempted round, certifying round, pivot steps spent in
failing attempts against the certifying one; with pivot norms in the dump, how
well a failing attempt's decay predicts the certifying round.

usage: python tools/pivot_rounds.py gpurun_out/piv.bin [--d0 128 --dd 128 --p 10]
"""
import argparse
import os
import sys
from collections import defaultdict

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from pivot_replay import read  # noqa: E402


def predict_rank(nrm, d, tol_rel):
    """rank at which the pivot norms of a failing attempt (d sample columns)
    would reach tol_rel * nrm[0]: log-linear extrapolation of the last third,
    with the small-sample factor sqrt((d - j) / d) divided out"""
    k = len(nrm)
    if k < 24:
        return None
    j = np.arange(k)
    corr = nrm / np.sqrt(np.maximum(d - j, 1) / d)
    lo = (2 * k) // 3
    hi = max(lo + 8, k - 12)
    y = np.log(np.maximum(corr[lo:hi], 1e-300) / nrm[0])
    x = j[lo:hi]
    sl, ic = np.polyfit(x, y, 1)
    if sl >= 0:
        return None
    return (np.log(tol_rel) - ic) / sl


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("path")
    ap.add_argument("--d0", type=int, default=128)
    ap.add_argument("--dd", type=int, default=128)
    ap.add_argument("--p", type=int, default=10)
    ap.add_argument("--eps", type=float, default=1e-4)
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    recs = [r for r in read(a.path) if r["side"] == 0]
    by = defaultdict(list)
    for r in recs:
        by[(r["inst"], r["m"], r["node"])].append(r)
    tot_fail = tot_ok = 0
    rows = []
    for key, rs in by.items():
        rs.sort(key=lambda r: r["round"])
        fails = [r for r in rs if not (r["cert"] and r["rank"] <= r["d"] - a.p)]
        oks = [r for r in rs if r["cert"] and r["rank"] <= r["d"] - a.p]
        fs = sum(r["rank"] for r in fails)
        os_ = sum(r["rank"] for r in oks)
        tot_fail += fs
        tot_ok += os_
        pred = None
        if fails and fails[0]["nrm"] is not None and oks:
            pk = predict_rank(fails[0]["nrm"], fails[0]["d"], a.eps)
            if pk is not None:
                pred = int(np.ceil((pk + a.p - a.d0) / a.dd)) + 1
        rows.append((fs + os_, key, rs[0]["mt"], rs[0]["round"], oks[0]["round"] if oks else -1,
                     oks[0]["rank"] if oks else -1, len(fails), fs, os_, pred))
    rows.sort(reverse=True)
    print("pivot steps in failing attempts %d, in certifying attempts %d (%.1fx)" %
          (tot_fail, tot_ok, tot_fail / max(tot_ok, 1)))
    print("%-24s %6s %6s %6s %6s %6s %9s %9s %6s" %
          ("(inst, m, node)", "mt", "first", "cert", "rank", "fails", "failsteps", "oksteps", "pred"))
    for r in rows[:a.top]:
        print("%-24s %6d %6d %6d %6d %6d %9d %9d %6s" %
              (str(r[1]), r[2], r[3], r[4], r[5], r[6], r[7], r[8], str(r[9])))
    # histogram of (cert - first)
    gaps = [r[4] - r[3] for r in rows if r[4] >= 0]
    print("rounds between first attempt and certification: mean %.2f, max %d, zero-gap %d of %d" %
          (np.mean(gaps), max(gaps), sum(g == 0 for g in gaps), len(gaps)))
    errs = [r[9] - r[4] for r in rows if r[9] is not None and r[4] >= 0 and r[6] > 0]
    if errs:
        e = np.array(errs)
        print("prediction from the first failing attempt: predicted - actual certifying round: "
              "mean %.2f, |err|<=1 in %d of %d, min %d max %d" %
              (e.mean(), int((np.abs(e) <= 1).sum()), e.size, e.min(), e.max()))


if __name__ == "__main__":
    main()
