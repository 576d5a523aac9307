"""Bitwise reproducibility of single GEMMs through the split-K / TMA entry: the
same product repeated, every result compared with the first and with numpy.
(c4's run-to-run variation was traced to the transposed-operand TMA launches;
HSSMF_TMA_TRANS=1 routes transposed operands to the TMA kernel.)

usage: HSSMF_TMA_TRANS=1 python tools/gemm_repro.py [--repeat 8]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_07405_b200.api as A  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--repeat", type=int, default=8)
a = ap.parse_args()
rng = np.random.default_rng(0)
cases = [("T", "N", 9000, 128, 9000), ("T", "N", 13954, 128, 13954), ("N", "T", 5000, 5000, 2600),
         ("N", "T", 3001, 2999, 2304), ("T", "T", 2000, 1500, 2100), ("N", "N", 13954, 128, 13954),
         ("T", "N", 4100, 4100, 2200)]
for (ta, tb, m, n, k) in cases:
    aa = rng.standard_normal((m, k) if ta == "N" else (k, m))
    bb = rng.standard_normal((k, n) if tb == "N" else (n, k))
    cc = np.zeros((m, n))
    ref = (aa if ta == "N" else aa.T) @ (bb if tb == "N" else bb.T)
    first, nd, worst = None, 0, 0.0
    for r in range(a.repeat):
        got = A.dev_gemm(ta, tb, 1.0, aa, bb, 0.0, cc)
        worst = max(worst, float(np.abs(got - ref).max() / np.abs(ref).max()))
        if first is None:
            first = got
        elif not np.array_equal(first, got):
            nd += 1
            d = np.argwhere(first != got)
            print(f"   repeat {r}: {len(d)} entries differ, first at {d[0].tolist()}, "
                  f"max |diff| {np.abs(first - got).max():.3e}", flush=True)
    print(f"gemm {ta}{tb} {m} x {n} x {k}: {a.repeat} repeats, {nd} differ from the first, "
          f"max rel error vs numpy {worst:.2e}", flush=True)
