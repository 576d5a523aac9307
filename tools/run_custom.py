"""Ad-hoc GPU run of a grid problem with explicit solver options.

usage: python tools/run_custom.py p3d 96 --nd-leaf 32 --min-hss 4000 --eps 1e-4 --leaf 256
       [--ls 64] [--mode auto] [--ref]   (--ref also runs oracle/_ref, build container only)
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1502_07405_b200 as P  # noqa: E402
from paper_1502_07405_b200.problems import csr_matvec, x_true  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("kind")
ap.add_argument("k", type=int)
ap.add_argument("--nd-leaf", type=int, default=32)
ap.add_argument("--ls", type=int, default=64)
ap.add_argument("--min-hss", type=int, default=4000)
ap.add_argument("--eps", type=float, default=1e-4)
ap.add_argument("--leaf", type=int, default=256)
ap.add_argument("--mode", default="auto")
ap.add_argument("--ref", action="store_true")
ap.add_argument("--gpu", action="store_true")
a = ap.parse_args()

op = P.ordered_grid(a.kind, a.k, a.nd_leaf)
ptr, ind, val = op.a.arrays()
b = csr_matvec(ptr, ind, val, x_true(op.a.size(), 1))
so = P.SolverOptions(nd_leaf=a.nd_leaf, ls=a.ls, min_hss=a.min_hss, eps=a.eps, leaf=a.leaf,
                     mode=a.mode)
out = {"kind": a.kind, "k": a.k}
if a.gpu:
    t0 = time.perf_counter()
    m = P.mf_factor(op.a, op.t, so)
    x = P.mf_solve_new(m, b)
    out["gpu"] = dict(wall=time.perf_counter() - t0, factor_ms=m.timing()[0],
                      relres=float(np.linalg.norm(op.a.matvec(x) - b) / np.linalg.norm(b)),
                      hss=m.hss_fronts, maxrank=m.max_front_rank,
                      ranks=[int(m.rank[i]) for i in np.nonzero(m.type == 1)[0]])
if a.ref:
    from oracle import ref
    o = ref.ordered_grid(a.kind, a.k, a.nd_leaf)
    t0 = time.perf_counter()
    F = ref.Factors(o, eps=a.eps, ls=a.ls, leaf=a.leaf, min_hss=a.min_hss,
                    mode={"auto": 0, "mf": 1, "mf-hss": 2}[a.mode])
    xr = F.solve(b)[:, 0]
    import scipy.sparse as sp
    A = sp.csr_matrix((o.val, o.ind, o.ptr), shape=(o.n, o.n))
    out["ref"] = dict(wall=time.perf_counter() - t0, relres=float(np.linalg.norm(A @ xr - b) / np.linalg.norm(b)),
                      hss=F.hss_fronts, maxrank=F.max_front_rank,
                      ranks=[int(F.rank[i]) for i in np.nonzero(F.type == 1)[0]])
print(json.dumps(out))
