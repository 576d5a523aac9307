"""Small invocations of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per process):
  compute-sanitizer --tool memcheck python tools/sanitize_small.py
Covers: dense-front assembly/LU/solves, HSS compression on both ID routes
(Gram cluster panels with st.async/mbarrier, Householder cluster CPQR),
ULV, densified updates, the 64x64 / 32x32 / TMA GEMMs, split-K, HSS matvec
and extraction, the native multi-GPU driver on one GPU."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_07405_b200 as P  # noqa: E402
import paper_1502_07405_b200.api as A  # noqa: E402
from paper_1502_07405_b200.problems import csr_matvec, dense_c2, x_true  # noqa: E402

op = P.ordered_grid("p3d", 20, 16)
ptr, ind, val = op.a.arrays()
b = csr_matvec(ptr, ind, val, x_true(op.a.size(), 1))
for eps in (1e-6, 1e-4):  # Householder route, Gram route
    so = P.SolverOptions(nd_leaf=16, ls=64, min_hss=200, eps=eps, leaf=32)
    m = P.mf_factor(op.a, op.t, so)
    x = P.mf_solve_new(m, b)
    print("mf eps", eps, "hss", m.hss_fronts, "relres",
          np.linalg.norm(op.a.matvec(x) - b) / np.linalg.norm(b), flush=True)
    del m
from paper_1502_07405_b200.parallel import native_local_solve  # noqa: E402
x2 = native_local_solve(op.a, op.t, P.SolverOptions(nd_leaf=16, mode="mf"), 2, b)
print("mgpu local", np.linalg.norm(op.a.matvec(x2) - b) / np.linalg.norm(b), flush=True)
a = dense_c2(512)
h = P.hss_compress(a, 64, P.HssOptions(eps=1e-8))
print("dense hss rank", h.hss_rank(), flush=True)
xx = np.random.default_rng(0).standard_normal((512, 3))
print("matvec", np.linalg.norm(h.matvec("N", xx) - a @ xx) / np.linalg.norm(a @ xx), flush=True)
print("extract", np.abs(h.extract([3, 200, 7], [500, 1, 64]) - a[np.ix_([3, 200, 7], [500, 1, 64])]).max())
rng = np.random.default_rng(1)
for (ta, tb, mm, nn, kk) in [("N", "N", 100, 70, 30), ("T", "N", 130, 96, 2048),
                             ("N", "T", 258, 130, 2050), ("N", "N", 96, 96, 5000)]:
    aa = rng.standard_normal((mm, kk) if ta == "N" else (kk, mm))
    bb = rng.standard_normal((kk, nn) if tb == "N" else (nn, kk))
    cc = rng.standard_normal((mm, nn))
    got = A.dev_gemm(ta, tb, 1.0, aa, bb, 0.5, cc)
    oa = aa if ta == "N" else aa.T
    ob = bb if tb == "N" else bb.T
    print("gemm", ta, tb, mm, nn, kk, np.abs(got - (oa @ ob + 0.5 * cc)).max(), flush=True)
y = rng.standard_normal((40, 300))
print("gram id rank", A.dev_gram_id(y, 1e-3)[1], flush=True)
