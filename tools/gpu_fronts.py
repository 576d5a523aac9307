"""Run one BASELINE config on the GPU and dump the same per-front / per-node
fields as tests/golden/make_golden.py (type, rank, node_u/v, rounds, d_final,
relres, timings), for a side-by-side comparison with the reference's run.

usage: python tools/gpu_fronts.py c5 --out gpurun_out/gpu_c5.npz
       (env HSSMF_ID_ALGO=householder / HSSMF_NO_SYM=1 select the variants)
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1502_07405_b200 as P  # noqa: E402
from paper_1502_07405_b200.problems import CONFIGS, csr_matvec, x_true  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--out", required=True)
ap.add_argument("--repeat", type=int, default=1)
ap.add_argument("--perturb", type=int, default=0,
                help="seed: move every matrix value by one ulp (seeded signs), as "
                     "tools/ref_sensitivity.py does for the reference")
a = ap.parse_args()

cfg = CONFIGS[a.config]
if cfg.kind == "cd3d":
    op = P.ordered_problem(P.generate_convdiff3d(cfg.k, 0.1), cfg.nd_leaf)
else:
    op = P.ordered_grid(cfg.kind, cfg.k, cfg.nd_leaf)
ptr, ind, val = op.a.arrays()
if a.perturb:
    rng = np.random.default_rng(a.perturb)
    val = np.where(rng.random(val.size) < 0.5, np.nextafter(val, np.inf),
                   np.nextafter(val, -np.inf))
    import paper_1502_07405_b200.api as API  # noqa: E402
    op = API.OrderedProblem(API.SparseMatrix.from_csr(op.a.n, ptr, ind, val), op.t, op.perm, op.geom)
b = csr_matvec(ptr, ind, val, x_true(op.a.size(), 1))
for rep in range(a.repeat):
    t0 = time.perf_counter()
    m = P.mf_factor(op.a, op.t, cfg.solver_options())
    x = P.mf_solve_new(m, b)
    wall = time.perf_counter() - t0
    res = float(np.linalg.norm(op.a.matvec(x) - b) / np.linalg.norm(b))
    hss = np.nonzero(m.type == 1)[0]
    node_u, node_v, node_ptr, rounds, dfin = [], [], [0], [], []
    for i in hss:
        u, v, r, d = m.front_hss(int(i))
        node_u.append(u)
        node_v.append(v)
        node_ptr.append(node_ptr[-1] + len(u))
        rounds.append(r)
        dfin.append(d)
    f, s = m.timing()
    env = {k: v for k, v in os.environ.items() if k.startswith("HSSMF_")}
    out = os.path.splitext(a.out)[0] + (f"_{rep}" if a.repeat > 1 else "") + ".npz"
    np.savez_compressed(
        out, relres=res, wall=wall, factor_ms=f, solve_ms=s, rank=m.rank, type=m.type,
        level=m.level, dim=m.dim, flops=m.flops, hss_ids=hss.astype(np.int32),
        node_ptr=np.array(node_ptr, np.int32),
        node_u=np.concatenate(node_u) if node_u else np.zeros(0, np.int32),
        node_v=np.concatenate(node_v) if node_v else np.zeros(0, np.int32),
        rounds=np.array(rounds, np.int32), d_final=np.array(dfin, np.int32), env=str(env))
    print(f"{a.config} {env}: wall {wall:.2f}s factor {f:.0f}ms relres {res:.4e} "
          f"hss {m.hss_fronts} maxrank {m.max_front_rank} rounds max {max(rounds, default=0)}",
          flush=True)
    del m
