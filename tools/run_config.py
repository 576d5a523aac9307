"""Run one BASELINE config on the GPU and compare with the reference golden
fixture (tests/golden/ref_<config>.npz) when present.

usage: python tools/run_config.py c3 [--profile]
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
from paper_1502_07405_b200.problems import CONFIGS, csr_matvec, dense_c2, x_true  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--repeat", type=int, default=1)
    ap.add_argument("--save-model", default=None,
                    help="write per-front (type, rank, d_final) for bench.py's CPU extrapolation")
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    out = {"config": a.config}
    if cfg.kind == "dense":
        A = dense_c2(cfg.k)
        b = x_true(cfg.k, 1)
        for _ in range(a.repeat):
            t0 = time.perf_counter()
            h = P.hss_compress(A, cfg.leaf, P.HssOptions(eps=cfg.eps))
            t1 = time.perf_counter()
            x = h.solve(b)
            t2 = time.perf_counter()
        out.update(compress_ms=h.compress_ms, ulv_ms=h.ulv_ms, wall_factor_s=t1 - t0,
                   wall_solve_s=t2 - t1, rounds=h.rounds, d_final=h.d_final,
                   rank=h.hss_rank(), relres=float(np.linalg.norm(A @ x - b) / np.linalg.norm(b)),
                   ranks=h.u_rank.tolist())
        print(json.dumps(out))
        return
    t0 = time.perf_counter()
    if cfg.kind == "cd3d":
        g = P.generate_convdiff3d(cfg.k, 0.1)
    else:
        g = P.generate_grid_problem(cfg.kind, cfg.k)
    op = P.ordered_problem(g, cfg.nd_leaf)
    out["analysis_s"] = time.perf_counter() - t0
    ptr, ind, val = op.a.arrays()
    b = csr_matvec(ptr, ind, val, x_true(op.a.size(), 1))
    so = cfg.solver_options()
    t0 = time.perf_counter()
    m = P.mf_factor(op.a, op.t, so)
    out["first_factor_wall_s"] = time.perf_counter() - t0
    for _ in range(a.repeat - 1):
        m.refactor()
    if a.profile:
        m.set_profile(True)
        m.reset_kernel_stats()
        m.refactor()
    t0 = time.perf_counter()
    x = P.mf_solve_new(m, b)
    out["solve_wall_s"] = time.perf_counter() - t0
    fms, sms = m.timing()
    out.update(factor_ms=fms, solve_ms=sms, hss_fronts=m.hss_fronts, fallbacks=m.fallbacks,
               max_front_rank=m.max_front_rank,
               relres=float(np.linalg.norm(op.a.matvec(x) - b) / np.linalg.norm(b)),
               device_gb=m.device_bytes() / 1e9)
    if a.profile:
        out["kernels"] = m.kernel_stats()
    if a.save_model:
        dfin = np.zeros(len(m.type), np.int32)
        for i in np.nonzero(m.type == 1)[0]:
            dfin[i] = m.front_hss(int(i))[3]
        np.savez_compressed(a.save_model, type=m.type, rank=m.rank, d_final=dfin,
                            level=m.level, dim=m.dim)
    gp = os.path.join(ROOT, "tests", "golden", f"ref_{a.config}.npz")
    if os.path.exists(gp):
        g = np.load(gp)
        out["ref"] = dict(factor_s=float(g["factor_s"]), solve_s=float(g["solve_s"]),
                          relres=float(g["relres"]), max_front_rank=int(g["max_front_rank"]),
                          threads=int(g["threads"]), hss_fronts=int(g["hss_fronts"]))
        out["types_equal"] = bool(np.array_equal(m.type, g["type"]))
        hs = g["hss_ids"]
        rm, rr = m.rank[hs].astype(float), g["rank"][hs].astype(float)
        out["front_rank_maxrel"] = float(np.max(np.abs(rm - rr) / np.maximum(rr, 1))) if len(hs) else 0
        devs = []
        for q, i in enumerate(hs):
            fh = m.front_hss(int(i))
            if fh is None:
                devs.append(1.0)
                continue
            u = fh[0][:-1].astype(float)
            ru = g["node_u"][g["node_ptr"][q]:g["node_ptr"][q + 1]][:-1].astype(float)
            devs.append(float(np.max(np.abs(u - ru) / np.maximum(ru, 10))) if len(u) else 0.0)
        out["node_rank_maxrel_floor10"] = max(devs) if devs else 0.0
        if "x" in g.files:
            out["x_relerr_vs_ref"] = float(np.linalg.norm(x - g["x"]) / np.linalg.norm(g["x"]))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
