"""Validation of the reference arm's sample scaling (bench.py reference_scaled):
on one host, time the reference (oracle/_ref) on the WHOLE workload and the
scaled sample estimate with the same threads, and print both.

usage: python tools/validate_ref_scaling.py c3 c5_96 [--budget 150] [--steps 5]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from oracle import ref  # noqa: E402
from paper_1502_07405_b200.problems import CONFIGS, csr_matvec, x_true  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="+")
ap.add_argument("--budget", type=float, default=150.0)
ap.add_argument("--steps", type=int, default=5)
a = ap.parse_args()
thr = bench.cpu_threads()
for name in a.configs:
    cfg = CONFIGS[name]
    o = bench.oracle_ordered(cfg)
    tv = bench.TreeView.of_oracle(o)
    ref.set_threads(thr)
    b = csr_matvec(o.ptr, o.ind, o.val, x_true(o.n, 1))
    t0 = time.perf_counter()
    F = ref.Factors(o, eps=cfg.eps, ls=cfg.ls, leaf=cfg.leaf, d0=cfg.d0, dd=cfg.dd, p=cfg.p,
                    min_hss=cfg.min_hss, mode={"auto": 0, "mf": 1, "mf-hss": 2}[cfg.mode])
    F.solve(b)
    full = time.perf_counter() - t0
    model = float(F.flops.astype(np.float64).sum())
    # the sample scaled by the full run's own per-front model (what bench.py
    # does once tests/golden/ref_<config>.npz holds the full run)
    est, t, scale, desc = bench.reference_scaled(cfg, tv, thr, a.steps, 1, a.budget,
                                                 full_model=F.flops)
    print(json.dumps({"config": name, "threads": thr, "full_s": full,
                      "full_factor_s": F.factor_seconds, "scaled_estimate_s": est,
                      "ratio_estimate_over_full": est / full, "sample_s": t, "scale": scale,
                      "full_model_flops": model, "sample": desc}), flush=True)
