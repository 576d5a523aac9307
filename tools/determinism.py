"""Run-to-run determinism of a config: factor it several times in one process and
compare per-front ranks and per-node ranks between the runs and with the
reference golden (tests/golden/ref_<config>.npz).

usage: python tools/determinism.py c4 [--repeat 3]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1502_07405_b200 as P  # noqa: E402
from paper_1502_07405_b200.problems import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--repeat", type=int, default=3)
a = ap.parse_args()
cfg = CONFIGS[a.config]
if cfg.kind == "cd3d":
    op = P.ordered_problem(P.generate_convdiff3d(cfg.k, 0.1), cfg.nd_leaf)
else:
    op = P.ordered_grid(cfg.kind, cfg.k, cfg.nd_leaf)
g = np.load(os.path.join(ROOT, "tests", "golden", f"ref_{a.config}.npz"))
hs = g["hss_ids"]
runs = []
for rep in range(a.repeat):
    m = P.mf_factor(op.a, op.t, cfg.solver_options())
    nodes = np.concatenate([m.front_hss(int(i))[0] for i in hs])
    runs.append((m.rank[hs].copy(), nodes))
    del m
env = {k: v for k, v in os.environ.items() if k.startswith("HSSMF_")}
ref_r, ref_n = g["rank"][hs], g["node_u"]
for rep, (r, n) in enumerate(runs):
    dr = np.abs(r - ref_r) / np.maximum(ref_r, 1)
    dn = np.abs(n - ref_n) / np.maximum(ref_n, 10) if n.shape == ref_n.shape else np.array([np.inf])
    print(f"{a.config} {env} run {rep}: fronts != ref {int((r != ref_r).sum())}/{r.size} (max rel {dr.max():.3f}), "
          f"nodes != ref {int((n != ref_n).sum()) if n.shape == ref_n.shape else -1}/{n.size} (max rel {dn.max():.3f}); "
          f"vs run 0: fronts differ {int((r != runs[0][0]).sum())}, nodes differ "
          f"{int((n != runs[0][1]).sum()) if n.shape == runs[0][1].shape else -1}")
