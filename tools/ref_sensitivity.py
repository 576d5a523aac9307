"""Sensitivity of the REFERENCE's own HSS ranks to a one-ulp perturbation of
the input (test infrastructure: runs oracle/_ref, the unmodified reference).

Runs the reference on the bench's self-contained subtree sample of config 5
rooted at front S (bench.subtree_sample: the subtree, a dense synthetic root
over its update indices), once on the original values and once with every
matrix value moved by at most one unit in the last place (seeded signs), and
prints per HSS front of the sample: rank and adaptive rounds of both runs and
whether the front assembles a compressed (HSS) child. The fronts whose ranks
move under a perturbation far below eps are the ones where no implementation
can be held to +-10% of one reference run (tests/test_gpu_hss.py C5 gate).

usage: python tools/ref_sensitivity.py 71485 [--threads 8] [--out file.json]
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
from paper_1502_07405_b200.problems import CONFIGS  # noqa: E402


def run(cfg, pieces, threads):
    ref.set_threads(threads)
    o = ref.ordered_from_arrays(pieces["n"], pieces["ptr"], pieces["ind"], pieces["val"],
                                pieces["sep_begin"], pieces["sep_end"], pieces["child0"],
                                pieces["child1"], pieces["parent"], pieces["upd_ptr"],
                                pieces["upd_ind"])
    mode = {"auto": 0, "mf": 1, "mf-hss": 2}[cfg.mode]
    t0 = time.perf_counter()
    F = ref.Factors(o, eps=cfg.eps, ls=cfg.ls, leaf=cfg.leaf, d0=cfg.d0, dd=cfg.dd, p=cfg.p,
                    min_hss=cfg.min_hss, mode=mode)
    t = time.perf_counter() - t0
    b = bench.ref_rhs(pieces["ptr"], pieces["ind"], pieces["val"], pieces["n"])
    x = F.solve(b)[:, 0]
    from paper_1502_07405_b200.problems import csr_matvec
    res = np.linalg.norm(csr_matvec(pieces["ptr"], pieces["ind"], pieces["val"], x) - b) / \
        np.linalg.norm(b)
    out = {}
    for i in np.nonzero(F.type == 1)[0]:
        u, v, r, d = F.front_hss(int(i))
        out[int(i)] = (int(F.rank[i]), int(r))
    return out, t, float(res)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("front", type=int)
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--seeds", type=int, default=1)
    ap.add_argument("--out")
    a = ap.parse_args()
    cfg = CONFIGS["c5"]
    tv = bench.TreeView.of_oracle(bench.oracle_ordered(cfg))
    pieces, ids, desc = bench.subtree_sample(tv, cfg, a.front)
    print(desc, flush=True)
    p0 = pieces["parent"]
    c0, c1 = pieces["child0"], pieces["child1"]
    runs = []
    for sd in range(a.seeds + 1):
        pc = dict(pieces)
        if sd:
            rng = np.random.default_rng(sd)
            v = pieces["val"].copy()
            pc["val"] = np.where(rng.random(v.size) < 0.5, np.nextafter(v, np.inf),
                                 np.nextafter(v, -np.inf))
        r, t, res = run(cfg, pc, a.threads)
        print(f"run {sd}: {t:.1f} s, relres {res:.3e}", flush=True)
        runs.append(dict(seed=sd, seconds=t, relres=res, fronts=r))
    base = runs[0]["fronts"]
    print("%7s %6s %5s  %s" % ("front", "hsskid", "ref", "perturbed runs: rank(rounds)"))
    rows = []
    for i in sorted(base):
        hk = any(c >= 0 and c in base for c in (c0[i], c1[i]))
        line = [(runs[k]["fronts"].get(i, (0, 0))) for k in range(1, len(runs))]
        print("%7d %6s %5d(%2d)  %s" % (i + ids[0] if i < len(ids) else -1, hk, base[i][0],
                                        base[i][1], " ".join("%d(%d)" % x for x in line)))
        rows.append(dict(front=int(ids[i]) if i < len(ids) else -1, hss_child=bool(hk),
                         ranks=[base[i][0]] + [x[0] for x in line],
                         rounds=[base[i][1]] + [x[1] for x in line]))
    del p0
    if a.out:
        json.dump(dict(sample=desc, threads=a.threads, runs=[{k: v for k, v in r.items()
                                                               if k != "fronts"} for r in runs],
                       fronts=rows), open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
