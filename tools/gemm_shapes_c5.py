"""Per-launch GEMM shape study of one c5 refactorization (probe dump):
where the DMMA grouped GEMM time goes by (CTA tiles, longest K)."""
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["HSSMF_PROBE_DUMP"] = os.path.join(ROOT, "gpurun_out", "probe_dump.csv")

import numpy as np  # noqa: E402

import paper_1502_07405_b200 as P  # noqa: E402
from paper_1502_07405_b200.problems import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
g = P.generate_grid_problem(cfg.kind, cfg.k)
op = P.ordered_problem(g, cfg.nd_leaf)
m = P.mf_factor(op.a, op.t, cfg.solver_options())
P.api.probe_read()
P.api.probe_enable(True)
m.refactor()
P.api.probe_read()
P.api.probe_enable(False)
rows = [l.strip().split(",") for l in open(os.environ["HSSMF_PROBE_DUMP"])][1:]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
PH = ["sample", "extract", "local", "cpqr", "finalize", "update_done", "ulv_elim", "ulv_top",
      "densify"]
byph = collections.defaultdict(lambda: [0, 0.0])
for kind, ms, fl, by, tiles, kmax, npb, ph in rows:
    k = ("gemm" if kind == "0" else "panel" if kind == "1" else "syrk") + "/" + \
        (PH[int(ph)] if 0 <= int(ph) < len(PH) else "dense")
    byph[k][0] += 1
    byph[k][1] += float(ms)
for k, (c, ms) in sorted(byph.items(), key=lambda x: -x[1][1]):
    print(f"{k:24s} {c:7d} launches {ms:9.1f} ms")
for kind, ms, fl, by, tiles, kmax, npb, ph in rows:
    if kind != "0":
        continue
    t, k = int(tiles), int(kmax)
    tb = "<148" if t < 148 else "<592" if t < 592 else ">=592"
    kb = "<256" if k < 256 else "<1024" if k < 1024 else "<4096" if k < 4096 else ">=4096"
    a = agg[(tb, kb)]
    a[0] += 1
    a[1] += float(ms)
    a[2] += float(fl)
tot = sum(v[1] for v in agg.values())
for key, (c, ms, fl) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"tiles {key[0]:>6} K {key[1]:>6}: {c:6d} launches {ms:9.1f} ms ({100 * ms / tot:5.1f}%) "
          f"{fl / max(ms, 1e-9) / 1e9:6.2f} TF/s")

# Gram panel launches by cluster size (rows per task up to 512 * CL)
pan = collections.defaultdict(lambda: [0, 0.0])
for kind, ms, fl, by, tiles, kmax, npb, ph in rows:
    if kind == "1":
        pan[int(tiles)][0] += 1
        pan[int(tiles)][1] += float(ms)
ptot = sum(v[1] for v in pan.values()) or 1.0
for cl, (c, ms) in sorted(pan.items()):
    print(f"gram panel CL {cl:2d}: {c:6d} launches {ms:9.1f} ms ({100 * ms / ptot:5.1f}%) "
          f"{1e3 * ms / max(c, 1):7.1f} us/launch")
