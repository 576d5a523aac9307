"""Per-front comparison of a tools/gpu_fronts.py dump with a reference golden
(tests/golden/ref_<config>.npz): front types, ranks within +-10%, rounds, relres.

usage: python tools/compare_fronts.py gpurun_out/gpu_c5.npz tests/golden/ref_c5.npz
"""
import sys

import numpy as np

d = np.load(sys.argv[1], allow_pickle=True)
g = np.load(sys.argv[2], allow_pickle=True)
hs = g["hss_ids"]
r, rr = d["rank"][hs].astype(float), g["rank"][hs].astype(float)
ok = np.abs(r - rr) <= 0.1 * rr
lv = g["level"][hs]
print("types equal:", bool(np.array_equal(d["type"], g["type"])), " HSS fronts:", hs.size)
print("relres: ours %.3f, reference %.3f" % (float(d["relres"]), float(g["relres"])))
print("fronts within +-10%%: %d / %d (tree level >= 3: %d / %d)" %
      (int(ok.sum()), ok.size, int(ok[lv >= 3].sum()), int((lv >= 3).sum())))
print("rounds equal: %d / %d" % (int((d["rounds"] == g["rounds"]).sum()), hs.size))
for q in np.nonzero(~ok)[0]:
    print("  front %d level %d: rank %d vs %d, rounds %d vs %d" %
          (hs[q], lv[q], r[q], rr[q], d["rounds"][q], g["rounds"][q]))
