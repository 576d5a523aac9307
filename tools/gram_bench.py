"""Per-step latency of the Gram-route pivoted-Cholesky ID kernel on the node
sizes of the HSS path (measurement only)."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1502_07405_b200 import _native as N  # noqa: E402

cases = [(256, 192, 1), (512, 320, 8), (1024, 640, 8), (2048, 1300, 4), (4096, 2600, 2),
         (7400, 3700, 1)]
if len(sys.argv) == 4:
    cases = [tuple(int(a) for a in sys.argv[1:4])]
out = []
for (n, d, nt) in cases:
    ms, steps, st = C.c_double(), C.c_int(), N.Status()
    rc = N.lib().hssmf_bench_gram(0, n, d, nt, 3, C.byref(ms), C.byref(steps), C.byref(st))
    if rc:
        out.append({"n": n, "error": st.msg.decode()})
        continue
    out.append({"n": n, "d": d, "tasks": nt, "steps": steps.value, "ms": round(ms.value, 3),
                "us_per_step": round(1e3 * ms.value / max(steps.value, 1), 3)})
print(json.dumps(out, indent=1))
