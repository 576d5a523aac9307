"""DMMA GEMM throughput on the shapes of the hot path (all transposes), for the
static-batch 64x64 cp.async kernel ("static"), the dynamic-batch entry that
routes eligible problems to the TMA 128x128 kernel ("mixed") and the split-K
entry of the sampling products ("splitk")."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1502_07405_b200 import _native as N  # noqa: E402

shapes = [(8192, 8192, 8192), (20480, 128, 20480), (8000, 8000, 64), (4096, 4096, 128),
          (3000, 3000, 960), (2048, 2048, 32), (6000, 128, 6000), (1024, 1024, 256)]
out = {}
for path in ["static", "mixed", "splitk"]:
    os.environ["HSSMF_BENCH_PATH"] = path
    for tr in ["NN", "TN", "NT"]:
        os.environ["HSSMF_BENCH_TRANS"] = tr
        for (m, n, k) in shapes:
            if path == "splitk" and n > 512:
                continue
            ms, st = C.c_double(), N.Status()
            N.lib().hssmf_bench_gemm(0, m, n, k, 5, C.byref(ms), C.byref(st))
            out[f"{path}_{tr}_{m}x{n}x{k}_tflops"] = round(2 * m * n * k / ms.value / 1e9, 2)
print(json.dumps(out, indent=1))
