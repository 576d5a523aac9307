import ctypes as C, sys, json
sys.path.insert(0, "/root/repo")
from paper_1502_07405_b200 import _native as N
out = {}
for (m, n, k) in [(640, 128, 128), (1280, 128, 256), (2560, 128, 128), (256, 128, 256), (4096, 128, 64), (3000, 128, 1500)]:
    ms, st = C.c_double(), N.Status()
    N.lib().hssmf_bench_gemm(0, m, n, k, 50, C.byref(ms), C.byref(st))
    out[f"{m}x{n}x{k}"] = {"us": round(ms.value * 1e3, 1), "tf": round(2 * m * n * k / ms.value / 1e9, 2)}
print(json.dumps(out))
