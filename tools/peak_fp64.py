"""Measure the FP64 roofline denominators on the box: cuBLAS DGEMM (torch
float64 matmul) burst and the project's DMMA GEMM at the same sizes."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1502_07405_b200 import _native as N  # noqa: E402

out = {}
for n in [4096, 8192]:
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out[f"cublas_dgemm_{n}_tflops"] = 2 * n ** 3 / best / 1e9
    ms = C.c_double()
    st = N.Status()
    rc = N.lib().hssmf_bench_gemm(0, n, n, n, 5, C.byref(ms), C.byref(st))
    out[f"dmma_gemm_{n}_tflops"] = 2 * n ** 3 / ms.value / 1e9 if rc == 0 else st.msg.decode()
for (m, n, k) in [(3000, 3000, 961), (2048, 2048, 32), (16384, 128, 16384), (8192, 8192, 64)]:
    ms = C.c_double()
    st = N.Status()
    N.lib().hssmf_bench_gemm(0, m, n, k, 5, C.byref(ms), C.byref(st))
    out[f"dmma_gemm_{m}x{n}x{k}_tflops"] = 2 * m * n * k / ms.value / 1e9
x = torch.empty(2 ** 28, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(3):
    y.copy_(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    y.copy_(x)
e1.record()
torch.cuda.synchronize()
out["copy_gbs"] = 10 * 2 * x.numel() * 8 / e0.elapsed_time(e1) / 1e6
print(json.dumps(out, indent=1))
