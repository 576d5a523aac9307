"""Kernel-level breakdown of one mf_solve on a BASELINE config under
torch.profiler (CUPTI). Diagnostic only: numbers under the tracer are never
bench values.

usage: python tools/trace_solve.py c5
"""
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1502_07405_b200 as P  # noqa: E402
from paper_1502_07405_b200.problems import CONFIGS  # noqa: E402


def main():
    cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
    g = P.generate_grid_problem(cfg.kind, cfg.k)
    op = P.ordered_problem(g, cfg.nd_leaf)
    m = P.mf_factor(op.a, op.t, cfg.solver_options())
    n = op.a.size()
    b = torch.ones(n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        m.solve_device(b.data_ptr(), n, 1)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        m.solve_device(b.data_ptr(), n, 1)
        torch.cuda.synchronize()
    path = os.path.join(ROOT, "gpurun_out", "trace_solve.json")
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    os.remove(path)
    kern = collections.defaultdict(lambda: [0, 0.0])
    t0, t1 = 1e30, 0
    for e in ev:
        if e.get("ph") != "X":
            continue
        if e.get("cat") == "kernel":
            nm = e["name"].replace("(anonymous namespace)::", "").split("(")[0]
            kern[nm][0] += 1
            kern[nm][1] += float(e["dur"])
        if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset", "cuda_runtime"):
            t0 = min(t0, float(e["ts"]))
            t1 = max(t1, float(e["ts"]) + float(e.get("dur", 0)))
    api = collections.Counter()
    for e in ev:
        if e.get("ph") == "X" and e.get("cat") == "cuda_runtime":
            api[e["name"]] += 1
    fms, sms = m.timing()
    print(json.dumps({"span_ms": (t1 - t0) / 1e3, "solve_ms_events": sms,
                      "kernels": sorted(([k, v[0], round(v[1] / 1e3, 2)] for k, v in kern.items()),
                                        key=lambda x: -x[2])[:25],
                      "api": api.most_common(10)}, indent=1))


if __name__ == "__main__":
    main()
