"""Host/GPU timeline of one refactorization under torch.profiler (CUPTI):
which CUDA runtime calls the host threads spend their time in, how busy the
GPU is, and the per-kernel totals. Diagnostic only — numbers taken under the
tracer are never bench values.

usage: python tools/trace.py c3 [--out gpurun_out/trace_c3.json.gz]
"""
import argparse
import collections
import gzip
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1502_07405_b200 as P  # noqa: E402
from paper_1502_07405_b200.problems import CONFIGS  # noqa: E402


def union_len(iv):
    iv.sort()
    tot, cs, ce = 0.0, None, None
    for s, e in iv:
        if cs is None or s > ce:
            if cs is not None:
                tot += ce - cs
            cs, ce = s, e
        else:
            ce = max(ce, e)
    if cs is not None:
        tot += ce - cs
    return tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--out", default=None)
    ap.add_argument("--tail-s", type=float, default=4.0)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    g = P.generate_convdiff3d(cfg.k, 0.1) if cfg.kind == "cd3d" else P.generate_grid_problem(cfg.kind, cfg.k)
    op = P.ordered_problem(g, cfg.nd_leaf)
    m = P.mf_factor(op.a, op.t, cfg.solver_options())
    m.refactor()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        m.refactor()
        torch.cuda.synchronize()
    path = a.out or os.path.join(ROOT, "gpurun_out", f"trace_{a.config}.json")
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    api = collections.defaultdict(lambda: [0, 0.0])
    kern = collections.defaultdict(lambda: [0, 0.0])
    kiv, t0, t1 = [], 1e30, 0
    threads = collections.defaultdict(float)
    sev = collections.defaultdict(list)
    for e in ev:
        if e.get("ph") != "X":
            continue
        c = e.get("cat", "")
        d = float(e.get("dur", 0))
        if c in ("cuda_runtime", "cuda_driver"):
            api[e["name"]][0] += 1
            api[e["name"]][1] += d
            threads[e.get("tid")] += d
        elif c == "kernel":
            nm = e["name"].replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
            nm = nm.split("(")[0].split("<")[0].split("::")[-1]
            kern[nm][0] += 1
            kern[nm][1] += d
            kiv.append((float(e["ts"]), float(e["ts"]) + d))
            st = e.get("args", {}).get("stream", -1)
            sev[st].append((float(e["ts"]), d, nm))
        if c in ("kernel", "cuda_runtime", "cuda_driver", "gpu_memcpy", "gpu_memset"):
            t0 = min(t0, float(e["ts"]))
            t1 = max(t1, float(e["ts"]) + d)
    span = t1 - t0
    mc = collections.Counter()
    for e in ev:
        if e.get("ph") == "X" and e.get("cat") in ("gpu_memcpy", "gpu_memset"):
            mc[e["name"]] += 1
    out = {"config": a.config, "span_ms": span / 1e3, "gpu_busy_ms": union_len(kiv) / 1e3,
           "copies": dict(mc),
           "api_ms_by_thread": {str(k): v / 1e3 for k, v in sorted(threads.items(), key=lambda x: -x[1])[:12]},
           "api": [(k, v[0], round(v[1] / 1e3, 2), round(v[1] / max(v[0], 1), 2))
                   for k, v in sorted(api.items(), key=lambda x: -x[1][1])[:20]],
           "kernels": [(k, v[0], round(v[1] / 1e3, 2)) for k, v in sorted(kern.items(), key=lambda x: -x[1][1])[:20]]}
    # per stream, over the final `tail_s` seconds of the timeline (the top
    # HSS levels): busy fraction and kernel-time breakdown
    tail_us = a.tail_s * 1e6
    per = []
    for st, lst in sev.items():
        w = [(ts, d, nm) for ts, d, nm in lst if ts >= t1 - tail_us]
        if not w:
            continue
        by = collections.Counter()
        cnt = collections.Counter()
        for ts, d, nm in w:
            by[nm] += d
            cnt[nm] += 1
        span_s = max(ts + d for ts, d, _ in w) - min(ts for ts, _, _ in w)
        per.append({"stream": st, "kernels": len(w), "busy_ms": round(sum(by.values()) / 1e3, 1),
                    "span_ms": round(span_s / 1e3, 1),
                    "top": [(k, cnt[k], round(v / 1e3, 1)) for k, v in by.most_common(12)]})
    per.sort(key=lambda x: -x["busy_ms"])
    out["tail_s"] = a.tail_s
    out["tail_streams"] = per[:6]
    print(json.dumps(out, indent=1))
    with open(path, "rb") as f, gzip.open(path + ".gz", "wb") as g2:
        g2.write(f.read())
    os.remove(path)


if __name__ == "__main__":
    main()
