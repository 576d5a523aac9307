#!/usr/bin/env python
"""Benchmark: HSS-multifrontal factor + solve on B200 (BASELINE.json metric
"factor+solve time (s) ... 3D Poisson 128^3").

A step = one numeric factorization + one solve of the configured workload
(default: BASELINE config 5, 3D Poisson 128^3). Analysis (ordering, etree,
symbolic) is input preparation and stays outside the timed region, as in the
reference's own measurement protocol.

  value : device-resident inputs (matrix values and b already in HBM), wall
          time of K steps bracketed by cuda synchronize + barrier, max over ranks
  e2e   : the public API call a user makes - mf_factor(A, tree, opts) with host
          CSR + mf_solve_new(m, b_host) - host<->device copies inside the region
  --impl reference : the reference CPU implementation (oracle/_ref, compiled
          from /root/reference) on the host cores, on a bounded subtree sample of
          the same workload, scaled by algorithmic flops to the full workload
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_CONFIG = "c5"


# per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the
# probed kernels from one `ncu --set full` capture of the bench workload,
# committed under profiles/ (null when absent)
def _traffic():
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


TRAFFIC = _traffic()


def dense_flops(ns, nu):
    ns = ns.astype(np.float64)
    nu = nu.astype(np.float64)
    return 2 * ns ** 3 / 3 + 2 * ns ** 2 * nu + 2 * ns * nu ** 2


def build_problem(cfg):
    import paper_1502_07405_b200 as P
    if cfg.kind == "cd3d":
        g = P.generate_convdiff3d(cfg.k, 0.1)
    else:
        g = P.generate_grid_problem(cfg.kind, cfg.k)
    return P.ordered_problem(g, cfg.nd_leaf)


# ---------------------------------------------------------------- clocks ----
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.p = None

    def _read(self):
        for line in self.p.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for nm, v in zip(names, r[3:7]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
            except Exception:
                pass
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ peaks --------
def measured_peaks(torch, dev):
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        peaks["hbm_gbs"] = float(mp["hbm_gbs"])
        peaks["hbm_src"] = "MEASURED_PEAKS.json"
    except Exception:
        peaks["hbm_gbs"] = 6650.0
        peaks["hbm_src"] = "fallback B200_PROFILING.md"
    # FP64: MEASURED_PEAKS.json has no FP64 entry; measure cuBLAS DGEMM (burst)
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    for _ in range(2):
        a @ b
    torch.cuda.synchronize(dev)
    best = 1e30
    for _ in range(3):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize(dev)
        best = min(best, e0.elapsed_time(e1))
    peaks["fp64_tflops"] = 2 * n ** 3 / best / 1e9
    peaks["fp64_src"] = "measured in-run: cuBLAS DGEMM 8192^3 burst (torch float64 matmul)"
    del a, b
    torch.cuda.empty_cache()
    return peaks


# ------------------------------------------------------ reference sample ---
class TreeView:
    """the arrays a sample needs, from the oracle's Ordered (reference arm: no
    product library is loaded) or from the product's OrderedProblem"""

    def __init__(self, ptr, ind, val, sep_begin, sep_end, child0, child1, parent, level,
                 upd_ptr, upd_ind):
        self.ptr, self.ind, self.val = ptr, ind, val
        self.sep_begin, self.sep_end = np.asarray(sep_begin), np.asarray(sep_end)
        self.child0, self.child1 = np.asarray(child0), np.asarray(child1)
        self.parent, self.level = np.asarray(parent), np.asarray(level)
        self.upd_ptr, self.upd_ind = np.asarray(upd_ptr), np.asarray(upd_ind)
        self.nn = len(self.sep_begin)

    def upd(self, i):
        return self.upd_ind[self.upd_ptr[i]:self.upd_ptr[i + 1]]

    @classmethod
    def of_oracle(cls, o):
        return cls(o.ptr, o.ind, o.val, o.sep_begin, o.sep_end, o.child0, o.child1, o.parent,
                   o.level, o.upd_ptr, o.upd_ind)

    @classmethod
    def of_product(cls, op):
        t = op.t
        ptr, ind, val = op.a.arrays()
        return cls(ptr, ind, val, t.sep_begin, t.sep_end, t.child0, t.child1, t.parent, t.level,
                   t.upd_ptr, t.upd_ind)


def oracle_ordered(cfg):
    """the reference's own ordering / tree for the workload (oracle/_ref)"""
    from oracle import ref
    if cfg.kind == "cd3d":  # config 4 has no reference generator
        import paper_1502_07405_b200 as P
        ptr, ind, val = P.generate_convdiff3d(cfg.k, 0.1).A.arrays()
        return ref.ordered_csr_geom(ptr, ind, val, (cfg.k,) * 3, 3, cfg.nd_leaf)
    return ref.ordered_grid(cfg.kind, cfg.k, cfg.nd_leaf)


def front_model(tv, cfg):
    """per-front cost by the reference's own FrontStat.flops estimate
    (multifrontal.hpp:389-396, 432-445: dense 2ns^3/3 + 2ns^2 nu + 2ns nu^2,
    HSS 4 m^2 d_final + 8 m r^2) with the HSS fronts' (rank, d_final) of the
    full reference run (tests/golden/ref_<config>.npz) when it exists, else of
    the recorded product run (tests/golden/<workload>_front_model.npz).
    Returns (flops per front, source)."""
    ns = (tv.sep_end - tv.sep_begin).astype(np.float64)
    nu = np.diff(tv.upd_ptr).astype(np.float64)
    fl = dense_flops(ns, nu)
    key = [k for k, v in __import__("paper_1502_07405_b200.problems",
                                     fromlist=["CONFIGS"]).CONFIGS.items() if v is cfg]
    for path, src in ((os.path.join(ROOT, "tests", "golden", f"ref_{key[0]}.npz") if key else "",
                       "reference run"),
                      (os.path.join(ROOT, "tests", "golden", f"{cfg.name}_front_model.npz"),
                       "product run")):
        if path and os.path.exists(path):
            g = np.load(path)
            if len(g["rank"]) != len(fl):
                continue
            h = np.asarray(g["type"]) == 1
            m = ns + nu
            if "d_final" in g and len(g["d_final"]) == len(fl):
                dfin = g["d_final"].astype(np.float64)
            else:  # per-HSS-front arrays (make_golden layout)
                dfin = np.zeros(len(fl))
                dfin[np.asarray(g["hss_ids"])] = g["d_final"]
            fl = np.where(h, 4 * m ** 2 * dfin + 8 * m * g["rank"].astype(np.float64) ** 2, fl)
            return fl, src + " " + os.path.basename(path)
    return fl, "dense-front model only"


def hss_wanted(tv, cfg):
    """structural HSS selection (multifrontal.hpp:410-412)"""
    ns = tv.sep_end - tv.sep_begin
    m = ns + np.diff(tv.upd_ptr)
    ls = 0 if cfg.mode == "mf" else cfg.ls
    return (tv.level < ls) & (m >= cfg.min_hss) & (ns > 0)


def sample_candidates(tv, cfg):
    """HSS-rooted subtrees of the workload (front s with its whole subtree),
    cheapest first: [(model cost, s)]; the model costs come from front_model"""
    fl, _ = front_model(tv, cfg)
    nn = tv.nn
    want = hss_wanted(tv, cfg)
    sub = fl.copy()
    for i in range(nn):  # postorder: children first
        for c in (tv.child0[i], tv.child1[i]):
            if c >= 0:
                sub[i] += sub[c]
    cand = np.nonzero(want & (tv.parent >= 0))[0]
    if not len(cand):  # no HSS front: dense subtrees along the root's child0 chain
        cand, s = [], int(tv.child0[nn - 1])
        while s >= 0:
            cand.append(s)
            s = int(tv.child0[s])
        cand = np.array(cand, np.int64)
    order = cand[np.argsort(sub[cand])]
    return [(float(sub[s]), int(s)) for s in order]


def subtree_sample(tv, cfg, s):
    """A bounded, self-contained piece of the same workload for the CPU
    reference: the subtree of front s plus a synthetic root front whose
    separator is upd(s), over the principal submatrix on those indices. Every
    front of the subtree keeps the (ns, nu) it has in the full run, so HSS
    fronts stay HSS. Returns (pieces, sample ids, description)."""
    nn = tv.nn
    ns = tv.sep_end - tv.sep_begin
    m = ns + np.diff(tv.upd_ptr)
    want = hss_wanted(tv, cfg)
    lo = np.arange(nn)
    for i in range(nn):  # postorder: children first
        for c in (tv.child0[i], tv.child1[i]):
            if c >= 0:
                lo[i] = min(lo[i], lo[c])
    ids = np.arange(lo[s], s + 1)
    start = int(tv.sep_begin[lo[s]])
    end = int(tv.sep_end[s])
    U = tv.upd(s).astype(np.int64)
    nin = end - start
    n_s = nin + len(U)

    def loc(v):
        v = np.asarray(v, np.int64)
        out = np.where((v >= start) & (v < end), v - start, -1)
        if len(U):
            pos = np.searchsorted(U, v)
            hit = (pos < len(U)) & (U[np.minimum(pos, len(U) - 1)] == v)
            out = np.where(hit, nin + pos, out)
        return out
    ptr, ind, val = tv.ptr, tv.ind, tv.val
    rows = np.concatenate([np.arange(start, end), U])
    sind, sval, rows_ptr = [], [], [0]
    for r in rows:
        cols = ind[ptr[r]:ptr[r + 1]]
        lc = loc(cols)
        keep = lc >= 0
        sind.append(lc[keep])
        sval.append(val[ptr[r]:ptr[r + 1]][keep])
        rows_ptr.append(rows_ptr[-1] + int(keep.sum()))
    sptr = np.array(rows_ptr, np.int32)
    sind = np.concatenate(sind).astype(np.int32)
    sval = np.concatenate(sval)
    off = lo[s]
    m_ids = len(ids)
    remap = lambda v: np.where(v >= 0, v - off, -1).astype(np.int32)  # noqa: E731
    par = remap(tv.parent[ids])
    par[-1] = m_ids + 1  # the synthetic root; an empty leaf is its second child
    upd = [loc(tv.upd(i)).astype(np.int32) for i in ids] + [np.zeros(0, np.int32)] * 2
    up = np.zeros(m_ids + 3, np.int32)
    for q, u in enumerate(upd):
        up[q + 1] = up[q] + len(u)
    pieces = dict(n=n_s, ptr=sptr, ind=sind, val=sval,
                  sep_begin=np.concatenate([tv.sep_begin[ids] - start, [nin, nin]]).astype(np.int32),
                  sep_end=np.concatenate([tv.sep_end[ids] - start, [nin, n_s]]).astype(np.int32),
                  child0=np.concatenate([remap(tv.child0[ids]), [-1, m_ids - 1]]).astype(np.int32),
                  child1=np.concatenate([remap(tv.child1[ids]), [-1, m_ids]]).astype(np.int32),
                  parent=np.concatenate([par, [m_ids + 1, -1]]).astype(np.int32),
                  upd_ptr=up, upd_ind=np.concatenate(upd))
    nh = int(want[ids].sum())
    desc = (f"subtree of front {s} (level {tv.level[s]}, m={m[s]}, {m_ids} fronts, {nh} HSS "
            f"fronts, n={nin}) + a dense root over its {len(U)} update indices")
    return pieces, ids, desc


def run_reference_sample(cfg, pieces, threads):
    from oracle import ref
    ref.set_threads(threads)
    o = ref.ordered_from_arrays(pieces["n"], pieces["ptr"], pieces["ind"], pieces["val"],
                                pieces["sep_begin"], pieces["sep_end"], pieces["child0"],
                                pieces["child1"], pieces["parent"], pieces["upd_ptr"],
                                pieces["upd_ind"])
    b = ref_rhs(pieces["ptr"], pieces["ind"], pieces["val"], pieces["n"])
    mode = {"auto": 0, "mf": 1, "mf-hss": 2}[cfg.mode]
    t0 = time.perf_counter()
    F = ref.Factors(o, eps=cfg.eps, ls=cfg.ls, leaf=cfg.leaf, d0=cfg.d0, dd=cfg.dd, p=cfg.p,
                    min_hss=cfg.min_hss, mode=mode)
    F.solve(b)
    t = time.perf_counter() - t0
    # the reference's own per-front cost model of what it actually did on the
    # sample (FrontStat.flops, multifrontal.hpp:432-445), the synthetic root
    # included: it is timed too (and is an HSS front when nu(s) >= min_hss)
    return t, float(F.flops.astype(np.float64).sum()), int(F.hss_fronts)


def ref_rhs(ptr, ind, val, n):
    from paper_1502_07405_b200.problems import csr_matvec, x_true  # numpy only
    return csr_matvec(ptr, ind, val, x_true(n, 1))


def reference_scaled(cfg, tv, threads, steps, warmup, budget_s, full_model=None):
    """Time the reference on a sample of the workload and scale it by the
    ratio of the full workload's model cost to the sample's (reference-
    reported) model cost. The warm-up runs (at least one) time the cheapest
    HSS-rooted subtree; the timed sample is then the largest HSS-rooted
    subtree whose predicted time (at the warm-up's model rate) fits
    budget_s / steps, so the whole arm stays within about budget_s."""
    full, src = front_model(tv, cfg)
    if full_model is not None:  # per-front costs supplied by the caller
        full, src = np.asarray(full_model, np.float64), "caller's per-front model"
    cands = sample_candidates(tv, cfg)
    p0, _, _ = subtree_sample(tv, cfg, cands[0][1])
    rate = None
    for _ in range(max(1, warmup)):
        tw, fw, _ = run_reference_sample(cfg, p0, threads)
        rate = fw / max(tw, 1e-6)
    per_step = budget_s / max(1, steps)
    pick = cands[0][1]
    for cost, s_ in cands:
        if cost / rate <= per_step:
            pick = s_
    pieces, ids, desc = subtree_sample(tv, cfg, pick)
    runs = [run_reference_sample(cfg, pieces, threads) for _ in range(steps)]
    t = float(np.mean([r[0] for r in runs]))
    sfl = runs[0][1]
    scale = float(full.sum()) / sfl
    desc += (f"; {runs[0][2]} HSS fronts factored by the reference in the sample; measured "
             f"{t:.3f} s per sample (mean of {steps}), scaled x{scale:.2f} by the reference's "
             f"per-front cost model (full workload from the {src}); sample picked for a "
             f"{budget_s:.0f} s arm budget from a warm-up rate of {rate / 1e9:.2f} model GF/s")
    return t * scale, t, scale, desc


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def reference_arm(args, cfg):
    from oracle import ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    o = oracle_ordered(cfg)
    tv = TreeView.of_oracle(o)
    thr = cpu_threads()
    scaled, t, scale, desc = reference_scaled(cfg, tv, thr, args.steps, args.warmup,
                                              args.ref_budget_s)
    line = {
        "metric": METRIC, "value": scaled, "unit": "s", "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": scaled * 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": config_json(cfg, None, args, n=o.n, nnz=len(o.ind), fronts=o.nnodes),
        "cpu_baseline": {"value": scaled, "unit": "s", "cores": thr, "kind": "reference",
                         "sample": desc},
        "e2e": {"value": scaled, "unit": "s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    line.update(full_reference_run(cfg))
    print(json.dumps(line))


def full_reference_run(cfg):
    """the committed full reference run of the workload, if any (validation
    of the scaled sample)"""
    from paper_1502_07405_b200.problems import CONFIGS
    key = [k for k, v in CONFIGS.items() if v is cfg]
    path = os.path.join(ROOT, "tests", "golden", f"ref_{key[0]}.npz") if key else ""
    if not path or not os.path.exists(path):
        return {}
    g = np.load(path)
    return {"reference_full_run": {
        "factor_s": float(g["factor_s"]), "solve_s": float(g["solve_s"]),
        "threads": int(g["threads"]), "relres": float(g["relres"]), "flops": int(g["flops"]),
        "host": str(g["host"]) if "host" in g else None,
        "source": f"tests/golden/{os.path.basename(path)} (tests/golden/make_golden.py)"}}


def _metric():
    # the headline metric exactly as BASELINE.json names it
    try:
        with open(os.path.join(ROOT, "BASELINE.json")) as f:
            return json.load(f)["metric"]
    except Exception:
        return "factor+solve time (s), FP64 TFLOP/s & HBM GB/s vs peak; 3D Poisson 128^3, 1-8 GPU"


METRIC = _metric()


def config_json(cfg, op, args, n=None, nnz=None, fronts=None):
    if op is not None:
        n, nnz, fronts = op.a.size(), op.a.nnz(), op.t.size()
    return {"workload": cfg.name, "n": n, "nnz": nnz, "fronts": fronts,
            "nd_leaf": cfg.nd_leaf, "hss": {"ls": cfg.ls, "min_hss": cfg.min_hss,
                                            "eps": cfg.eps, "leaf": cfg.leaf, "mode": cfg.mode},
            "parallelism": f"subtree{args.gpus}" if args.gpus > 1 else "single",
            "l2": "inputs > L2 (factor storage tens of GB), no flush needed"}


def reference_counted(cfg, ms):
    """the reference's own counters::flops of its full run of this workload
    (counters.hpp:15-42, tests/golden/ref_<config>.npz) over this step's time:
    the reference-counted algorithmic rate of the GPU step"""
    from paper_1502_07405_b200.problems import CONFIGS
    key = [k for k, v in CONFIGS.items() if v is cfg]
    path = os.path.join(ROOT, "tests", "golden", f"ref_{key[0]}.npz") if key else ""
    if not path or not os.path.exists(path):
        return {}
    f = float(np.load(path)["flops"])
    return {"reference_counters_flops": f,
            "reference_counters_tflops": f / (ms * 1e-3) / 1e12,
            "reference_counters_note": "counters::flops of the reference's full run (factor "
                                       "only) / this step's factor+solve time"}


def spawn_ranks(n, dry):
    """re-exec this command under torch.distributed.run with n local ranks;
    returns the launcher's exit code"""
    import socket
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    env = dict(os.environ)
    if not dry:
        env.setdefault("NCCL_DEBUG", "INFO")  # NVLS / transport choice on stderr
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def dry_run(args, cfg, world, rank):
    """gloo, CPU: the ranks the GPU run would launch, the subtree partition of
    the workload and the phased factor/solve protocol (parallel.protocol_check)
    with a stand-in engine; prints the JSON line shape with n_gpus = world"""
    import torch.distributed as dist
    from paper_1502_07405_b200.parallel import TorchTransport, protocol_check, subtree_partition
    if world > 1:
        dist.init_process_group("gloo")
    op = build_problem(cfg)
    part = subtree_partition(op.t, world)
    ok = protocol_check(op.t, part, rank, TorchTransport(None)) if world > 1 else True
    oks = [ok]
    if world > 1:
        import torch
        tt = torch.tensor([1 if ok else 0])
        dist.all_reduce(tt, op=dist.ReduceOp.MIN)
        oks = [bool(tt.item())]
    if rank == 0:
        cj = config_json(cfg, op, args)
        cj["parallelism"] = f"subtree{world}" if world > 1 else "single"
        print(json.dumps({"metric": METRIC, "value": None, "unit": "s", "n_gpus": world,
                          "dry_run": True, "protocol_ok": oks[0], "steps": args.steps,
                          "warmup": args.warmup, "config": cj,
                          "partition": {"level": part.level, "edges": len(part.edges),
                                        "update_bytes": part.factor_bytes()}}))
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget-s", type=float, default=150.0,
                    help="--impl reference: seconds of timed reference work in total "
                         "(the sample is sized to fit budget / steps)")
    ap.add_argument("--gmres", action="store_true",
                    help="also run GMRES(30) preconditioned by the timed factors (informational)")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU only: launch the ranks over gloo and run the phased multi-GPU "
                         "protocol with a stand-in engine (no GPU work, no timing)")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        # `python bench.py --gpus N` outside torchrun: launch the N ranks here
        # (one process per GPU, the driver's own torchrun command line)
        sys.exit(spawn_ranks(args.gpus, args.dry_run))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    from paper_1502_07405_b200.problems import CONFIGS
    cfg = CONFIGS[args.config]

    if args.impl == "reference":
        if rank != 0:
            return
        reference_arm(args, cfg)
        return
    if args.dry_run:
        dry_run(args, cfg, world, rank)
        return

    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    import paper_1502_07405_b200 as P
    from paper_1502_07405_b200 import _native
    from paper_1502_07405_b200.problems import csr_matvec, x_true

    op = build_problem(cfg)
    n = op.a.size()
    ptr, ind, val = op.a.arrays()
    b = csr_matvec(ptr, ind, val, x_true(n, 1))
    opts = cfg.solver_options()
    peaks = measured_peaks(torch, dev)

    b_dev = torch.from_numpy(b).to(dev)
    x_dev = torch.empty_like(b_dev)
    dist_mode = world > 1
    if dist_mode:
        # subtree-to-GPU partition: rank r factors its subtree
        # and the top fronts it owns; updates / bupd / x(upd) cross GPUs over
        # NCCL point-to-point at the subtree roots only
        from paper_1502_07405_b200.parallel import DistributedMf, TorchTransport
        m = DistributedMf(op.a, op.t, opts, world, rank=rank, transport=TorchTransport(dev),
                          device=local)
        eng = m.engines[rank].m
        xs = {rank: x_dev.view(1, n)}

        def step():
            m.factor()
            x_dev.copy_(b_dev)
            torch.cuda.current_stream(dev).synchronize()
            m.solve_device(xs)
    else:
        # first factorization (upload + schedule + numeric)
        m = P.mf_factor(op.a, op.t, opts, device=local)
        eng = m

        def step():
            m.refactor()
            x_dev.copy_(b_dev)
            torch.cuda.current_stream(dev).synchronize()
            m.solve_device(x_dev.data_ptr(), n, 1)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    l0 = _native.lib().hssmf_launch_count()
    t0 = time.perf_counter()
    dev_ms = 0.0
    solve_ms = []
    for _ in range(args.steps):
        step()
        f, s = eng.timing()
        dev_ms += f + s
        solve_ms.append(s)
    barrier()
    t1 = time.perf_counter()
    launches = (_native.lib().hssmf_launch_count() - l0) // args.steps
    factor_nnz_val = float(eng.factor_nnz()) if not dist_mode else 0.0
    ck = clocks.stop()
    ms = (t1 - t0) / args.steps * 1e3
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())

    # correctness of the timed factors (relative residual); multi-GPU: every
    # rank holds its own separators, summed once into the full solution
    if dist_mode:
        xc = m.combine(xs)
        dist.all_reduce(xc)
        x = xc.view(-1).cpu().numpy()
    else:
        x = x_dev.cpu().numpy()
    relres = float(np.linalg.norm(op.a.matvec(x) - b) / np.linalg.norm(b))
    # the paper's use of the compressed factors: preconditioner of restarted
    # GMRES (krylov.hpp:93-184), everything on the device; informational, not
    # part of the timed metric
    gm = None
    if args.gmres and not dist_mode:
        tg = time.perf_counter()
        xg, rep = P.gmres(op.a, m, b, restart=30, rtol=1e-10, atol=0.0, maxit=300)
        tg = time.perf_counter() - tg
        gm = {"restart": 30, "rtol": 1e-10, "iterations": rep.iterations,
              "converged": rep.converged,
              "relres": float(np.linalg.norm(op.a.matvec(xg) - b) / np.linalg.norm(b)),
              "wall_s": round(tg, 3)}

    # e2e through the public API: factor from the host CSR + solve of host b
    del m, eng
    torch.cuda.empty_cache()
    barrier()
    e0 = time.perf_counter()
    for _ in range(max(1, min(args.steps, 2))):
        if dist_mode:
            md = DistributedMf(op.a, op.t, opts, world, rank=rank, transport=TorchTransport(dev),
                               device=local)
            md.factor()
            xl = md.solve(b)
            xt = torch.from_numpy(np.ascontiguousarray(xl)).to(dev)
            dist.all_reduce(xt)
            xh = xt.cpu().numpy()
            del md
        else:
            md = P.mf_factor(op.a, op.t, opts, device=local)
            xh = P.mf_solve_new(md, b)
            del md
    barrier()
    e_ms = (time.perf_counter() - e0) / max(1, min(args.steps, 2)) * 1e3
    h2d = int(ptr.nbytes + ind.nbytes + val.nbytes + b.nbytes)
    d2h = int(xh.nbytes)

    # per-kernel-class profile pass (events around each launch)
    # HSS fronts of a level normally run concurrently on several streams; the
    # profiled step runs them one at a time so per-class device times add up
    # (multi-GPU: rank 0's share of a partitioned step)
    os.environ["HSSMF_HSS_STREAMS"] = "1"
    if dist_mode:
        mp_ = DistributedMf(op.a, op.t, opts, world, rank=rank, transport=TorchTransport(dev),
                            device=local)
        ep = mp_.engines[rank].m
        ep.set_profile(True)
        ep.reset_kernel_stats()
        mp_.factor()
        x_dev.copy_(b_dev)
        mp_.solve_device({rank: x_dev.view(1, n)})
    else:
        ep = P.mf_factor(op.a, op.t, opts, device=local)
        ep.set_profile(True)
        ep.reset_kernel_stats()
        P.api.probe_read()
        P.api.probe_enable(True)
        ep.refactor()
        ep.solve_device(x_dev.data_ptr(), n, 1)
    probes = P.api.probe_read()
    P.api.probe_enable(False)
    ks = ep.kernel_stats()
    ep.set_profile(False)
    os.environ.pop("HSSMF_HSS_STREAMS", None)
    # hss_front_total wraps the hss_* phases: keep the leaves of the breakdown
    ks = [k for k in ks if k["name"] != "hss_front_total"]
    tot_ms = sum(k["ms"] for k in ks) or 1.0
    # roofline of the dominant kernel: per-launch CUDA events on the launching
    # stream (probes) with the launch's algorithmic flops / bytes
    roofs = []
    for name, pr in probes.items():
        if not pr["launches"] or pr["ms"] <= 0:
            continue
        e = {"kernel": name, "launches": pr["launches"], "ms": round(pr["ms"], 2),
             "avg_launch_us": round(1e3 * pr["ms"] / pr["launches"], 2),
             "share_of_step": pr["ms"] / tot_ms}
        if pr["flops"] > 0:
            ach = pr["flops"] / (pr["ms"] * 1e-3) / 1e12
            e.update(bound="tensor", achieved=ach, peak=peaks["fp64_tflops"], unit="TFLOP/s",
                     frac=ach / peaks["fp64_tflops"], peak_src=peaks["fp64_src"],
                     algorithmic="2mnk per GEMM (mnk for lower-triangle SYRK updates)")
            if pr["bytes"] > 0:
                # A and B read once, C written (beta 0) or read + written
                e.update(algorithmic_bytes_per_launch=pr["bytes"] / pr["launches"],
                         flop_per_byte=pr["flops"] / pr["bytes"],
                         hbm_gbs_at_algorithmic_bytes=pr["bytes"] / (pr["ms"] * 1e-3) / 1e9)
        elif pr["bytes"] > 0:
            ach = pr["bytes"] / (pr["ms"] * 1e-3) / 1e9
            e.update(bound="hbm", achieved=ach, peak=peaks["hbm_gbs"], unit="GB/s",
                     frac=ach / peaks["hbm_gbs"], peak_src=peaks["hbm_src"],
                     algorithmic="16 B per lower-triangle Gram element per panel (read + write)")
        else:
            # a panel launch runs at most 48 dependent pivot steps
            e.update(bound="latency", us_per_pivot_step=round(e["avg_launch_us"] / 48, 3),
                     note="pivot chain: one cluster-wide argmax per elimination step; "
                          "us_per_pivot_step = avg launch / 48 steps (an upper bound when "
                          "tasks stop inside a panel)")
        e["traffic"] = TRAFFIC.get(name)
        roofs.append(e)
    # the assembly kernels (north_star (1)): bracketed per level by CUDA events on
    # the engine stream, algorithmic bytes from the analysis (extend-add:
    # 24 B per child update entry + 4 B per child row)
    for k in ks:
        # (the sparse assembly's bytes are mostly the level's zeroing memsets:
        # write-only traffic, which runs above the copy peak; it stays in `kernels`)
        if k["name"] == "extend_add" and k["ms"] > 0 and k["bytes"] > 0:
            ach = k["bytes"] / (k["ms"] * 1e-3) / 1e9
            roofs.append({"kernel": k["name"], "launches": k["launches"], "ms": round(k["ms"], 2),
                          "avg_launch_us": round(1e3 * k["ms"] / k["launches"], 2),
                          "share_of_step": k["ms"] / tot_ms, "bound": "hbm", "achieved": ach,
                          "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": ach / peaks["hbm_gbs"],
                          "peak_src": peaks["hbm_src"],
                          "algorithmic": "24 B per child update entry (read it, read and write its "
                                         "target) + 4 B of position map per child row",
                          "traffic": TRAFFIC.get(k["name"])})
    roofs.sort(key=lambda e: -e["ms"])
    dom = [e for e in roofs if e.get("bound") in ("tensor", "hbm")]
    roof = dict(dom[0]) if dom else {"kernel": None}
    flops_total = sum(k["flops"] for k in ks)
    # the reference's own per-front cost model over the fronts this run
    # factored (FrontStat.flops, multifrontal.hpp:389-396, 432-445: dense
    # 2ns^3/3 + 2ns^2 nu + 2ns nu^2, HSS 4 m^2 d_final + 8 m r^2 with this run's
    # ranks and d_final): the algorithmic work of the step beside the executed
    # flops (which include the dense-front sampling and densified updates the
    # reference does not perform)
    model_flops = float(np.asarray(ep.flops, np.float64).sum()) if hasattr(ep, "flops") else None

    # the solve's HBM roofline: every stored factor scalar is read once per
    # solve (the forward sweep reads L / L21 and the ULV lower factors, the
    # backward sweep U / U12 and the upper ones): 8 B x factor_nnz (the
    # reference's own count, multifrontal.hpp:463-467), plus the solution
    # vector read and written once per sweep (2 x 16 B x n)
    solve_entry = None
    if not dist_mode and solve_ms:
        fb = 8.0 * factor_nnz_val + 32.0 * n
        sm = float(np.median(solve_ms))
        if fb > 0 and sm > 0:
            ach = fb / (sm * 1e-3) / 1e9
            solve_entry = {"ms": round(sm, 3), "algorithmic_bytes": fb, "achieved": ach,
                           "unit": "GB/s", "peak": peaks["hbm_gbs"], "frac": ach / peaks["hbm_gbs"],
                           "note": "8 B x factor_nnz (each stored scalar read once over the "
                                   "two sweeps) + 32 B x n (x read + written per sweep)"}
    line = {
        "metric": METRIC, "value": ms / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_json(cfg, op, args),
        "device_ms_per_step": dev_ms / args.steps,
        "relres": relres,
        "gmres_preconditioned": gm,
        "fp64_tflops_step": flops_total / (ms * 1e-3) / 1e12,
        "flops_per_step": dict({"executed": flops_total, "reference_front_model": model_flops,
                                "reference_model_tflops": (model_flops / (ms * 1e-3) / 1e12
                                                           if model_flops else None)},
                               **reference_counted(cfg, ms)),
        "e2e": {"value": e_ms / 1e3, "unit": "s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": int(launches),
        "clocks": ck,
        "roofline": roof,
        "rooflines": roofs,
        "solve_roofline": solve_entry,
        "kernels": [{k2: (round(v, 4) if isinstance(v, float) else v) for k2, v in k.items()}
                    for k in ks if k["launches"]],
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import ref
            if ref.available():
                thr = cpu_threads()
                tv = TreeView.of_oracle(oracle_ordered(cfg))
                scaled, t, scale, desc = reference_scaled(cfg, tv, thr, 1, 1, 30.0)
                line["cpu_baseline"] = {"value": scaled, "unit": "s", "cores": thr,
                                        "kind": "reference", "sample": desc}
                line["cpu_baseline"].update(full_reference_run(cfg))
        except Exception as e:  # reported, never fatal for the GPU arm
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
