"""Run statistics in the reference's report formats (schema version 1 JSON and
the one-line CSV; reference stats.hpp / src/stats.cpp:37-123), filled from a
device factorization (MfFactors) and its solve."""
from __future__ import annotations

import json
from dataclasses import dataclass, field

CSV_FIELDS = ("source,strategy,mode,n,nnz,ls,eps,leaf,d0,dd,p,min_hss,rank_guard,threads,rtol,"
              "atol,restart,maxit,nd_leaf,analysis_s,factor_s,solve_s,total_s,factor_flops,"
              "solve_flops,factor_nnz,factor_nnz_bytes,peak_bytes,max_rank,fronts,hss_fronts,"
              "hss_fallbacks,tree_depth,method,iterations,relres,absres,converged,error")


@dataclass
class RunStats:
    source: str = ""
    strategy: str = "geometric"
    mode: str = "auto"
    n: int = 0
    nnz: int = 0
    ls: int = 0
    eps: float = 0.0
    leaf: int = 0
    d0: int = 0
    dd: int = 0
    p: int = 0
    min_hss: int = 0
    rank_guard: int = 0
    threads: int = 1
    rtol: float = 1e-6
    atol: float = 1e-10
    restart: int = 30
    maxit: int = 500
    nd_leaf: int = 0
    t_analysis: float = 0.0
    t_factor: float = 0.0
    t_solve: float = 0.0
    t_total: float = 0.0
    factor_flops: int = 0
    solve_flops: int = 0
    factor_nnz: int = 0
    factor_nnz_bytes: int = 0
    peak_bytes: int = 0
    max_rank: int = 0
    fronts: int = 0
    hss_fronts: int = 0
    hss_fallbacks: int = 0
    tree_depth: int = 0
    method: str = "direct"
    iterations: int = 0
    relres: float = 0.0
    absres: float = 0.0
    converged: bool = True
    error: str = ""
    per_front: list = field(default_factory=list)


def run_stats(m, opts, a, source="", t_analysis=0.0, relres=0.0, absres=0.0, method="direct",
              iterations=0, converged=True, threads=1):
    """RunStats of a factorization m (MfFactors) of a with SolverOptions opts;
    times are the device factor/solve times of m's last calls"""
    tf, tsv = m.timing()
    n = m.n
    rg = opts.max_rank if opts.max_rank > 0 else min(n // 2, 5000)
    return RunStats(
        source=source, mode=opts.mode, n=n, nnz=a.nnz(), ls=opts.ls, eps=opts.eps,
        leaf=opts.leaf, d0=opts.d0, dd=opts.dd, p=opts.p, min_hss=opts.min_hss, rank_guard=rg,
        threads=threads, nd_leaf=opts.nd_leaf, t_analysis=t_analysis, t_factor=tf * 1e-3,
        t_solve=tsv * 1e-3, t_total=t_analysis + (tf + tsv) * 1e-3,
        factor_flops=int(m.flops.sum()), factor_nnz=int(m.factor_nnz()),
        factor_nnz_bytes=8 * int(m.factor_nnz()), peak_bytes=int(m.device_bytes()),
        max_rank=m.max_front_rank, fronts=len(m.level), hss_fronts=m.hss_fronts,
        hss_fallbacks=m.fallbacks, tree_depth=int(m.level.max(initial=0)) + 1, method=method,
        iterations=iterations, relres=relres, absres=absres, converged=converged,
        per_front=[dict(id=f.id, level=f.level, dim=f.dim, sep=f.sep, rank=f.rank,
                        flops=f.flops, type=f.type) for f in m.front_stats])


def stats_to_json(s: RunStats, include_per_front: bool = True) -> str:
    """schema_version 1 (stats.cpp:37-83); keys sorted as nlohmann::json emits them"""
    j = {
        "schema_version": 1,
        "config": {"source": s.source, "strategy": s.strategy, "mode": s.mode, "n": s.n,
                   "nnz": s.nnz, "ls": s.ls, "eps": s.eps, "leaf": s.leaf, "d0": s.d0,
                   "dd": s.dd, "p": s.p, "min_hss": s.min_hss, "rank_guard": s.rank_guard,
                   "threads": s.threads, "rtol": s.rtol, "atol": s.atol, "restart": s.restart,
                   "maxit": s.maxit, "nd_leaf": s.nd_leaf},
        "timings": {"analysis": s.t_analysis, "factor": s.t_factor, "solve": s.t_solve,
                    "total": s.t_total},
        "factor": {"factor_flops": s.factor_flops, "solve_flops": s.solve_flops,
                   "factor_nnz": s.factor_nnz, "factor_nnz_bytes": s.factor_nnz_bytes,
                   "peak_bytes": s.peak_bytes, "max_rank": s.max_rank, "fronts": s.fronts,
                   "hss_fronts": s.hss_fronts, "hss_fallbacks": s.hss_fallbacks,
                   "tree_depth": s.tree_depth},
        "solve": {"method": s.method, "iterations": s.iterations, "relres": s.relres,
                  "absres": s.absres, "converged": s.converged},
    }
    if s.error:
        j["error"] = s.error
    if include_per_front:
        j["per_front"] = [dict(f) for f in s.per_front]
    return json.dumps(j, indent=1, sort_keys=True) + "\n"


def _g(v):
    return "%.17g" % v


def _q(s):
    if not any(c in s for c in ',"\n'):
        return s
    return '"' + s.replace('"', '""') + '"'


def stats_csv_header() -> str:
    return CSV_FIELDS


def stats_csv_row(s: RunStats) -> str:
    """stats.cpp:107-121, %.17g for reals, RFC-4180 quoting"""
    vals = [_q(s.source), s.strategy, s.mode, s.n, s.nnz, s.ls, _g(s.eps), s.leaf, s.d0, s.dd,
            s.p, s.min_hss, s.rank_guard, s.threads, _g(s.rtol), _g(s.atol), s.restart, s.maxit,
            s.nd_leaf, _g(s.t_analysis), _g(s.t_factor), _g(s.t_solve), _g(s.t_total),
            s.factor_flops, s.solve_flops, s.factor_nnz, s.factor_nnz_bytes, s.peak_bytes,
            s.max_rank, s.fronts, s.hss_fronts, s.hss_fallbacks, s.tree_depth, s.method,
            s.iterations, _g(s.relres), _g(s.absres), 1 if s.converged else 0, _q(s.error)]
    return ",".join(str(v) for v in vals)
