"""Generate golden fixtures from the reference (oracle/_ref) for the BASELINE
configs: per-front stats, per-HSS-node ranks, relres, timings and (for the
smaller configs) the solution. Runs in the build container, where
/root/reference exists; the .npz files are committed so the GPU box needs no
reference at run time.

usage: python tests/golden/make_golden.py c1 c1_mf c3 c4 c5 [--threads N] [--out-dir D]

c5 (P3D 128^3) needs more host RAM than the build container has (OOM at 65 GB);
it is run on the GPU-box host (tools/ref_c5_box.sh) and the .npz brought back.
"""
import argparse
import os
import resource
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402
from paper_1502_07405_b200.problems import CONFIGS, csr_matvec, x_true  # noqa: E402


def ordered(cfg):
    if cfg.kind == "cd3d":
        import paper_1502_07405_b200 as P  # product generator: config 4 is not a ref generator
        g = P.generate_convdiff3d(cfg.k, 0.1)
        ptr, ind, val = g.A.arrays()
        return ref.ordered_csr_geom(ptr, ind, val, (cfg.k,) * 3, 3, cfg.nd_leaf)
    return ref.ordered_grid(cfg.kind, cfg.k, cfg.nd_leaf)


def host_info():
    info = {"cpu_count": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    info["cpu_model"] = line.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as f:
            info["mem_total_kb"] = int(f.readline().split()[1])
    except OSError:
        pass
    return info


def run_dense(name, cfg, threads, out_dir):
    """BASELINE config 2: standalone dense HSS (hss_compress.hpp:373-383 +
    ulv_factor / UlvFactors::solve) on A_ij = 1/(1+|i-j|) + 4 delta_ij"""
    from paper_1502_07405_b200.problems import dense_c2
    ref.set_threads(threads)
    a = dense_c2(cfg.k)
    h = ref.DenseHss(a, leaf=cfg.leaf, eps=cfg.eps, d0=cfg.d0, dd=cfg.dd, p=cfg.p)
    b = x_true(cfg.k, 1)
    x = h.solve(b)[:, 0]
    relres = np.linalg.norm(a @ x - b) / np.linalg.norm(b)
    out = dict(name=name, n=cfg.k, threads=threads, u_rank=h.u_rank, v_rank=h.v_rank,
               rounds=h.rounds, d_final=h.d_final, compress_s=h.t_compress, ulv_s=h.t_ulv,
               relres=relres, x=x, host=str(host_info()))
    np.savez_compressed(os.path.join(out_dir, f"ref_{name}.npz"), **out)
    print(f"{name}: compress {h.t_compress:.2f}s ulv {h.t_ulv:.3f}s rounds {h.rounds} d_final "
          f"{h.d_final} max rank {int(h.u_rank[:-1].max())} relres {relres:.3e}", flush=True)


def run(name, threads, out_dir):
    cfg = CONFIGS[name]
    if cfg.kind == "dense":
        return run_dense(name, cfg, threads, out_dir)
    ref.set_threads(threads)
    t0 = time.time()
    o = ordered(cfg)
    t_an = time.time() - t0
    b = csr_matvec(o.ptr, o.ind, o.val, x_true(o.n, 1))
    mode = {"auto": 0, "mf": 1, "mf-hss": 2}[cfg.mode]
    ref.lib().ref_reset_counters()
    F = ref.Factors(o, eps=cfg.eps, ls=cfg.ls, leaf=cfg.leaf, d0=cfg.d0, dd=cfg.dd, p=cfg.p,
                    min_hss=cfg.min_hss, mode=mode)
    flops = ref.lib().ref_flops()
    x = F.solve(b)[:, 0]
    import scipy.sparse as sp
    A = sp.csr_matrix((o.val, o.ind, o.ptr), shape=(o.n, o.n))
    relres = np.linalg.norm(A @ x - b) / np.linalg.norm(b)
    hss = [i for i in range(o.nnodes) if F.type[i] == 1]
    node_u, node_v, node_ptr, rounds, dfin = [], [], [0], [], []
    for i in hss:
        u, v, r, d = F.front_hss(i)
        node_u.append(u)
        node_v.append(v)
        node_ptr.append(node_ptr[-1] + len(u))
        rounds.append(r)
        dfin.append(d)
    out = dict(
        name=name, n=o.n, nnodes=o.nnodes, threads=threads, analysis_s=t_an,
        factor_s=F.factor_seconds, solve_s=F.solve_seconds, flops=flops, relres=relres,
        hss_fronts=F.hss_fronts, fallbacks=F.fallbacks, max_front_rank=F.max_front_rank,
        factor_nnz=F.factor_nnz, rank=F.rank, type=F.type, level=F.level, dim=F.dim,
        hss_ids=np.array(hss, np.int32),
        node_ptr=np.array(node_ptr, np.int32),
        node_u=np.concatenate(node_u) if node_u else np.zeros(0, np.int32),
        node_v=np.concatenate(node_v) if node_v else np.zeros(0, np.int32),
        rounds=np.array(rounds, np.int32), d_final=np.array(dfin, np.int32),
        perm_sum=np.int64((o.perm.astype(np.int64) * np.arange(o.n)).sum()),
        peak_rss_kb=resource.getrusage(resource.RUSAGE_SELF).ru_maxrss,
        host=str(host_info()),
    )
    if o.n <= 300000:
        out["x"] = x
    path = os.path.join(out_dir, f"ref_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: factor {F.factor_seconds:.2f}s solve {F.solve_seconds:.3f}s relres "
          f"{relres:.3e} hss {F.hss_fronts} maxrank {F.max_front_rank} flops {flops:.3e}",
          flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--out-dir", default=os.path.join(ROOT, "tests", "golden"))
    a = ap.parse_args()
    print(host_info(), flush=True)
    for c in a.configs:
        run(c, a.threads, a.out_dir)
