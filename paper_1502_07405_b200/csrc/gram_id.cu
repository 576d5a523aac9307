#include "gram_id.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <climits>

#include "gemm.cuh"

namespace hssmf_b200 {

  namespace {
    namespace cg = cooperative_groups;
    constexpr int GT = 256, GW = GT / 32, NB = kGramNB;

    struct Cand {
      double v;
      int pos, idx;
    };
    __device__ __forceinline__ bool better(double v, int p, double bv, int bp) {
      return v > bv || (v == bv && p < bp);
    }

    // nb steps of symmetric pivoted Cholesky on the Gram matrix for every
    // task; one thread-block cluster per task, rows of the task split into
    // contiguous blocks over the CTAs of the cluster
    __global__ void __launch_bounds__(GT)
    gram_panel_kernel(const GramTask* __restrict__ tasks, int k0, int nb, double eps,
                      double abs_tol, int CL, int init) {
      cg::cluster_group cl = cg::this_cluster();
      const int rank = (int)cl.block_rank();
      const GramTask T = tasks[blockIdx.x / CL];
      const int n = T.n;
      const int rows = (n + CL - 1) / CL;
      const int r0 = rank * rows, r1 = min(n, r0 + rows);
      const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
      __shared__ Cand pub;
      __shared__ double wv[GW];
      __shared__ int wp[GW], wi[GW];
      __shared__ int s_stop, s_pj, s_cert;
      __shared__ double s_ljj, s_r11;
      __shared__ double prow[NB];
      if (init) {
        for (int i = r0 + tid; i < r1; i += GT) {
          __stcg(T.dg + i, __ldcg(T.G + i + (size_t)i * n));
          __stcg(T.flag + i, 0);
          __stcg(T.orig_at + i, i);
          __stcg(T.pos_of + i, i);
        }
        if (rank == 0 && tid == 0) {
          __stcg(T.state + 0, 0);
          __stcg(T.state + 1, 0);
          __stcg(T.state + 2, 0);
        }
        cl.sync();
      }
      if (__ldcg(T.state + 1)) return;  // finished in an earlier panel
      if (n == 0 || T.kmax_dim == 0) {
        cl.sync();
        if (rank == 0 && tid == 0) {
          __stcg(T.state + 0, 0);
          __stcg(T.state + 1, 1);
          __stcg(T.state + 2, 1);
        }
        return;
      }
      int j = k0;
      int stopped = 0;
      for (int jj = 0; jj < nb; jj++, j++) {
        // (a) local candidate: largest residual norm, lowest position on ties
        double bv = -1.0;
        int bp = INT_MAX, bi = -1;
        for (int i = r0 + tid; i < r1; i += GT) {
          if (__ldcg(T.flag + i)) continue;
          const double v = __ldcg(T.dg + i);
          const int p = __ldcg(T.pos_of + i);
          if (better(v, p, bv, bp)) { bv = v; bp = p; bi = i; }
        }
        for (int o = 16; o > 0; o >>= 1) {
          const double v2 = __shfl_down_sync(0xffffffffu, bv, o);
          const int p2 = __shfl_down_sync(0xffffffffu, bp, o);
          const int i2 = __shfl_down_sync(0xffffffffu, bi, o);
          if (better(v2, p2, bv, bp)) { bv = v2; bp = p2; bi = i2; }
        }
        if (lane == 0) { wv[warp] = bv; wp[warp] = bp; wi[warp] = bi; }
        __syncthreads();
        if (tid == 0) {
          Cand c{wv[0], wp[0], wi[0]};
          for (int w = 1; w < GW; w++)
            if (better(wv[w], wp[w], c.v, c.pos)) c = {wv[w], wp[w], wi[w]};
          pub = c;
        }
        cl.sync();
        // (b) identical decision in every CTA (rrqr.hpp:62-77)
        if (tid == 0) {
          Cand c{-1.0, INT_MAX, -1};
          for (int r = 0; r < CL; r++) {
            const Cand* q = cl.map_shared_rank(&pub, r);
            if (better(q->v, q->pos, c.v, c.pos)) c = *q;
          }
          const double pv = c.v > 0.0 ? sqrt(c.v) : 0.0;
          int stop = 0, cert = 0;
          if (j == 0) {
            s_r11 = pv;
            if (pv == 0.0 || pv <= abs_tol) { stop = 1; cert = 1; }
          } else {
            s_r11 = __ldcg(T.r11);
            if (pv <= eps * s_r11 || pv <= abs_tol) { stop = 1; cert = 1; }
          }
          if (!stop && j == T.kmax) {
            stop = 1;
            cert = (j == T.kmax_dim);
          }
          s_stop = stop;
          s_cert = cert;
          s_pj = c.idx;
          s_ljj = pv;
        }
        __syncthreads();
        if (s_stop) {
          stopped = 1;
          break;
        }
        const int pj = s_pj;
        const double ljj = s_ljj;
        if (tid < jj) prow[tid] = __ldcg(T.L + pj + (size_t)(k0 + tid) * n);
        if (rank == 0 && tid == 0) {
          if (j == 0) __stcg(T.r11, s_r11);
          // CPQR column swap of positions j and pos(pj)
          const int pp = __ldcg(T.pos_of + pj);
          const int ok = __ldcg(T.orig_at + j);
          __stcg(T.orig_at + j, pj);
          __stcg(T.orig_at + pp, ok);
          __stcg(T.pos_of + pj, j);
          __stcg(T.pos_of + ok, pp);
          __stcg(T.flag + pj, 1);
          __stcg(T.L + pj + (size_t)j * n, ljj);
        }
        __syncthreads();
        // (c) column j of L on own rows; residual norms downdated (clamped at 0)
        const double* gcol = T.G + (size_t)pj * n;
        for (int i = r0 + tid; i < r1; i += GT) {
          if (i == pj || __ldcg(T.flag + i)) continue;
          double s = __ldcg(gcol + i);
          for (int q = 0; q < jj; q++) s -= __ldcg(T.L + i + (size_t)(k0 + q) * n) * prow[q];
          const double lo = s / ljj;
          __stcg(T.L + i + (size_t)j * n, lo);
          double d = __ldcg(T.dg + i) - lo * lo;
          if (d < 0.0) d = 0.0;
          __stcg(T.dg + i, d);
        }
        cl.sync();
        if (j + 1 == T.kmax_dim) {  // factorization exhausted exactly
          if (rank == 0 && tid == 0) {
            __stcg(T.state + 0, j + 1);
            __stcg(T.state + 1, 1);
            __stcg(T.state + 2, 1);
          }
          return;
        }
      }
      cl.sync();
      if (rank == 0 && tid == 0) {
        __stcg(T.state + 0, j);
        if (stopped) {
          __stcg(T.state + 1, 1);
          __stcg(T.state + 2, s_cert);
        }
      }
    }
  }  // namespace

  void gram_cholesky_run(const std::vector<GramTask>& tasks, double eps, double abs_tol,
                         cudaStream_t s, std::vector<int>& rank, std::vector<int>& cert,
                         double* flops) {
    const int nt = (int)tasks.size();
    rank.assign(nt, 0);
    cert.assign(nt, 0);
    if (!nt) return;
    static bool attr = false;
    if (!attr) {
      HSSMF_CUDA(cudaFuncSetAttribute(gram_panel_kernel,
                                      cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      attr = true;
    }
    int max_n = 0;
    for (const auto& t : tasks) max_n = std::max(max_n, t.n);
    int CL = 1;
    while (CL < 16 && max_n > CL * 256) CL *= 2;
    GramTask* d = nullptr;
    HSSMF_CUDA(cudaMallocAsync((void**)&d, nt * sizeof(GramTask), s));
    HSSMF_CUDA(cudaMemcpyAsync(d, tasks.data(), nt * sizeof(GramTask), cudaMemcpyHostToDevice, s));
    std::vector<int> hst(3 * nt);
    int kmax = 0;
    for (const auto& t : tasks) kmax = std::max(kmax, t.kmax);
    // all panels are queued without host round trips: a finished task's
    // panel kernel returns at once and its trailing GEMM is skipped on device
    for (int k0 = 0; k0 <= kmax; k0 += NB) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(nt * CL);
      cfg.blockDim = dim3(GT);
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CL;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      HSSMF_CUDA(cudaLaunchKernelEx(&cfg, gram_panel_kernel, (const GramTask*)d, k0, NB, eps,
                                    abs_tol, CL, k0 == 0 ? 1 : 0));
      HSSMF_LAUNCH_CHECK();
      if (k0 + NB > kmax) break;
      std::vector<GemmProblem> p;
      for (int t = 0; t < nt; t++) {
        const auto& T = tasks[t];
        if (k0 > T.kmax) continue;
        GemmProblem g{T.L + (size_t)k0 * T.n, T.L + (size_t)k0 * T.n, T.G, T.n, T.n, NB, T.n,
                      T.n, T.n};
        g.skip = T.state + 1;
        p.push_back(g);
      }
      if (flops) *flops += gemm_flops(p);
      gemm_run_host(p, 'N', 'T', -1.0, 1.0, s);
    }
    for (int t = 0; t < nt; t++)
      HSSMF_CUDA(cudaMemcpyAsync(&hst[3 * t], tasks[t].state, 3 * sizeof(int),
                                 cudaMemcpyDeviceToHost, s));
    HSSMF_CUDA(cudaStreamSynchronize(s));
    for (int t = 0; t < nt; t++) {
      rank[t] = hst[3 * t];
      cert[t] = hst[3 * t + 2];
    }
    HSSMF_CUDA(cudaFreeAsync(d, s));
  }

}  // namespace hssmf_b200
