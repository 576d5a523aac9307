#include "gram_id.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <climits>

#include "gemm.cuh"
#include "staging.cuh"

namespace hssmf_b200 {

  namespace {
    namespace cg = cooperative_groups;
    constexpr int GT = 256, GW = GT / 32;
    constexpr int kSmemCap = 200 * 1024;

    struct Cand {
      double v;
      int pos, idx;
    };
    __device__ __forceinline__ bool better(double v, int p, double bv, int bp) {
      return v > bv || (v == bv && p < bp);
    }

    // dynamic shared memory of one CTA (rows = own contiguous row block):
    //   Lp[nb * rows]  panel columns of own rows, column-major (double) so
    //                  that the per-row dot products of a warp hit distinct banks
    //   dg[rows]       residual norms^2 of own rows    (double)
    //   orig[n], pos[n] replicated position bookkeeping (int)
    //   flg[rows]      pivoted flags of own rows        (int)
    __host__ __device__ inline size_t gram_smem(int n, int rows, int nb) {
      return (size_t)rows * nb * 8 + (size_t)rows * 8 + (size_t)n * 8 + (size_t)rows * 4 + 64;
    }

    __device__ void block_cand(double bv, int bp, int bi, Cand* out, double* wv, int* wp, int* wi) {
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_down_sync(0xffffffffu, bv, o);
        const int p2 = __shfl_down_sync(0xffffffffu, bp, o);
        const int i2 = __shfl_down_sync(0xffffffffu, bi, o);
        if (better(v2, p2, bv, bp)) { bv = v2; bp = p2; bi = i2; }
      }
      if (lane == 0) { wv[warp] = bv; wp[warp] = bp; wi[warp] = bi; }
      __syncthreads();
      if (threadIdx.x == 0) {
        Cand c{wv[0], wp[0], wi[0]};
        for (int w = 1; w < GW; w++)
          if (better(wv[w], wp[w], c.v, c.pos)) c = {wv[w], wp[w], wi[w]};
        *out = c;
      }
    }

    // nb steps of symmetric pivoted Cholesky on the Gram matrix, one
    // thread-block cluster per task. Rows are split in contiguous blocks over
    // the CTAs; each CTA keeps its rows' panel columns, residual norms and
    // flags plus a replicated copy of the position bookkeeping in shared
    // memory, so one cluster barrier per elimination step suffices: the
    // candidates for step j+1 are published together with column j.
    __global__ void __launch_bounds__(GT)
    gram_panel_kernel(const GramTask* __restrict__ tasks, int k0, int nb, double eps,
                      double abs_tol, int CL, int init) {
      cg::cluster_group cl = cg::this_cluster();
      const int rank = (int)cl.block_rank();
      const GramTask T = tasks[blockIdx.x / CL];
      const int n = T.n;
      const int rows = (n + CL - 1) / CL;
      const int r0 = min(n, rank * rows), r1 = min(n, r0 + rows), nr = r1 - r0;
      const int tid = threadIdx.x;
      extern __shared__ double sm[];
      double* Lp = sm;
      double* dg = Lp + (size_t)rows * nb;
      int* orig = reinterpret_cast<int*>(dg + rows);
      int* pos = orig + n;
      int* flg = pos + n;
      __shared__ Cand pub[2];
      __shared__ double wv[GW];
      __shared__ int wp[GW], wi[GW];
      __shared__ int s_stop, s_pj, s_cert;
      __shared__ double s_ljj, s_r11;
      __shared__ double prow[64];

      if (__ldcg(T.state + 1) && !init) return;  // finished in an earlier panel
      // load / initialise the state
      if (init) {
        for (int i = tid; i < nr; i += GT) {
          dg[i] = T.G[(r0 + i) + (size_t)(r0 + i) * n];
          flg[i] = 0;
        }
        for (int i = tid; i < n; i += GT) { orig[i] = i; pos[i] = i; }
      } else {
        for (int i = tid; i < nr; i += GT) {
          dg[i] = __ldcg(T.dg + r0 + i);
          flg[i] = __ldcg(T.flag + r0 + i);
        }
        for (int i = tid; i < n; i += GT) {
          orig[i] = __ldcg(T.orig_at + i);
          pos[i] = __ldcg(T.pos_of + i);
        }
      }
      for (int e = tid; e < rows * nb; e += GT) Lp[e] = 0.0;
      if (tid == 0) s_r11 = init ? 0.0 : __ldcg(T.r11);
      __syncthreads();
      int j = k0, stopped = 0, cert = 0;
      if (n == 0 || T.kmax_dim == 0) {
        stopped = 1;
        cert = 1;
      } else {
        double bv = -1.0;
        int bp = INT_MAX, bi = -1;
        for (int i = tid; i < nr; i += GT)
          if (!flg[i] && better(dg[i], pos[r0 + i], bv, bp)) { bv = dg[i]; bp = pos[r0 + i]; bi = r0 + i; }
        block_cand(bv, bp, bi, &pub[0], wv, wp, wi);
      }
      cl.sync();
      for (int jj = 0; jj < nb && !stopped; jj++, j++) {
        const int buf = jj & 1;
        // decision for step j (identical in every CTA, rrqr.hpp:62-77): one
        // lane per peer CTA fetches its candidate over DSMEM, warp reduction
        if (tid < 32) {
          Cand c{-1.0, INT_MAX, -1};
          if (tid < CL) c = *cl.map_shared_rank(&pub[buf], tid);
          for (int o = 16; o > 0; o >>= 1) {
            const double v2 = __shfl_down_sync(0xffffffffu, c.v, o);
            const int p2 = __shfl_down_sync(0xffffffffu, c.pos, o);
            const int i2 = __shfl_down_sync(0xffffffffu, c.idx, o);
            if (better(v2, p2, c.v, c.pos)) c = {v2, p2, i2};
          }
          if (tid == 0) {
          const double pv = c.v > 0.0 ? sqrt(c.v) : 0.0;
          int stop = 0, ct = 0;
          if (j == 0) {
            s_r11 = pv;
            if (pv == 0.0 || pv <= abs_tol) { stop = 1; ct = 1; }
          } else if (pv <= eps * s_r11 || pv <= abs_tol) {
            stop = 1;
            ct = 1;
          }
          if (!stop && j == T.kmax) {
            stop = 1;
            ct = (j == T.kmax_dim);
          }
          s_stop = stop;
          s_cert = ct;
          s_pj = c.idx;
          s_ljj = pv;
          }
        }
        __syncthreads();
        if (s_stop) {
          stopped = 1;
          cert = s_cert;
          break;
        }
        const int pj = s_pj;
        const double ljj = s_ljj;
        const int owner = min(pj / rows, CL - 1);
        // pivot row's panel values from its owner (DSMEM)
        if (tid < jj) prow[tid] = cl.map_shared_rank(Lp, owner)[(size_t)tid * rows + (pj - owner * rows)];
        __syncthreads();
        // CPQR column swap of positions j and pos(pj), replicated in every CTA
        if (tid == 0) {
          const int pp = pos[pj], ok = orig[j];
          orig[j] = pj;
          orig[pp] = ok;
          pos[pj] = j;
          pos[ok] = pp;
        }
        // column j of L on own rows, residual norms downdated (clamped at 0)
        const double* gcol = T.G + (size_t)pj * n;
        double bv = -1.0;
        int bp = INT_MAX, bi = -1;
        __syncthreads();
        for (int i = tid; i < nr; i += GT) {
          const int gi = r0 + i;
          if (flg[i]) {
            T.L[gi + (size_t)j * n] = 0.0;
            continue;
          }
          if (gi == pj) {
            flg[i] = 1;
            Lp[(size_t)jj * rows + i] = ljj;
            T.L[gi + (size_t)j * n] = ljj;
            continue;
          }
          // lower triangle of G only (the trailing updates skip the upper one)
          double s = gi >= pj ? gcol[gi] : T.G[pj + (size_t)gi * n];
          for (int q = 0; q < jj; q++) s -= Lp[(size_t)q * rows + i] * prow[q];
          const double lo = s / ljj;
          Lp[(size_t)jj * rows + i] = lo;
          T.L[gi + (size_t)j * n] = lo;
          double dd = dg[i] - lo * lo;
          if (dd < 0.0) dd = 0.0;
          dg[i] = dd;
          if (better(dd, pos[gi], bv, bp)) { bv = dd; bp = pos[gi]; bi = gi; }
        }
        if (j + 1 == T.kmax_dim) {  // factorization exhausted exactly
          stopped = 1;
          cert = 1;
          j++;
          break;
        }
        block_cand(bv, bp, bi, &pub[buf ^ 1], wv, wp, wi);
        cl.sync();
      }
      // write back the state for the next panel / the host
      for (int i = tid; i < nr; i += GT) {
        __stcg(T.dg + r0 + i, dg[i]);
        __stcg(T.flag + r0 + i, flg[i]);
      }
      if (rank == 0) {
        for (int i = tid; i < n; i += GT) {
          __stcg(T.orig_at + i, orig[i]);
          __stcg(T.pos_of + i, pos[i]);
        }
        if (tid == 0) {
          if (k0 == 0) __stcg(T.r11, s_r11);
          __stcg(T.state + 0, j);
          __stcg(T.state + 1, stopped);
          __stcg(T.state + 2, cert);
        }
      }
      cl.sync();  // peers may still read this CTA's shared memory
    }
  }  // namespace

  void gram_cholesky_run(const std::vector<GramTask>& tasks, double eps, double abs_tol,
                         cudaStream_t s, std::vector<int>& rank, std::vector<int>& cert,
                         double* flops, const std::function<void()>& before_sync) {
    const int nt = (int)tasks.size();
    rank.assign(nt, 0);
    cert.assign(nt, 0);
    if (!nt) return;
    static bool attr = false;
    if (!attr) {
      HSSMF_CUDA(cudaFuncSetAttribute(gram_panel_kernel,
                                      cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      HSSMF_CUDA(cudaFuncSetAttribute(gram_panel_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemCap));
      attr = true;
    }
    int max_n = 0, kmax = 0;
    for (const auto& t : tasks) {
      max_n = std::max(max_n, t.n);
      kmax = std::max(kmax, t.kmax);
    }
    int CL = 1;
    while (CL < 16 && max_n > CL * 128) CL *= 2;
    const int rows = (max_n + CL - 1) / CL;
    int nb = kGramNB;
    while (nb > 8 && gram_smem(max_n, rows, nb) > (size_t)kSmemCap) nb /= 2;
    if (gram_smem(max_n, rows, nb) > (size_t)kSmemCap)
      throw CudaError("gram id: node too large for the cluster shared memory");
    GramTask* d = nullptr;
    bool owned = false;
    if (Staging* st = current_staging(s)) d = static_cast<GramTask*>(st->put(tasks.data(), nt * sizeof(GramTask)));
    if (!d) {
      owned = true;
      HSSMF_CUDA(cudaMallocAsync((void**)&d, nt * sizeof(GramTask), s));
      HSSMF_CUDA(cudaMemcpyAsync(d, tasks.data(), nt * sizeof(GramTask), cudaMemcpyHostToDevice, s));
    }
    std::vector<int> hst(3 * nt);
    // all panels are queued without host round trips: a finished task's
    // panel kernel returns at once and its trailing GEMM is skipped on device
    for (int k0 = 0; k0 <= kmax; k0 += nb) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(nt * CL);
      cfg.blockDim = dim3(GT);
      cfg.dynamicSmemBytes = gram_smem(max_n, rows, nb);
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CL;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      HSSMF_CUDA(cudaLaunchKernelEx(&cfg, gram_panel_kernel, (const GramTask*)d, k0, nb, eps,
                                    abs_tol, CL, k0 == 0 ? 1 : 0));
      HSSMF_LAUNCH_CHECK();
      if (k0 + nb > kmax) break;
      std::vector<GemmProblem> p;
      for (int t = 0; t < nt; t++) {
        const auto& T = tasks[t];
        if (k0 > T.kmax) continue;
        GemmProblem g{T.L + (size_t)k0 * T.n, T.L + (size_t)k0 * T.n, T.G, T.n, T.n, nb, T.n,
                      T.n, T.n};
        g.skip = T.state + 1;
        g.lower = 1;
        p.push_back(g);
      }
      if (flops) *flops += 0.5 * gemm_flops(p);
      gemm_run_host(p, 'N', 'T', -1.0, 1.0, s);
    }
    // the tasks' state triples are contiguous when the caller packs them
    bool packed = true;
    for (int t = 1; t < nt; t++) packed &= tasks[t].state == tasks[0].state + 3 * t;
    if (packed) {
      HSSMF_CUDA(cudaMemcpyAsync(hst.data(), tasks[0].state, 3 * nt * sizeof(int),
                                 cudaMemcpyDeviceToHost, s));
    } else {
      for (int t = 0; t < nt; t++)
        HSSMF_CUDA(cudaMemcpyAsync(&hst[3 * t], tasks[t].state, 3 * sizeof(int),
                                   cudaMemcpyDeviceToHost, s));
    }
    if (before_sync) before_sync();
    stream_sync(s);
    for (int t = 0; t < nt; t++) {
      rank[t] = hst[3 * t];
      cert[t] = hst[3 * t + 2];
    }
    if (owned) HSSMF_CUDA(cudaFreeAsync(d, s));
  }

}  // namespace hssmf_b200
