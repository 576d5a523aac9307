#include "gram_id.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <climits>
#include <cstdlib>

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

    // ---- cluster push messaging: st.async into the peers' shared memory,
    // completion counted in bytes on the receiver's mbarrier (no cluster
    // barrier, no remote loads on the per-step critical path)
    __device__ __forceinline__ uint32_t smem_u32(const void* p) {
      return (uint32_t)__cvta_generic_to_shared(p);
    }
    __device__ __forceinline__ uint32_t mapa(uint32_t a, int rank) {
      uint32_t r;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
      return r;
    }
    __device__ __forceinline__ void st_async_b64(uint32_t ra, unsigned long long v, uint32_t rbar) {
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
                   :: "r"(ra), "l"(v), "r"(rbar) : "memory");
    }
    __device__ __forceinline__ void st_async_v2(uint32_t ra, unsigned long long a,
                                                unsigned long long b, uint32_t rbar) {
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];"
                   :: "r"(ra), "l"(a), "l"(b), "r"(rbar) : "memory");
    }
    __device__ __forceinline__ void mbar_init(uint32_t a, int count) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(a), "r"(count) : "memory");
    }
    __device__ __forceinline__ void mbar_arrive_expect(uint32_t a, uint32_t bytes) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(a), "r"(bytes)
                   : "memory");
    }
    __device__ __forceinline__ void mbar_wait(uint32_t a, int parity) {
      asm volatile(
          "{\n"
          ".reg .pred P1;\n"
          "WAIT_%=:\n"
          "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
          "@!P1 bra WAIT_%=;\n"
          "}\n" :: "r"(a), "r"(parity) : "memory");
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

    // CTA-wide best candidate: warp shuffles, then every thread combines the
    // per-warp winners itself (no serial step, no second barrier)
    __device__ __forceinline__ Cand block_best(double bv, int bp, int bi, double* wv, int* wp,
                                               int* wi) {
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_down_sync(0xffffffffu, bv, o);
        const int p2 = __shfl_down_sync(0xffffffffu, bp, o);
        const int i2 = __shfl_down_sync(0xffffffffu, bi, o);
        if (better(v2, p2, bv, bp)) { bv = v2; bp = p2; bi = i2; }
      }
      if (lane == 0) { wv[warp] = bv; wp[warp] = bp; wi[warp] = bi; }
      __syncthreads();
      Cand c{wv[0], wp[0], wi[0]};
      for (int w = 1; w < GW; w++)
        if (better(wv[w], wp[w], c.v, c.pos)) c = {wv[w], wp[w], wi[w]};
      return c;
    }

    // nb steps of symmetric pivoted Cholesky on the Gram matrix, one
    // thread-block cluster per task. Rows are split in contiguous blocks over
    // the CTAs; each CTA keeps its rows' panel columns, residual norms and
    // flags plus a replicated copy of the position bookkeeping in shared
    // memory. Per elimination step there is ONE cluster barrier and ONE DSMEM
    // round trip: every CTA publishes its best candidate together with that
    // row's panel values, every CTA fetches all of them, and every thread
    // takes the (identical) pivot decision itself.
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
      // every CTA's candidate and that row's panel values, pushed by the
      // owners (double-buffered by step parity, one mbarrier per buffer)
      __shared__ __align__(16) Cand stc[2][16];
      __shared__ __align__(16) double strow[2][16][kGramNB];
      __shared__ __align__(8) unsigned long long mbar[2];
      __shared__ double wv[GW];
      __shared__ int wp[GW], wi[GW];

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
      double r11 = init ? 0.0 : __ldcg(T.r11);
      if (tid == 0) {
        mbar_init(smem_u32(&mbar[0]), 1);
        mbar_init(smem_u32(&mbar[1]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      }
      __syncthreads();
      // push this CTA's candidate (and nv values of its panel row) for the
      // step whose buffer is b into every peer, this CTA included
      auto push = [&](int b, const Cand& c, int nv) {
        if (tid >= CL * 16) return;
        const int peer = tid >> 4, l = tid & 15;
        const uint32_t rbar = mapa(smem_u32(&mbar[b]), peer);
        if (l == 0)
          st_async_v2(mapa(smem_u32(&stc[b][rank]), peer), (unsigned long long)__double_as_longlong(c.v),
                      (unsigned long long)(unsigned)c.pos | ((unsigned long long)(unsigned)c.idx << 32),
                      rbar);
        const uint32_t rrow = mapa(smem_u32(&strow[b][rank][0]), peer);
        const int ci = c.idx - r0;
        for (int q = l; q < nv; q += 16)
          st_async_b64(rrow + 8u * q,
                       (unsigned long long)__double_as_longlong(c.idx >= 0 ? Lp[(size_t)q * rows + ci] : 0.0),
                       rbar);
      };
      int j = k0, stopped = 0, cert = 0;
      Cand c0{-1.0, INT_MAX, -1};
      if (n == 0 || T.kmax_dim == 0) {
        stopped = 1;
        cert = 1;
      } else {
        double bv = -1.0;
        int bp = INT_MAX, bi = -1;
        for (int i = tid; i < nr; i += GT)
          if (!flg[i] && better(dg[i], pos[r0 + i], bv, bp)) { bv = dg[i]; bp = pos[r0 + i]; bi = r0 + i; }
        c0 = block_best(bv, bp, bi, wv, wp, wi);
      }
      cl.sync();  // every peer's mbarriers are initialised
      if (!stopped) push(0, c0, 0);
      for (int jj = 0; jj < nb && !stopped; jj++, j++) {
        const int buf = jj & 1;
        // wait for every CTA's candidate and panel row of this step
        if (tid == 0) mbar_arrive_expect(smem_u32(&mbar[buf]), (uint32_t)(CL * (16 + 8 * jj)));
        mbar_wait(smem_u32(&mbar[buf]), (jj >> 1) & 1);
        // decision for step j, taken identically by every thread of every
        // CTA (rrqr.hpp:62-77: largest residual norm, lowest position on ties)
        int w = 0;
        Cand best = stc[buf][0];
        for (int c = 1; c < CL; c++)
          if (better(stc[buf][c].v, stc[buf][c].pos, best.v, best.pos)) { best = stc[buf][c]; w = c; }
        const double pv = best.v > 0.0 ? sqrt(best.v) : 0.0;
        {
          int stop = 0, ct = 0;
          if (j == 0) {
            r11 = pv;
            if (pv == 0.0 || pv <= abs_tol) { stop = 1; ct = 1; }
          } else if (pv <= eps * r11 || pv <= abs_tol) {
            stop = 1;
            ct = 1;
          }
          if (!stop && j == T.kmax) {
            stop = 1;
            ct = (j == T.kmax_dim);
          }
          if (stop) {
            stopped = 1;
            cert = ct;
            break;
          }
        }
        const int pj = best.idx;
        const double ljj = pv;
        const double* prow = strow[buf][w];
        // CPQR column swap of positions j and pos(pj) (applied below by
        // thread 0 once every thread has read the old values)
        const int pp = pos[pj], ok = orig[j];
        // column j of L on own rows, residual norms downdated (clamped at 0)
        const double* gcol = T.G + (size_t)pj * n;
        double bv = -1.0;
        int bp = INT_MAX, bi = -1;
        for (int i = tid; i < nr; i += GT) {
          const int gi = r0 + i;
          if (flg[i]) continue;  // Lp stays 0 on pivoted rows
          if (gi == pj) {
            flg[i] = 1;
            Lp[(size_t)jj * rows + i] = ljj;
            continue;
          }
          // lower triangle of G only (the trailing updates skip the upper one);
          // the panel product is summed while the G load is in flight
          const double gv = gi >= pj ? gcol[gi] : T.G[pj + (size_t)gi * n];
          double t0 = 0.0, t1 = 0.0;
          int q = 0;
          for (; q + 1 < jj; q += 2) {
            t0 += Lp[(size_t)q * rows + i] * prow[q];
            t1 += Lp[(size_t)(q + 1) * rows + i] * prow[q + 1];
          }
          if (q < jj) t0 += Lp[(size_t)q * rows + i] * prow[q];
          const double lo = (gv - (t0 + t1)) / ljj;
          Lp[(size_t)jj * rows + i] = lo;
          double dd = dg[i] - lo * lo;
          if (dd < 0.0) dd = 0.0;
          dg[i] = dd;
          const int pgi = gi == ok ? pp : pos[gi];
          if (better(dd, pgi, bv, bp)) { bv = dd; bp = pgi; bi = gi; }
        }
        const Cand c = block_best(bv, bp, bi, wv, wp, wi);  // barrier inside
        if (tid == 0) {
          orig[j] = pj;
          orig[pp] = ok;
          pos[pj] = j;
          pos[ok] = pp;
        }
        if (j + 1 == T.kmax_dim) {  // factorization exhausted exactly
          stopped = 1;
          cert = 1;
          j++;
          break;
        }
        // push the candidate for step j + 1 with its panel row (q <= jj)
        push(buf ^ 1, c, jj + 1);
      }
      __syncthreads();
      // the panel's columns of L, written once from shared memory (no global
      // stores inside the step loop, so the per-step cluster barrier's release
      // fence has nothing to drain); pivoted rows hold 0
      {
        const int ncol = j - k0;
        for (int e = tid; e < ncol * nr; e += GT) {
          const int q = e / nr, i = e - q * nr;
          T.L[(r0 + i) + (size_t)(k0 + q) * n] = Lp[(size_t)q * rows + i];
        }
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
          if (k0 == 0) __stcg(T.r11, r11);
          __stcg(T.state + 0, j);
          __stcg(T.state + 1, stopped);
          __stcg(T.state + 2, cert);
        }
      }
      cl.sync();  // no CTA leaves while a peer may still address its shared memory
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
    // cluster size: one row per thread up to 16 CTAs (HSSMF_GRAM_MAXCL caps it;
    // measurement knob: wide clusters need co-resident SMs of one GPC)
    static const int max_cl = [] {
      const char* e = getenv("HSSMF_GRAM_MAXCL");
      const int v = e ? atoi(e) : 16;
      return (v == 1 || v == 2 || v == 4 || v == 8) ? v : 16;
    }();
    while (CL < max_cl && max_n > CL * GT) CL *= 2;
    const int rows = (max_n + CL - 1) / CL;
    int nb = kGramNB;
    while (nb > 8 && gram_smem(max_n, rows, nb) > (size_t)kSmemCap) nb -= 8;
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
      d2h(hst.data(), tasks[0].state, 3 * nt * sizeof(int), s);
    } else {
      for (int t = 0; t < nt; t++)
        d2h(&hst[3 * t], tasks[t].state, 3 * sizeof(int), s);
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
