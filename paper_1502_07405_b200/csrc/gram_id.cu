#include "gram_id.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>

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
        // push the candidate for step j + 1 with its panel row (q <= jj); not
        // after the panel's last step: no peer waits on that phase, and an
        // st.async still in flight when a peer exits could land in a later
        // cluster's shared memory
        if (jj + 1 < nb) push(buf ^ 1, c, jj + 1);
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

    // ---- v2 panel: one row per thread, the row's panel columns in registers
    // (the step loop is unrolled, so every panel column has a fixed register),
    // a shared-memory copy only for the candidate push. Per step the critical
    // path is: mbarrier wake -> warp-parallel decision over the CL candidates
    // -> G(i, pj) load (the winner's panel row is read while it is in
    // flight) -> division / downdate -> warp argmax -> one CTA barrier ->
    // warp w pushes the CTA's candidate and its panel row to peer w
    // (st.async, byte-counted mbarrier). No replicated position arrays: the
    // CPQR column swap is resolved locally (the row at position j is the one
    // whose position equals j; it takes the pivot's old position, which
    // travels with the candidate).
    // warp-wide best candidate (largest v, lowest position on ties), returned
    // to every lane. Non-negative doubles order like their bit patterns, so the
    // argmax is three redux.sync operations (high word, low word among the
    // high-word winners, lowest position among the value winners) and one
    // broadcast instead of a five-level butterfly of four shuffles each. A lane
    // without a candidate passes v = -1 (p = INT_MAX, ix = -1): it keys as
    // zero and loses every tie on its position.
    __device__ __forceinline__ void warp_best(double& v, int& p, int& ix) {
      const unsigned full = 0xffffffffu;
      const unsigned long long bits = v > 0.0 ? (unsigned long long)__double_as_longlong(v) : 0ull;
      const unsigned hi = (unsigned)(bits >> 32), lo = (unsigned)bits;
      const unsigned mh = __reduce_max_sync(full, hi);
      const unsigned ml = __reduce_max_sync(full, hi == mh ? lo : 0u);
      const bool top = hi == mh && lo == ml;
      const unsigned mp = __reduce_min_sync(full, top ? (unsigned)p : 0xffffffffu);
      const unsigned win = __ballot_sync(full, top && (unsigned)p == mp);
      const int src = __ffs(win) - 1;  // (some lane always matches: mp is a top lane's position)
      ix = __shfl_sync(full, ix, src);
      p = (int)mp;
      v = ix >= 0 ? __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml)) : -1.0;
    }

    // best of the first cnt (<= 32) candidates in shared memory, returned to
    // every lane: a short sequential scan for a few entries, otherwise the
    // warp argmax over the low lanes
    __device__ __forceinline__ void best_of(const Cand* c, int cnt, double& v, int& p, int& ix) {
      if (cnt <= 4) {
        v = c[0].v;
        p = c[0].pos;
        ix = c[0].idx;
        for (int q = 1; q < cnt; q++) {
          const Cand x = c[q];
          if (better(x.v, x.pos, v, p)) { v = x.v; p = x.pos; ix = x.idx; }
        }
        return;
      }
      const int lane = threadIdx.x & 31;
      if (lane < cnt) {
        const Cand x = c[lane];
        v = x.v;
        p = x.pos;
        ix = x.idx;
      } else {
        v = -1.0;
        p = INT_MAX;
        ix = -1;
      }
      warp_best(v, p, ix);
    }

    template <int R, int NB>
    __global__ void __launch_bounds__(512, 1)
    gram_panel2_kernel(const GramTask* __restrict__ tasks, int k0, double eps, double abs_tol,
                       int CL, int init, unsigned long long* tprobe) {
      // T threads (a multiple of 32, <= 512, sized to the rows on the host)
      const int T = blockDim.x, NW = T / 32, RPC = T * R;  // rows per CTA
      cg::cluster_group cl = cg::this_cluster();
      const int rank = (int)cl.block_rank();
      const GramTask Tk = tasks[blockIdx.x / CL];
      const int n = Tk.n;
      const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
      const int row0 = rank * RPC + tid;  // own rows row0 + a T, a < R
      extern __shared__ __align__(16) double sm2[];
      double* Lp = sm2;  // [NB][RPC]: own rows' panel columns (pivoted rows stay 0)
      __shared__ __align__(16) Cand stc[2][16];
      __shared__ __align__(16) double strow[2][16][NB];
      __shared__ __align__(8) unsigned long long mbar[2];
      __shared__ Cand wred[2][16];

      // (a warm-started task resumes at step kw from the state the fixed-order
      // panels left; only cold tasks initialise in their first panel)
      init = init && Tk.kw == 0;
      k0 += Tk.kw;
      if (__ldcg(Tk.state + 1) && !init) return;  // finished in an earlier panel (uniform)
      double dg[R];
      int pos[R], flg[R];
#pragma unroll
      for (int a = 0; a < R; a++) {
        const int i = row0 + a * T;
        dg[a] = 0.0;
        pos[a] = INT_MAX;
        flg[a] = 1;
        if (i < n) {
          if (init) {
            dg[a] = Tk.G[i + (size_t)i * n];
            pos[a] = i;
            flg[a] = 0;
          } else {
            dg[a] = __ldcg(Tk.dg + i);
            pos[a] = __ldcg(Tk.pos_of + i);
            flg[a] = __ldcg(Tk.flag + i);
          }
        }
      }
      for (int e = tid; e < NB * RPC; e += T) Lp[e] = 0.0;
      double r11 = init ? 0.0 : __ldcg(Tk.r11);
      if (tid == 0) {
        mbar_init(smem_u32(&mbar[0]), 1);
        mbar_init(smem_u32(&mbar[1]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      }
      // candidate of this CTA for the step whose buffer is b; the panel row
      // carries nv values; warp w pushes it to peers w, w + NW, ...
      auto propose = [&](int b, int nv) {
        double v = -1.0;
        int p = INT_MAX, ix = -1;
#pragma unroll
        for (int a = 0; a < R; a++)
          if (!flg[a] && better(dg[a], pos[a], v, p)) {
            v = dg[a];
            p = pos[a];
            ix = row0 + a * T;
          }
        warp_best(v, p, ix);
        if (lane == 0) wred[b][warp] = {v, p, ix};
        __syncthreads();
        if (warp >= CL) return;
        best_of(wred[b], NW, v, p, ix);
        // the winner's panel row: nv <= NB values, lane c carries columns
        // c and c + 32 (NB <= 64)
        static_assert(NB <= 64, "panel rows are pushed by two lanes' worth of columns");
        const double rv = (lane < nv && ix >= 0) ? Lp[lane * RPC + (ix - rank * RPC)] : 0.0;
        const double rv2 =
            (lane + 32 < nv && ix >= 0) ? Lp[(lane + 32) * RPC + (ix - rank * RPC)] : 0.0;
        for (int peer = warp; peer < CL; peer += NW) {
          const uint32_t rbar = mapa(smem_u32(&mbar[b]), peer);
          if (lane == 0)
            st_async_v2(mapa(smem_u32(&stc[b][rank]), peer),
                        (unsigned long long)__double_as_longlong(v),
                        (unsigned long long)(unsigned)p | ((unsigned long long)(unsigned)ix << 32),
                        rbar);
          if (lane < nv)
            st_async_b64(mapa(smem_u32(&strow[b][rank][lane]), peer),
                         (unsigned long long)__double_as_longlong(rv), rbar);
          if (lane + 32 < nv)
            st_async_b64(mapa(smem_u32(&strow[b][rank][lane + 32]), peer),
                         (unsigned long long)__double_as_longlong(rv2), rbar);
        }
      };
      int stopped = 0, cert = 0, jend = k0;
      if (n == 0 || Tk.kmax_dim == 0) {
        stopped = 1;
        cert = 1;
      }
      cl.sync();  // every peer's mbarriers are initialised
      if (!stopped) propose(0, 0);
      // rolled step loop: an unrolled one overflows the instruction cache
#pragma unroll 1
      for (int jj = 0; jj < NB; jj++) {
        if (stopped) break;
        const int j = k0 + jj, buf = jj & 1;
        // per-step segment timing of CTA 0 / thread 0 (HSSMF_GRAM_TPROBE)
        const bool tp = tprobe && blockIdx.x == 0 && tid == 0;
        long long c_a = tp ? clock64() : 0;
        if (tid == 0) mbar_arrive_expect(smem_u32(&mbar[buf]), (uint32_t)(CL * (16 + 8 * jj)));
        mbar_wait(smem_u32(&mbar[buf]), (jj >> 1) & 1);
        long long c_b = tp ? clock64() : 0;
        // decision (rrqr.hpp:62-77: largest residual norm, lowest position on
        // ties): every lane scans the CL candidates itself
        double bv;
        int bp, bi;
        best_of(stc[buf], CL, bv, bp, bi);
        // the pivot's G column is requested before the stop tests (a stopped
        // step discards the values)
        double gv[R];
#pragma unroll
        for (int a = 0; a < R; a++) {
          const int i = row0 + a * T;
          gv[a] = 0.0;
          if (bi >= 0 && i < n && !flg[a] && i != bi)
            gv[a] = i >= bi ? Tk.G[i + (size_t)bi * n] : Tk.G[bi + (size_t)i * n];
        }
        const double pv = bv > 0.0 ? sqrt(bv) : 0.0;
        int stop = 0, ct = 0;
        if (j == 0) {
          r11 = pv;
          if (pv == 0.0 || pv <= abs_tol) { stop = 1; ct = 1; }
        } else if (pv <= eps * r11 || pv <= abs_tol) {
          stop = 1;
          ct = 1;
        }
        if (!stop && j == Tk.kmax) {
          stop = 1;
          ct = (j == Tk.kmax_dim);
        }
        if (stop) {
          stopped = 1;
          cert = ct;
          jend = j;
          if (Tk.pvlast && rank == 0 && tid == 0) {
            __stcg(Tk.pvlast + 0, pv);
            __stcg(Tk.pvlast + 1, r11);
          }
          break;
        }
        const int pj = bi, pp = bp;
        const double ljj = pv;
        long long c_c = tp ? clock64() : 0;
        const double* prow = strow[buf][pj / RPC];
        double t0[R], t1[R];
#pragma unroll
        for (int a = 0; a < R; a++) t0[a] = t1[a] = 0.0;
        const double* lrow = Lp + tid;
        int q = 0;
#pragma unroll 2
        for (; q + 1 < jj; q += 2) {
          const double p0 = prow[q], p1 = prow[q + 1];
#pragma unroll
          for (int a = 0; a < R; a++) {
            t0[a] += lrow[q * RPC + a * T] * p0;
            t1[a] += lrow[(q + 1) * RPC + a * T] * p1;
          }
        }
        if (q < jj) {
#pragma unroll
          for (int a = 0; a < R; a++) t0[a] += lrow[q * RPC + a * T] * prow[q];
        }
#pragma unroll
        for (int a = 0; a < R; a++) {
          const int i = row0 + a * T;
          if (i >= n) continue;
          if (!flg[a]) {
            double lo;
            if (i == pj) {
              flg[a] = 1;
              lo = ljj;
            } else {
              lo = (gv[a] - (t0[a] + t1[a])) / ljj;
              double dd = dg[a] - lo * lo;
              if (dd < 0.0) dd = 0.0;
              dg[a] = dd;
            }
            Lp[jj * RPC + a * T + tid] = lo;
          }
          if (i == pj) pos[a] = j;
          else if (pos[a] == j) pos[a] = pp;
        }
        jend = j + 1;
        if (j + 1 == Tk.kmax_dim) {  // factorization exhausted exactly
          stopped = 1;
          cert = 1;
          break;
        }
        long long c_d = tp ? clock64() : 0;
        if (jj + 1 < NB) propose(buf ^ 1, jj + 1);  // (no peer waits after the last step)
        if (tp) {
          const long long c_e = clock64();
          atomicAdd(tprobe + 0, (unsigned long long)(c_b - c_a));
          atomicAdd(tprobe + 1, (unsigned long long)(c_c - c_b));
          atomicAdd(tprobe + 2, (unsigned long long)(c_d - c_c));
          atomicAdd(tprobe + 3, (unsigned long long)(c_e - c_d));
          atomicAdd(tprobe + 4, 1ull);
        }
      }
      // the panel's columns of L (pivoted rows hold 0), state for the next
      // panel / the host, the current ID permutation
      const int ncol = jend - k0;
#pragma unroll
      for (int a = 0; a < R; a++) {
        const int i = row0 + a * T;
        if (i >= n) continue;
        for (int q = 0; q < ncol; q++) Tk.L[i + (size_t)(k0 + q) * n] = Lp[q * RPC + a * T + tid];
        __stcg(Tk.dg + i, dg[a]);
        __stcg(Tk.flag + i, flg[a]);
        __stcg(Tk.pos_of + i, pos[a]);
        __stcg(Tk.orig_at + pos[a], i);
      }
      if (rank == 0 && tid == 0) {
        if (k0 == 0) __stcg(Tk.r11, r11);
        __stcg(Tk.state + 0, jend);
        __stcg(Tk.state + 1, stopped);
        __stcg(Tk.state + 2, cert);
      }
      cl.sync();  // no CTA leaves while a peer may still address its shared memory
    }

    // trailing update of the Gram matrix after a panel: G_lower -= Lp Lp^T,
    // Lp = the panel's NB columns of L (n x NB, ld n). HBM-bound (each lower
    // element read and written once, 2 NB flops): 64 x 64 tiles of the lower
    // triangle, the two L row blocks staged in shared memory, 4 x 4 outputs
    // per thread, the G tile loads issued before the products. Tasks that
    // stopped in the panel are skipped.
    template <int NB>
    __global__ void __launch_bounds__(256, 2)
    gram_syrk_kernel(const GramTask* __restrict__ tasks, int k0, unsigned long long* probe_bytes) {
      const GramTask Tk = tasks[blockIdx.y];
      k0 += Tk.kw;
      const int n = Tk.n;
      const int nbt = (n + 63) >> 6;
      const int t = blockIdx.x;
      if (t >= nbt * (nbt + 1) / 2) return;
      if (__ldcg(Tk.state + 1)) return;
      // algorithmic bytes of a live task: its lower triangle read and written once
      if (probe_bytes && t == 0 && threadIdx.x == 0)
        atomicAdd(probe_bytes, (unsigned long long)n * (n + 1) / 2 * 16ull);
      int ti = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
      while (ti * (ti + 1) / 2 > t) ti--;
      while ((ti + 1) * (ti + 2) / 2 <= t) ti++;
      const int tj = t - ti * (ti + 1) / 2;
      const int i0 = ti * 64, j0 = tj * 64;
      extern __shared__ __align__(16) double sm3[];
      double (*As)[64] = reinterpret_cast<double (*)[64]>(sm3);
      double (*Bs)[64] = reinterpret_cast<double (*)[64]>(sm3 + NB * 64);
      // thread (tx, ty) owns rows i0 + tx + 16 a and columns j0 + 4 ty + b, so
      // that a warp's G accesses are 128-byte row runs of two columns
      const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
      // the two L row blocks by cp.async (all in flight at once), then the G
      // tile loads, which complete while the products run
      const double* Lk = Tk.L + (size_t)k0 * n;
#pragma unroll
      for (int e = tid; e < NB * 64; e += 256) {
        const int q = e >> 6, r = e & 63;
        const bool va = i0 + r < n, vb = j0 + r < n;
        cp_async8(&As[q][r], va ? Lk + i0 + r + (size_t)q * n : Lk, va);
        cp_async8(&Bs[q][r], vb ? Lk + j0 + r + (size_t)q * n : Lk, vb);
      }
      cp_async_commit();
      double* G = Tk.G + i0 + tx + (size_t)(j0 + ty * 4) * n;
      const int jm = n - (j0 + ty * 4), im = n - (i0 + tx);
      double c[4][4];
#pragma unroll
      for (int b = 0; b < 4; b++)
#pragma unroll
        for (int a = 0; a < 4; a++)
          c[a][b] = (16 * a < im && b < jm) ? G[16 * a + (size_t)b * n] : 0.0;
      cp_async_wait<0>();
      __syncthreads();
      double acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) acc[a][b] = 0.0;
#pragma unroll 8
      for (int q = 0; q < NB; q++) {
        const double2 b01 = *reinterpret_cast<const double2*>(&Bs[q][ty * 4]);
        const double2 b23 = *reinterpret_cast<const double2*>(&Bs[q][ty * 4 + 2]);
        const double bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
        for (int a = 0; a < 4; a++) {
          const double av = As[q][tx + 16 * a];
#pragma unroll
          for (int b = 0; b < 4; b++) acc[a][b] = fma(av, bv[b], acc[a][b]);
        }
      }
#pragma unroll
      for (int b = 0; b < 4; b++)
#pragma unroll
        for (int a = 0; a < 4; a++)
          if (16 * a < im && b < jm && i0 + tx + 16 * a >= j0 + ty * 4 + b)
            G[16 * a + (size_t)b * n] = c[a][b] - acc[a][b];
    }

    // the same trailing update on the FP64 tensor pipe (DMMA m8n8k4): 64 x 64
    // lower tiles, 8 warps of 32 x 16, operands staged by cp.async into
    // padded shared tiles (stride 68: a warp's fragment loads hit every bank
    // pair exactly twice), the tile's G entries loaded into registers before
    // the products. Two shared loads feed 256 FMAs instead of 32.
    template <int NB>
    __global__ void __launch_bounds__(256, 2)
    gram_syrk_dmma_kernel(const GramTask* __restrict__ tasks, int k0,
                          unsigned long long* probe_bytes, int warm) {
      constexpr int SP = 68;
      const GramTask Tk = tasks[blockIdx.y];
      // warm phase: absolute panel k0 of the tasks still inside their warm
      // part; search phase: panels counted from each task's kw
      if (warm) {
        if (k0 >= Tk.kw) return;
      } else {
        k0 += Tk.kw;
      }
      const int n = Tk.n;
      const int nbt = (n + 63) >> 6;
      const int t = blockIdx.x;
      if (t >= nbt * (nbt + 1) / 2) return;
      if (__ldcg(Tk.state + 1)) return;
      if (probe_bytes && t == 0 && threadIdx.x == 0)
        atomicAdd(probe_bytes, (unsigned long long)n * (n + 1) / 2 * 16ull);
      // column-major order of the lower tiles: CTAs running together sweep
      // long contiguous column strips of G (DRAM page locality)
      auto before = [&](int c) { return c * nbt - c * (c - 1) / 2; };
      const double bb = 2.0 * nbt + 1.0;
      int tj = (int)((bb - sqrt(fmax(bb * bb - 8.0 * t, 0.0))) * 0.5);
      tj = max(0, min(tj, nbt - 1));
      while (tj > 0 && before(tj) > t) tj--;
      while (tj + 1 < nbt && before(tj + 1) <= t) tj++;
      const int ti = tj + (t - before(tj));
      const int i0 = ti * 64, j0 = tj * 64;
      extern __shared__ __align__(16) double sm5[];
      double* As = sm5;            // [NB][SP]: As[q][r] = L(i0 + r, k0 + q)
      double* Bs = sm5 + NB * SP;  // [NB][SP]: Bs[q][r] = L(j0 + r, k0 + q)
      const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
      const double* Lk = Tk.L + (size_t)k0 * n;
      for (int e = tid; e < NB * 64; e += 256) {
        const int q = e >> 6, r = e & 63;
        const bool va = i0 + r < n, vb = j0 + r < n;
        cp_async8(As + q * SP + r, va ? Lk + i0 + r + (size_t)q * n : Lk, va);
        cp_async8(Bs + q * SP + r, vb ? Lk + j0 + r + (size_t)q * n : Lk, vb);
      }
      cp_async_commit();
      const int wm = warp & 1, wn = warp >> 1;  // warp tile rows 32 wm, cols 16 wn
      const int lr = lane >> 2, lc = lane & 3;
      double* G = Tk.G;
      double c[4][2][2];
#pragma unroll
      for (int mi = 0; mi < 4; mi++)
#pragma unroll
        for (int ni = 0; ni < 2; ni++)
#pragma unroll
          for (int v = 0; v < 2; v++) {
            const int i = i0 + 32 * wm + 8 * mi + lr, j = j0 + 16 * wn + 8 * ni + 2 * lc + v;
            c[mi][ni][v] = (i < n && j < n && i >= j) ? G[i + (size_t)j * n] : 0.0;
          }
      cp_async_wait<0>();
      __syncthreads();
      double acc[4][2][2];
#pragma unroll
      for (int mi = 0; mi < 4; mi++)
#pragma unroll
        for (int ni = 0; ni < 2; ni++) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
#pragma unroll
      for (int kk = 0; kk < NB; kk += 4) {
        double a[4], b[2];
#pragma unroll
        for (int mi = 0; mi < 4; mi++) a[mi] = As[(kk + lc) * SP + 32 * wm + 8 * mi + lr];
#pragma unroll
        for (int ni = 0; ni < 2; ni++) b[ni] = Bs[(kk + lc) * SP + 16 * wn + 8 * ni + lr];
#pragma unroll
        for (int mi = 0; mi < 4; mi++)
#pragma unroll
          for (int ni = 0; ni < 2; ni++) dmma8x8x4(acc[mi][ni], a[mi], b[ni]);
      }
#pragma unroll
      for (int mi = 0; mi < 4; mi++)
#pragma unroll
        for (int ni = 0; ni < 2; ni++)
#pragma unroll
          for (int v = 0; v < 2; v++) {
            const int i = i0 + 32 * wm + 8 * mi + lr, j = j0 + 16 * wn + 8 * ni + 2 * lc + v;
            if (i < n && j < n && i >= j) G[i + (size_t)j * n] = c[mi][ni][v] - acc[mi][ni][v];
          }
    }

    // Persistent form of the trailing update (opt-in, HSSMF_GRAM_SYRK=persist):
    // every CTA walks the lower 64 x 64 tiles of all tasks (stride gridDim.x)
    // and double-buffers them through shared memory, the next tile's G and L
    // blocks streaming in (cp.async) while the current tile's DMMA products run.
    // One 136 KB CTA per SM hides less latency than two one-tile CTAs per SM:
    // measured 1.92 TB/s on c5 against 2.51 TB/s. Same arithmetic per element.
    constexpr int kSyrkMaxTasks = 128;
    struct SyrkParam {
      int nt;
      int pre[kSyrkMaxTasks + 1];  // tile prefix per task
    };
    template <int NB>
    __global__ void __launch_bounds__(256, 1)
    gram_syrk_persist_kernel(const GramTask* __restrict__ tasks, int k0,
                             const __grid_constant__ SyrkParam prm,
                             unsigned long long* probe_bytes) {
      constexpr int SP = 68, GP = 65;
      extern __shared__ __align__(16) double sm6[];
      // stage st: As[NB][SP], Bs[NB][SP], Gs[64][GP] (Gs[c][r] = G(i0 + r, j0 + c))
      constexpr int STAGE = 2 * NB * SP + 64 * GP;
      __shared__ int live[kSyrkMaxTasks];
      const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
      for (int q = tid; q < prm.nt; q += blockDim.x) live[q] = !__ldcg(tasks[q].state + 1);
      __syncthreads();
      if (probe_bytes && blockIdx.x == 0 && tid == 0)
        for (int q = 0; q < prm.nt; q++)
          if (live[q]) {
            const unsigned long long n = tasks[q].n;
            atomicAdd(probe_bytes, n * (n + 1) / 2 * 16ull);
          }
      const int total = prm.pre[prm.nt];
      struct Tile { int q, i0, j0, n; const double* Lk; double* G; };
      auto locate = [&](int T) {
        int lo = 0, hi = prm.nt - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (prm.pre[mid] <= T) lo = mid; else hi = mid - 1;
        }
        Tile x;
        x.q = lo;
        const GramTask& Tk = tasks[lo];
        x.n = Tk.n;
        const int nbt = (x.n + 63) >> 6;
        const int t = T - prm.pre[lo];
        auto before = [&](int c) { return c * nbt - c * (c - 1) / 2; };
        const double bb = 2.0 * nbt + 1.0;
        int tj = (int)((bb - sqrt(fmax(bb * bb - 8.0 * t, 0.0))) * 0.5);
        tj = max(0, min(tj, nbt - 1));
        while (tj > 0 && before(tj) > t) tj--;
        while (tj + 1 < nbt && before(tj + 1) <= t) tj++;
        x.i0 = (tj + (t - before(tj))) * 64;
        x.j0 = tj * 64;
        x.Lk = Tk.L + (size_t)(k0 + Tk.kw) * x.n;
        x.G = Tk.G;
        return x;
      };
      // next live tile at or after T (stride gridDim.x)
      auto next_live = [&](int T) {
        while (T < total) {
          int lo = 0, hi = prm.nt - 1;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (prm.pre[mid] <= T) lo = mid; else hi = mid - 1;
          }
          if (live[lo]) return T;
          T += gridDim.x;
        }
        return total;
      };
      auto load = [&](const Tile& x, int st) {
        double* As = sm6 + st * STAGE;
        double* Bs = As + NB * SP;
        double* Gs = Bs + NB * SP;
        const int n = x.n;
        for (int e = tid; e < NB * 64; e += 256) {
          const int q = e >> 6, r = e & 63;
          const bool va = x.i0 + r < n, vb = x.j0 + r < n;
          cp_async8(As + q * SP + r, va ? x.Lk + x.i0 + r + (size_t)q * n : x.Lk, va);
          cp_async8(Bs + q * SP + r, vb ? x.Lk + x.j0 + r + (size_t)q * n : x.Lk, vb);
        }
        for (int e = tid; e < 64 * 64; e += 256) {
          const int c = e >> 6, r = e & 63;
          const bool v = x.i0 + r < n && x.j0 + c < n && x.i0 + r >= x.j0 + c;
          cp_async8(Gs + c * GP + r, v ? x.G + x.i0 + r + (size_t)(x.j0 + c) * n : x.G, v);
        }
      };
      const int wm = warp & 1, wn = warp >> 1;  // warp tile rows 32 wm, cols 16 wn
      const int lr = lane >> 2, lc = lane & 3;
      int T = next_live(blockIdx.x), st = 0;
      if (T < total) load(locate(T), 0);
      cp_async_commit();
      while (T < total) {
        const Tile x = locate(T);
        const int Tn = next_live(T + gridDim.x);
        if (Tn < total) load(locate(Tn), st ^ 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        const double* As = sm6 + st * STAGE;
        const double* Bs = As + NB * SP;
        const double* Gs = Bs + NB * SP;
        double acc[4][2][2];
#pragma unroll
        for (int mi = 0; mi < 4; mi++)
#pragma unroll
          for (int ni = 0; ni < 2; ni++) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < NB; kk += 4) {
          double a[4], b[2];
#pragma unroll
          for (int mi = 0; mi < 4; mi++) a[mi] = As[(kk + lc) * SP + 32 * wm + 8 * mi + lr];
#pragma unroll
          for (int ni = 0; ni < 2; ni++) b[ni] = Bs[(kk + lc) * SP + 16 * wn + 8 * ni + lr];
#pragma unroll
          for (int mi = 0; mi < 4; mi++)
#pragma unroll
            for (int ni = 0; ni < 2; ni++) dmma8x8x4(acc[mi][ni], a[mi], b[ni]);
        }
        const int n = x.n;
#pragma unroll
        for (int mi = 0; mi < 4; mi++)
#pragma unroll
          for (int ni = 0; ni < 2; ni++)
#pragma unroll
            for (int v = 0; v < 2; v++) {
              const int r = 32 * wm + 8 * mi + lr, c = 16 * wn + 8 * ni + 2 * lc + v;
              const int i = x.i0 + r, j = x.j0 + c;
              if (i < n && j < n && i >= j)
                x.G[i + (size_t)j * n] = Gs[c * GP + r] - acc[mi][ni][v];
            }
        __syncthreads();  // stage st is refilled in the next iteration
        st ^= 1;
        T = Tn;
      }
      cp_async_wait<0>();
    }

    // ---- warm start: fixed-order panels -------------------------------------
    // state of a warm-started task before its first fixed-order panel: the
    // permutation the earlier ID ended with, residual norms = diag(G), the
    // first kw positions flagged as pivoted, r11 = the largest diagonal entry
    // (what the pivot search would have taken first), state = {kw, 0, 0}
    __global__ void __launch_bounds__(256) gram_warm_init_kernel(const GramTask* __restrict__ tasks) {
      const GramTask Tk = tasks[blockIdx.x];
      if (Tk.kw <= 0) return;
      const int n = Tk.n;
      double mx = 0.0;
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double g = Tk.G[i + (size_t)i * n];
        const int p = Tk.warm_pos[i];
        Tk.dg[i] = g;
        Tk.pos_of[i] = p;
        Tk.orig_at[i] = Tk.warm_orig[i];
        Tk.flag[i] = p < Tk.kw ? 1 : 0;
        mx = fmax(mx, g);
      }
      __shared__ double sm[8];
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = mx;
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int w = 1; w < 8; w++) mx = fmax(mx, sm[w]);
        *Tk.r11 = mx > 0.0 ? sqrt(mx) : 0.0;
        Tk.state[0] = Tk.kw;
        Tk.state[1] = 0;
        Tk.state[2] = 0;
      }
    }

    // one fixed-order panel: the NB pivots orig_at[k0 .. k0 + NB) of every task
    // with kw > k0. Every CTA factors the panel's NB x NB diagonal block of the
    // (updated) Gram matrix in shared memory, then each thread solves its
    // row's NB panel entries against it: L(i, k0 + c) = (G(i, p_c) - sum_{q<c}
    // L(i, q) Lbb(c, q)) / Lbb(c, c), downdates the row's residual norm and
    // stores the row. No pivot search, no cluster: rows are independent once
    // the diagonal block is known. Rows pivoted in earlier panels hold 0.
    // A non-positive pivot (roundoff on a dependent row) stops the task with
    // state[1] = 3: the host repeats its ID with the pivot search from step 0.
    template <int NB>
    __global__ void __launch_bounds__(128) gram_fixed_panel_kernel(const GramTask* __restrict__ tasks,
                                                                   int k0) {
      const GramTask Tk = tasks[blockIdx.y];
      if (k0 >= Tk.kw) return;
      const int n = Tk.n;
      const int row0 = blockIdx.x * 128;
      if (row0 >= n) return;
      if (__ldcg(Tk.state + 1)) return;
      __shared__ double Lb[NB][NB + 1];
      __shared__ int piv[NB];
      __shared__ int bad;
      const int tid = threadIdx.x;
      if (tid < NB) piv[tid] = Tk.orig_at[k0 + tid];
      if (tid == 0) bad = 0;
      __syncthreads();
      for (int e = tid; e < NB * NB; e += 128) {
        const int a = e / NB, c = e % NB;  // a >= c: lower triangle of the diagonal block
        if (a >= c) {
          const int pa = piv[a], pc = piv[c];
          Lb[a][c] = pa >= pc ? Tk.G[pa + (size_t)pc * n] : Tk.G[pc + (size_t)pa * n];
        }
      }
      __syncthreads();
      // in-place Cholesky of the block (right-looking, column by column)
      for (int c = 0; c < NB; c++) {
        const double dcc = Lb[c][c];
        if (!(dcc > 0.0)) {
          if (tid == 0) bad = 1;
        }
        __syncthreads();
        if (bad) break;
        const double l = sqrt(dcc);
        if (tid > c && tid < NB) Lb[tid][c] /= l;
        __syncthreads();
        if (tid == 0) Lb[c][c] = l;
        for (int e = tid; e < (NB - c - 1) * (NB - c - 1); e += 128) {
          const int a = c + 1 + e / (NB - c - 1), b = c + 1 + e % (NB - c - 1);
          if (a >= b) Lb[a][b] -= Lb[a][c] * Lb[b][c];
        }
        __syncthreads();
      }
      if (bad) {
        if (blockIdx.x == 0 && tid == 0) {
          __stcg(Tk.state + 1, 3);
          __stcg(Tk.state + 2, 0);
        }
        return;
      }
      const int i = row0 + tid;
      if (i >= n) return;
      const int pi = Tk.pos_of[i];
      double* Li = Tk.L + i + (size_t)k0 * n;
      if (pi < k0) {  // pivoted in an earlier panel
#pragma unroll 4
        for (int c = 0; c < NB; c++) Li[(size_t)c * n] = 0.0;
        return;
      }
      const int own = pi < k0 + NB ? pi - k0 : NB;  // this panel's pivot rows end at their own column
      double x[NB];
#pragma unroll
      for (int c = 0; c < NB; c++) {
        const int pc = piv[c];
        x[c] = i >= pc ? Tk.G[i + (size_t)pc * n] : Tk.G[pc + (size_t)i * n];
      }
      double dsum = 0.0;
#pragma unroll
      for (int c = 0; c < NB; c++) {
        double v = x[c];
#pragma unroll
        for (int q = 0; q < c; q++) v -= x[q] * Lb[c][q];
        v = c <= own ? v / Lb[c][c] : 0.0;
        if (c == own) v = Lb[c][c];
        x[c] = v;
        dsum += v * v;
      }
#pragma unroll
      for (int c = 0; c < NB; c++) Li[(size_t)c * n] = x[c];
      if (own == NB) {
        double dd = Tk.dg[i] - dsum;
        Tk.dg[i] = dd > 0.0 ? dd : 0.0;
      }
    }

  }  // namespace

  // per-step segment cycles of the panel kernel (measurement knob): wait,
  // decision, row update, propose + push; printed by gram_tprobe_report()
  unsigned long long* gram_tprobe() {
    static unsigned long long* p = [] {
      unsigned long long* q = nullptr;
      if (getenv("HSSMF_GRAM_TPROBE")) {
        HSSMF_CUDA(cudaMalloc(&q, 8 * sizeof(unsigned long long)));
        HSSMF_CUDA(cudaMemset(q, 0, 8 * sizeof(unsigned long long)));
      }
      return q;
    }();
    return p;
  }
  void gram_tprobe_report() {
    unsigned long long* p = gram_tprobe();
    if (!p) return;
    unsigned long long h[8];
    HSSMF_CUDA(cudaMemcpy(h, p, sizeof(h), cudaMemcpyDeviceToHost));
    const double n = h[4] ? (double)h[4] : 1.0;
    fprintf(stderr, "[gram] steps %llu  cycles/step: wait %.0f decide %.0f update %.0f propose %.0f\n",
            h[4], h[0] / n, h[1] / n, h[2] / n, h[3] / n);
    HSSMF_CUDA(cudaMemset(p, 0, sizeof(h)));
  }

  namespace {
    // HSSMF_LANES=1: GEMMs only; HSSMF_LANES=all: the Gram trailing updates too
    bool lanes_for_syrk() {
      static const bool v = getenv("HSSMF_LANES") && !strcmp(getenv("HSSMF_LANES"), "all");
      return v;
    }
  }  // namespace

  void gram_cholesky_run(const std::vector<GramTask>& tasks0, double eps, double abs_tol,
                         cudaStream_t s, std::vector<int>& rank, std::vector<int>& cert,
                         double* flops, const std::function<void()>& before_sync) {
    const int nt = (int)tasks0.size();
    rank.assign(nt, 0);
    cert.assign(nt, 0);
    if (!nt) return;
    static std::atomic<unsigned long long> attr{0};
    once_per_device(attr, [] {
      HSSMF_CUDA(cudaFuncSetAttribute(gram_panel_kernel,
                                      cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      HSSMF_CUDA(cudaFuncSetAttribute(gram_panel_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemCap));
    });
    int max_n = 0, kmax = 0;
    for (const auto& t : tasks0) max_n = std::max(max_n, t.n);
    // warm starts need the one-row-per-thread panels (n <= 8192) and whole
    // panels of fixed pivots
    std::vector<GramTask> tasks(tasks0);
    int max_kw = 0;
    for (auto& t : tasks) {
      if (max_n > 16 * 512 || getenv("HSSMF_GRAM_V1") || !t.warm_orig || !t.warm_pos) t.kw = 0;
      t.kw = std::min(t.kw, t.kmax) / kGramPanel * kGramPanel;
      if (!t.kw) t.warm_orig = t.warm_pos = nullptr;
      max_kw = std::max(max_kw, t.kw);
      kmax = std::max(kmax, t.kmax - t.kw);  // steps of the pivot search
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
    // v2 panel: one row per thread, up to 512 rows per CTA in clusters of up
    // to 16, the CTA sized to its rows (no idle warps in the per-step
    // decision work); HSSMF_GRAM_V1=1 keeps the older shared-memory kernel
    const bool force_v1 = getenv("HSSMF_GRAM_V1") != nullptr;
    // panel width of the one-row-per-thread panel: 48 steps (three panels of 32
    // per two of 48: a third fewer trailing updates, which move the whole
    // lower Gram matrix each; 512 rows x 48 columns of L = 192 KB of shared memory)
    constexpr int NB2 = 48, RPC_MAX = 512;
    constexpr int kSyrkPersistSmem = 2 * (2 * NB2 * 68 + 64 * 65) * 8;
    const bool v2 = !force_v1 && max_n <= 16 * RPC_MAX;
    int T2 = 32, CL2 = 1;
    if (v2) {
      static std::atomic<unsigned long long> attr2{0};
      once_per_device(attr2, [] {
        HSSMF_CUDA(cudaFuncSetAttribute(gram_panel2_kernel<1, NB2>,
                                        cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        HSSMF_CUDA(cudaFuncSetAttribute(gram_panel2_kernel<1, NB2>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        RPC_MAX * NB2 * 8));
        HSSMF_CUDA(cudaFuncSetAttribute(gram_syrk_kernel<NB2>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * NB2 * 64 * 8));
        HSSMF_CUDA(cudaFuncSetAttribute(gram_syrk_dmma_kernel<NB2>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * NB2 * 68 * 8));
        HSSMF_CUDA(cudaFuncSetAttribute(gram_syrk_persist_kernel<NB2>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        kSyrkPersistSmem));

      });
      while (CL2 * RPC_MAX < max_n) CL2 *= 2;
      T2 = std::max(32, ((max_n + CL2 - 1) / CL2 + 31) / 32 * 32);
      CL = CL2;
      nb = NB2;
    }
    // trailing update on the FP64 tensor pipe unless HSSMF_GRAM_SYRK=fma
    const char* esy = getenv("HSSMF_GRAM_SYRK");
    const bool syrk_cuda_cores = esy && !strcmp(esy, "fma");
    // HSSMF_GRAM_SYRK=persist: the persistent double-buffered update (measured
    // slower on c5: 1.92 TB/s against 2.51 for one tile per CTA, 2 CTAs per SM,
    // profiles/r02/README.md)
    const bool syrk_persist = esy && !strcmp(esy, "persist");
    // (a variant that reads and writes the G tile after the products, 64-80
    // registers and 3-4 CTAs per SM, measured slower: 6.7-8.4 us per step at
    // n = 7400 against 6.1, tools/gram_bench.py)
    // warm-started tasks: their first kw pivots as fixed-order panels (one
    // grid over the rows per panel, no pivot search), each followed by the
    // trailing update
    if (v2 && max_kw > 0) {
      gram_warm_init_kernel<<<nt, 256, 0, s>>>((const GramTask*)d);
      HSSMF_LAUNCH_CHECK();
      const int nbt = (max_n + 63) / 64;
      for (int k0 = 0; k0 < max_kw; k0 += NB2) {
        gram_fixed_panel_kernel<NB2><<<dim3((max_n + 127) / 128, nt), 128, 0, s>>>((const GramTask*)d, k0);
        HSSMF_LAUNCH_CHECK();
        ProbeScope prs(PROBE_GRAM_SYRK, s, 0.0, 0.0);
        unsigned long long* pb = probe_enabled() ? probe_device_bytes() : nullptr;
        {
          BigLaunch bl(s, lanes_for_syrk() && (long long)nbt * (nbt + 1) / 2 * nt >= 2 * 148);
          gram_syrk_dmma_kernel<NB2><<<dim3(nbt * (nbt + 1) / 2, nt), 256, 2 * NB2 * 68 * 8, bl.stream()>>>(
              (const GramTask*)d, k0, pb, 1);
        }
        HSSMF_LAUNCH_CHECK();
        if (flops)
          for (const auto& T : tasks)
            if (k0 < T.kw) *flops += (double)T.n * T.n * NB2;
      }
    }
    // all panels are queued without host round trips: a finished task's
    // panel kernel returns at once and its trailing GEMM is skipped on device
    for (int k0 = 0; k0 <= kmax; k0 += nb) {
      if (v2) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(nt * CL2);
        cfg.blockDim = dim3(T2);
        cfg.dynamicSmemBytes = (size_t)T2 * NB2 * 8;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = CL2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        {
          ProbeScope prp(PROBE_GRAM_PANEL, s, 0.0, 0.0);
          prp.tiles = CL2;
          prp.kmax = max_n;
          prp.nprob = nt;
          HSSMF_CUDA(cudaLaunchKernelEx(&cfg, gram_panel2_kernel<1, NB2>, (const GramTask*)d, k0,
                                        eps, abs_tol, CL2, k0 == 0 ? 1 : 0, gram_tprobe()));
          HSSMF_LAUNCH_CHECK();
        }
        if (k0 + nb > kmax) break;
        const int nbt = (max_n + 63) / 64;
        {
          ProbeScope prs(PROBE_GRAM_SYRK, s, 0.0, 0.0);
          unsigned long long* pb = probe_enabled() ? probe_device_bytes() : nullptr;
          if (syrk_persist && nt <= kSyrkMaxTasks) {
            SyrkParam sp;
            sp.nt = nt;
            sp.pre[0] = 0;
            for (int q = 0; q < nt; q++) {
              const int b = (tasks[q].n + 63) / 64;
              sp.pre[q + 1] = sp.pre[q] + b * (b + 1) / 2;
            }
            const int grid = std::max(1, std::min(sp.pre[nt], 148));
            gram_syrk_persist_kernel<NB2><<<grid, 256, kSyrkPersistSmem, s>>>(
                (const GramTask*)d, k0, sp, pb);
          } else if (syrk_cuda_cores)
            gram_syrk_kernel<NB2><<<dim3(nbt * (nbt + 1) / 2, nt), 256, 2 * NB2 * 64 * 8, s>>>(
                (const GramTask*)d, k0, pb);
          else {
            BigLaunch bl(s, lanes_for_syrk() && (long long)nbt * (nbt + 1) / 2 * nt >= 2 * 148);
            gram_syrk_dmma_kernel<NB2><<<dim3(nbt * (nbt + 1) / 2, nt), 256, 2 * NB2 * 68 * 8, bl.stream()>>>(
                (const GramTask*)d, k0, pb, 0);
          }
          HSSMF_LAUNCH_CHECK();
        }
        if (flops)
          for (const auto& T : tasks)
            if (k0 + T.kw <= T.kmax) *flops += (double)T.n * T.n * NB2;
        continue;
      }
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
      // a fixed-order panel met a non-positive pivot: the caller repeats the
      // ID without the warm start
      if (hst[3 * t + 1] == 3) rank[t] = -1;
    }
    if (owned) HSSMF_CUDA(cudaFreeAsync(d, s));
  }

}  // namespace hssmf_b200
