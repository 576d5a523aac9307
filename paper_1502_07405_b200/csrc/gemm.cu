// Grouped variable-size DGEMM on DMMA (mma.sync m8n8k4 f64), cp.async-staged.
//
// CTA tile 64x64, k-step 16, 4 warps in a 2x2 grid of 32x32 warp tiles
// (4x4 DMMA 8x8 accumulators per warp), 3-stage cp.async pipeline. One
// launch covers all problems of a batch: blockIdx.x enumerates tiles, the
// owning problem is found by binary search over the tile prefix.
#include "gemm.cuh"
#include "staging.cuh"

#include <cstdlib>
#include <cstring>


namespace hssmf_b200 {

  namespace {
    constexpr int BM = kGemmBM, BN = kGemmBN, BK = 16, STAGES = 3, THREADS = 128;
    // shared memory of a TM x TN tile: A stored [k][m] (ld TM + 4), B stored
    // [n][k] (ld BK + 4): conflict-free fragment loads
    template<int TM, int TN> constexpr int smem_of() {
      return STAGES * (BK * (TM + 4) + TN * (BK + 4)) * 8;
    }
    constexpr int SMEM = smem_of<BM, BN>();
    // small batches (fewer 64 x 64 tiles than two per SM) run 32 x 32 tiles:
    // four times the CTAs for launches that cannot fill the GPU otherwise
    constexpr int SM_BM = 32, SM_BN = 32;
    constexpr int SMEM_SMALL = smem_of<SM_BM, SM_BN>();

    // descriptors passed by value as a __grid_constant__ kernel parameter:
    // a dynamic-phase launch then needs no separate descriptor upload
    constexpr int kParamProbs = 96;
    struct GemmParam {
      int nprob;
      int pre[kParamProbs + 1];
      GemmProblem p[kParamProbs];
    };

    // problem owning this CTA's tile (binary search over the tile prefix)
    __device__ __forceinline__ int find_problem(const int* prefix, int nprob, int tile) {
      int lo = 0, hi = nprob - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (prefix[mid] <= tile) lo = mid; else hi = mid - 1;
      }
      return lo;
    }

    // one TM x TN output tile t of problem P (4 warps in a 2 x 2 grid of
    // (TM/2) x (TN/2) warp tiles)
    template<bool TA, bool TB, int TM = BM, int TN = BN>
    __device__ __forceinline__ void gemm_tile(const GemmProblem& P, int t, double alpha,
                                              double beta) {
      constexpr int BM = TM, BN = TN;
      constexpr int SA = BM + 4, SB = BK + 4;
      constexpr int MI = BM / 16, NJ = BN / 16;  // 8 x 8 DMMA tiles per warp
      extern __shared__ __align__(16) double gsm[];
      double (*As)[BK * SA] = reinterpret_cast<double (*)[BK * SA]>(gsm);
      double (*Bs)[BN * SB] = reinterpret_cast<double (*)[BN * SB]>(gsm + STAGES * BK * SA);

      if (P.skip && __ldcg(P.skip)) return;
      const int tiles_m = (P.m + BM - 1) / BM;
      const int m0 = (t % tiles_m) * BM, n0 = (t / tiles_m) * BN;
      // lower-triangle problems: the 64 x 64 blocks on or below the diagonal
      if (P.lower && (n0 >> 6) > (m0 >> 6)) return;
      const int K = P.k;

      const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
      const int wm = warp & 1, wn = warp >> 1;

      double acc[MI][NJ][2];
#pragma unroll
      for (int i = 0; i < MI; i++)
#pragma unroll
        for (int j = 0; j < NJ; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

      auto load_stage = [&](int st, int k0) {
        // A tile: BM x BK logical (rows m, cols k)
#pragma unroll
        for (int r = 0; r < (BM * BK) / THREADS; r++) {
          int mm, kk;
          if (!TA) { mm = tid % BM; kk = tid / BM + r * (THREADS / BM); }
          else { kk = tid % BK; mm = tid / BK + r * (THREADS / BK); }
          const int gm = m0 + mm, gk = k0 + kk;
          const bool ok = gm < P.m && gk < K;
          const double* src = ok ? (TA ? P.A + gk + (size_t)gm * P.lda
                                       : P.A + gm + (size_t)gk * P.lda)
                                 : P.A;
          cp_async8(&As[st][kk * SA + mm], src, ok);
        }
        // B tile: BK x BN logical (rows k, cols n)
#pragma unroll
        for (int r = 0; r < (BN * BK) / THREADS; r++) {
          int nn, kk;
          if (!TB) { kk = tid % BK; nn = tid / BK + r * (THREADS / BK); }
          else { nn = tid % BN; kk = tid / BN + r * (THREADS / BN); }
          const int gn = n0 + nn, gk = k0 + kk;
          const bool ok = gn < P.n && gk < K;
          const double* src = ok ? (TB ? P.B + gn + (size_t)gk * P.ldb
                                       : P.B + gk + (size_t)gn * P.ldb)
                                 : P.B;
          cp_async8(&Bs[st][nn * SB + kk], src, ok);
        }
      };

      const int nk = (K + BK - 1) / BK;
#pragma unroll
      for (int s = 0; s < STAGES - 1; s++) {
        if (s < nk) load_stage(s, s * BK);
        cp_async_commit();
      }
      const int am = wm * (BM / 2) + (lane >> 2), bn = wn * (BN / 2) + (lane >> 2), kq = lane & 3;
      for (int kt = 0; kt < nk; kt++) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        {
          const int nxt = kt + STAGES - 1;
          if (nxt < nk) load_stage(nxt % STAGES, nxt * BK);
          cp_async_commit();
        }
        const double* as = As[kt % STAGES];
        const double* bs = Bs[kt % STAGES];
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
          double a[MI], b[NJ];
#pragma unroll
          for (int i = 0; i < MI; i++) a[i] = as[(kk + kq) * SA + am + i * 8];
#pragma unroll
          for (int j = 0; j < NJ; j++) b[j] = bs[(bn + j * 8) * SB + kk + kq];
#pragma unroll
          for (int i = 0; i < MI; i++)
#pragma unroll
            for (int j = 0; j < NJ; j++) dmma8x8x4(acc[i][j], a[i], b[j]);
        }
      }
      cp_async_wait<0>();

      // epilogue
#pragma unroll
      for (int i = 0; i < MI; i++) {
        const int r = m0 + wm * (BM / 2) + i * 8 + (lane >> 2);
        if (r >= P.m) continue;
#pragma unroll
        for (int j = 0; j < NJ; j++)
#pragma unroll
          for (int v = 0; v < 2; v++) {
            const int c = n0 + wn * (BN / 2) + j * 8 + 2 * kq + v;
            if (c >= P.n) continue;
            double* cp = P.C + r + (size_t)c * P.ldc;
            const double x = alpha * acc[i][j][v];
            *cp = beta == 0.0 ? x : x + beta * *cp;
          }
      }
    }

    template<bool TA, bool TB>
    __global__ void __launch_bounds__(THREADS)
    gemm_grouped_kernel(const GemmProblem* __restrict__ probs, const int* __restrict__ prefix,
                        int nprob, double alpha, double beta) {
      const int lo = find_problem(prefix, nprob, blockIdx.x);
      const GemmProblem P = probs[lo];
      gemm_tile<TA, TB>(P, blockIdx.x - prefix[lo], alpha, beta);
    }

    // mixed batch: every problem carries its own transposes and alpha / beta
    template<int TM, int TN>
    __global__ void __launch_bounds__(THREADS)
    gemm_param_kernel(const __grid_constant__ GemmParam b) {
      const int lo = find_problem(b.pre, b.nprob, blockIdx.x);
      const GemmProblem& P = b.p[lo];
      const int t = blockIdx.x - b.pre[lo];
      switch (P.trans) {
        case 0: gemm_tile<false, false, TM, TN>(P, t, P.alpha, P.beta); break;
        case 1: gemm_tile<true, false, TM, TN>(P, t, P.alpha, P.beta); break;
        case 2: gemm_tile<false, true, TM, TN>(P, t, P.alpha, P.beta); break;
        default: gemm_tile<true, true, TM, TN>(P, t, P.alpha, P.beta); break;
      }
    }

    // C = sum_s W_s + beta C over the split-K partial products (fixed order)
    __global__ void splitk_reduce_kernel(const double* __restrict__ W, int S, int m, int n,
                                         double beta, double* __restrict__ C, int ldc) {
      const long long tot = (long long)m * n, stride = (long long)gridDim.x * blockDim.x;
      for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += stride) {
        double v = W[e];
        for (int q = 1; q < S; q++) v += W[e + q * tot];
        const int i = (int)(e % m), j = (int)(e / m);
        double* c = C + i + (size_t)j * ldc;
        *c = beta == 0.0 ? v : v + beta * *c;
      }
    }

    void set_gemm_attrs() {
      static std::atomic<unsigned long long> done{0};
      once_per_device(done, [] {
      HSSMF_CUDA(cudaFuncSetAttribute(gemm_grouped_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
      HSSMF_CUDA(cudaFuncSetAttribute(gemm_grouped_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
      HSSMF_CUDA(cudaFuncSetAttribute(gemm_grouped_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
      HSSMF_CUDA(cudaFuncSetAttribute(gemm_grouped_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
      HSSMF_CUDA(cudaFuncSetAttribute(gemm_param_kernel<BM, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
      HSSMF_CUDA(cudaFuncSetAttribute(gemm_param_kernel<SM_BM, SM_BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_SMALL));
      });
    }
  }  // namespace

  std::vector<int> gemm_tile_prefix(const std::vector<GemmProblem>& p) {
    std::vector<int> pre(p.size() + 1, 0);
    for (size_t i = 0; i < p.size(); i++)
      pre[i + 1] = pre[i] + ceil_div(p[i].m, BM) * ceil_div(p[i].n, BN);
    return pre;
  }

  double gemm_flops(const std::vector<GemmProblem>& p) {
    double f = 0;
    for (const auto& q : p) f += 2.0 * q.m * q.n * q.k;
    return f;
  }

  double gemm_ab_bytes(const std::vector<GemmProblem>& p) {
    double f = 0;
    for (const auto& q : p) f += 8.0 * ((double)q.m * q.k + (double)q.k * q.n);
    return f;
  }

  double gemm_c_elems(const std::vector<GemmProblem>& p) {
    double f = 0;
    for (const auto& q : p) f += (q.lower ? 0.5 : 1.0) * q.m * q.n;
    return f;
  }

  void gemm_run(const GemmBatchDev& b, char ta, char tb, double alpha, double beta,
                cudaStream_t s) {
    if (b.nprob == 0 || b.tiles == 0) return;
    const bool TA = ta != 'N', TB = tb != 'N';
    set_gemm_attrs();
    dim3 grid(b.tiles), block(THREADS);
    ProbeScope pr(PROBE_GEMM, s, probe_enabled() ? b.flops : 0.0,
                  probe_enabled() ? gemm_bytes(b.ab_bytes, b.c_elems, beta) : 0.0);
    if (!TA && !TB) gemm_grouped_kernel<false, false><<<grid, block, SMEM, s>>>(b.probs, b.prefix, b.nprob, alpha, beta);
    else if (TA && !TB) gemm_grouped_kernel<true, false><<<grid, block, SMEM, s>>>(b.probs, b.prefix, b.nprob, alpha, beta);
    else if (!TA && TB) gemm_grouped_kernel<false, true><<<grid, block, SMEM, s>>>(b.probs, b.prefix, b.nprob, alpha, beta);
    else gemm_grouped_kernel<true, true><<<grid, block, SMEM, s>>>(b.probs, b.prefix, b.nprob, alpha, beta);
    HSSMF_LAUNCH_CHECK();
  }

  void gemm_run_host(const std::vector<GemmProblem>& p, char ta, char tb, double alpha,
                     double beta, cudaStream_t s) {
    std::vector<GemmProblem> q(p);
    for (auto& x : q) gemm_set_op(x, ta, tb, alpha, beta);
    gemm_run_mixed(q, s);
  }

  int gemm_splitk_factor(int m, int n, int k, bool tma) {
    // resident CTAs: 4 per SM for the 64 x 64 tile kernel, 1 per SM for the
    // 128 x 128 TMA kernel
    const long long slots = tma ? 148LL : 148LL * 4;
    const long long tiles = tma ? (long long)ceil_div(m, 128) * ceil_div(n, 128)
                                : (long long)ceil_div(m, BM) * ceil_div(n, BN);
    if (tiles >= 4 * slots || k < 2048) return 1;
    int best = 1;
    double best_eff = 0;
    for (int S = 1; S <= 8 && k / S >= 512; S++) {
      const long long c = tiles * S;
      const double eff = (double)c / (double)(((c + slots - 1) / slots) * slots);
      if (eff > best_eff + 0.02) {
        best_eff = eff;
        best = S;
      }
    }
    return best;
  }

  void gemm_run_splitk(const GemmProblem& p0, char ta, char tb, double alpha, double beta,
                       cudaStream_t s) {
    if (p0.m <= 0 || p0.n <= 0) return;
    // TMA slices when the operands allow it: each slice keeps >= 512 of K,
    // long enough for the 128 x 128 kernel (6000 x 128 x 6000 in 6 slices:
    // 26.6 TF/s, 20480 x 128 x 20480 in 8: 30.6 TF/s)
    GemmProblem pt = p0;
    gemm_set_op(pt, ta, tb, alpha, beta);
    const bool tma = gemm_tma_aligned(pt) && p0.k >= 2048;
    int S = gemm_splitk_factor(p0.m, p0.n, p0.k, tma);
    // HSSMF_SPLITK_KSLICE=k: slices of at most k (>= 512) of K on the TMA
    // kernel: its CTAs hold a whole SM each (164 KB of shared memory), so
    // shorter CTAs return SMs to the other fronts' latency-bound chains sooner
    static const int kslice = getenv("HSSMF_SPLITK_KSLICE") ? std::max(512, atoi(getenv("HSSMF_SPLITK_KSLICE"))) : 0;
    if (tma && kslice > 0) S = std::max(S, std::min(ceil_div(p0.k, kslice), 64));
    if (S <= 1) {
      gemm_run_host({p0}, ta, tb, alpha, beta, s);
      return;
    }
    // K slices rounded to the k-step; partial products into a workspace,
    // then one deterministic reduction
    const int kc = ceil_div(ceil_div(p0.k, S), BK) * BK;
    const long long mn = (long long)p0.m * p0.n;
    double* W = nullptr;
    HSSMF_CUDA(cudaMallocAsync((void**)&W, (size_t)mn * S * sizeof(double), s));
    std::vector<GemmProblem> parts;
    int used = 0;
    for (int q = 0; q < S; q++) {
      const int k0 = q * kc, k1 = std::min(p0.k, k0 + kc);
      if (k1 <= k0) break;
      GemmProblem g = p0;
      g.A = ta == 'N' ? p0.A + (size_t)k0 * p0.lda : p0.A + k0;
      g.B = tb == 'N' ? p0.B + k0 : p0.B + (size_t)k0 * p0.ldb;
      g.k = k1 - k0;
      g.C = W + q * mn;
      g.ldc = p0.m;
      g.lower = 0;
      gemm_set_op(g, ta, tb, alpha, 0.0);
      parts.push_back(g);
      used++;
    }
    if (tma) gemm_tma_run(parts, s);
    else gemm_run_mixed(parts, s);
    const int blocks = (int)std::min<long long>((mn + 255) / 256, 148LL * 16);
    splitk_reduce_kernel<<<blocks, 256, 0, s>>>(W, used, p0.m, p0.n, beta, p0.C, p0.ldc);
    HSSMF_LAUNCH_CHECK();
    HSSMF_CUDA(cudaFreeAsync(W, s));
  }

  void gemm_run_mixed(const std::vector<GemmProblem>& p0, cudaStream_t s) {
    // big aligned problems go to the TMA kernel, the rest stay here
    std::vector<GemmProblem> big, p;
    for (const auto& x : p0) (gemm_tma_eligible(x) ? big : p).push_back(x);
    if (!big.empty()) gemm_tma_run(big, s);
    if (p.empty()) return;
    set_gemm_attrs();
    // tile size of the launch: 32 x 32 when the whole list has fewer 64 x 64
    // tiles than two per SM (latency-bound batches of the adaptive rounds)
    // (long-K products keep 64 x 64 tiles: 6000 x 128 x 6000 ran at 10.6 TF/s
    // on 32 x 32 tiles against 18.5)
    long long t64 = 0;
    int kmax_all = 0;
    for (const auto& x : p)
      if (x.m > 0 && x.n > 0) {
        t64 += (long long)ceil_div(x.m, BM) * ceil_div(x.n, BN);
        kmax_all = std::max(kmax_all, x.k);
      }
    static const bool no_small = getenv("HSSMF_GEMM_NO_SMALL") != nullptr;
    const bool small = !no_small && t64 < 2 * 148 && kmax_all <= 1024;
    const int tm = small ? SM_BM : BM, tn = small ? SM_BN : BN;
    GemmParam b;
    b.nprob = 0;
    b.pre[0] = 0;
    auto flush = [&] {
      if (!b.nprob) return;
      const int tiles = b.pre[b.nprob];
      if (tiles) {
        double fl = 0, by = 0;
        int km = 0;
        if (probe_enabled())
          for (int q = 0; q < b.nprob; q++) {
            const GemmProblem& g = b.p[q];
            fl += (g.lower ? 1.0 : 2.0) * g.m * g.n * g.k;
            by += gemm_bytes(8.0 * ((double)g.m * g.k + (double)g.k * g.n),
                             (g.lower ? 0.5 : 1.0) * g.m * g.n, g.beta);
            km = std::max(km, g.k);
          }
        ProbeScope pr(PROBE_GEMM, s, fl, by);
        pr.tiles = tiles;
        pr.kmax = km;
        pr.nprob = b.nprob;
        // (full-device launches of a worker stream go through its
        // low-priority lane, staging.cuh)
        BigLaunch bl(s, !small && tiles >= 2 * 148);
        if (small) gemm_param_kernel<SM_BM, SM_BN><<<tiles, THREADS, SMEM_SMALL, bl.stream()>>>(b);
        else gemm_param_kernel<BM, BN><<<tiles, THREADS, SMEM, bl.stream()>>>(b);
        HSSMF_LAUNCH_CHECK();
      }
      b.nprob = 0;
    };
    // problems of one call are independent (distinct outputs), so a list
    // longer than one parameter block is split over several launches
    for (const auto& x : p) {
      if (x.m <= 0 || x.n <= 0) continue;
      if (b.nprob == kParamProbs) flush();
      b.p[b.nprob] = x;
      b.pre[b.nprob + 1] = b.pre[b.nprob] + ceil_div(x.m, tm) * ceil_div(x.n, tn);
      b.nprob++;
    }
    flush();
  }

}  // namespace hssmf_b200
