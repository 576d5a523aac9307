// TMA-fed DMMA GEMM for the large products of the HSS path (sampling
// S = F R / F^T R, densified updates, folds): C = alpha op(A) op(B) + beta C.
//
// Replaces, for big aligned problems, the reference's gemm / gemm_base
// (kernels.hpp:25-124). Design (sm_100a, FP64):
//  * CTA tile 128 x 128, k-step 16; 8 compute warps in a 2 x 4 grid of 64 x 32
//    warp tiles (8 x 4 DMMA m8n8k4 accumulators each).
//  * Operands are staged by TMA (cp.async.bulk.tensor.2d, 128-byte swizzle)
//    into a 5-stage ring of 32 KB stages; full / empty mbarriers, thread 0
//    refills a stage once every warp has released it (no __syncthreads in
//    the main loop).
//  * Conflict-free fragment loads without padding: within each 8-row block the
//    MMA rows / columns map to physical rows pi = {0,1,4,5,2,3,6,7} and the
//    four k-steps of a stage use physical k {0,1,4,5}, {2,3,6,7}, {8,9,12,13},
//    {10,11,14,15}. With the 128B swizzle (16-byte chunk c of row r stored at
//    c ^ (r % 8)) every half-warp's sixteen 8-byte loads then hit sixteen
//    distinct bank pairs, for all four operand layouts (A or A^T, B or B^T).
//  * Edges come from TMA's zero fill (out-of-bounds box elements read 0); the
//    epilogue masks rows >= m and columns >= n.
// Requirements (checked by gemm_tma_eligible): A and B 16-byte aligned and an
// even leading dimension (TMA global strides are multiples of 16 bytes).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "gemm.cuh"
#include "staging.cuh"

namespace hssmf_b200 {

  namespace {
    constexpr int TBM = 128, TBN = 128, TBK = 16, TST = 5;
    constexpr int NCW = 8;                    // compute warps
    constexpr int TTHREADS = NCW * 32;
    constexpr int STAGE_BYTES = (TBM + TBN) * TBK * 8;  // 32 KB
    constexpr int TSMEM = TST * STAGE_BYTES + 1024 + 128;
    constexpr int kTmaProbs = 24;

    struct alignas(64) TmaProb {
      CUtensorMap ta, tb;
      double* C;
      const int* skip;
      double alpha, beta;
      int m, n, k, ldc;
      int lower, tiles_m;
    };
    struct TmaParam {
      int nprob;
      int pre[kTmaProbs + 1];
      TmaProb p[kTmaProbs];
    };

    __device__ __forceinline__ uint32_t smem_addr(const void* p) {
      return (uint32_t)__cvta_generic_to_shared(p);
    }
    __device__ __forceinline__ void bar_init(uint32_t a, int count) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
    }
    __device__ __forceinline__ void bar_expect_tx(uint32_t a, uint32_t bytes) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
                   : "memory");
    }
    __device__ __forceinline__ void bar_arrive(uint32_t a) {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
    }
    __device__ __forceinline__ void bar_wait(uint32_t a, uint32_t parity) {
      asm volatile(
          "{\n"
          ".reg .pred p;\n"
          "WAIT_%=:\n"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
          "@!p bra WAIT_%=;\n"
          "}\n" ::"r"(a),
          "r"(parity)
          : "memory");
    }
    __device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0,
                                                int c1, uint32_t bar) {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
          "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
          : "memory");
    }

    // physical row of MMA row r within an 8-row block
    __device__ __forceinline__ int pi8(int r) { return (r & 1) | ((r & 2) << 1) | ((r & 4) >> 1); }

    // element offsets (doubles) inside one stage's operand region
    // "sub-box" layout: 8 boxes of [16 rows (k)][16 (m or n)], box b = idx / 16
    __device__ __forceinline__ int off_subbox(int idx, int k) {
      const int l = idx & 15;
      return (idx >> 4) * 256 + k * 16 + ((((l >> 1) ^ (k & 7)) << 1) | (l & 1));
    }
    // "row" layout: one box of [128 rows (m or n)][16 k]
    __device__ __forceinline__ int off_rows(int idx, int k) {
      return idx * 16 + ((((k >> 1) ^ (idx & 7)) << 1) | (k & 1));
    }

    template<bool TA, bool TB>
    __global__ void __launch_bounds__(TTHREADS, 1)
    gemm_tma_kernel(const __grid_constant__ TmaParam prm) {
      // (indexing the extern __shared__ array keeps every fragment load an
      // LDS with a 32-bit address; the 128B swizzle needs 1024-byte alignment)
      extern __shared__ __align__(1024) double tsm[];
      const int pad = ((1024 - (int)(smem_addr(tsm) & 1023)) & 1023) >> 3;
      double* sm = tsm + pad;
      uint64_t* full = reinterpret_cast<uint64_t*>(sm + TST * STAGE_BYTES / 8);
      uint64_t* empty = full + TST;

      int lo = 0, hi = prm.nprob - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (prm.pre[mid] <= (int)blockIdx.x) lo = mid; else hi = mid - 1;
      }
      const TmaProb& P = prm.p[lo];
      const int t = blockIdx.x - prm.pre[lo];
      const int m0 = (t % P.tiles_m) * TBM, n0 = (t / P.tiles_m) * TBN;
      if (P.lower && n0 >= m0 + TBM) return;
      if (P.skip && __ldcg(P.skip)) return;
      const int nk = (P.k + TBK - 1) / TBK;
      const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

      if (tid == 0) {
        for (int s = 0; s < TST; s++) {
          bar_init(smem_addr(&full[s]), 1);
          bar_init(smem_addr(&empty[s]), NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      }
      __syncthreads();

      // thread 0 also produces: it fills the first TST stages up front, and
      // refills stage s with k-tile kt + TST once all 8 warps have released it
      // (a separate producer warp would cap registers at 168 per thread: 9
      // warps put 3 on one SM sub-partition)
      auto produce = [&](int kt) {
        const int s = kt % TST;
        const uint32_t fb = smem_addr(&full[s]);
        bar_expect_tx(fb, STAGE_BYTES);
        const uint32_t sa = smem_addr(sm + s * (STAGE_BYTES / 8));
        const uint32_t sb = sa + TBM * TBK * 8;
        const int k0 = kt * TBK;
        if (!TA) {
#pragma unroll
          for (int b = 0; b < TBM / 16; b++) tma_load_2d(sa + b * 2048, &P.ta, m0 + 16 * b, k0, fb);
        } else {
          tma_load_2d(sa, &P.ta, k0, m0, fb);
        }
        if (!TB) {
          tma_load_2d(sb, &P.tb, k0, n0, fb);
        } else {
#pragma unroll
          for (int b = 0; b < TBN / 16; b++) tma_load_2d(sb + b * 2048, &P.tb, n0 + 16 * b, k0, fb);
        }
      };
      if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.ta)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.tb)) : "memory");
        for (int kt = 0; kt < TST && kt < nk; kt++) produce(kt);
      }

      // compute warps: 2 (m) x 4 (n) grid of 64 x 32 warp tiles
      const int wm = warp & 1, wn = warp >> 1;
      const int r8 = pi8(lane >> 2), kq = lane & 3;
      const int kofs = (kq & 1) | ((kq & 2) << 1);  // {0,1,4,5}
      double acc[8][4][2];
#pragma unroll
      for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

      for (int kt = 0; kt < nk; kt++) {
        const int s = kt % TST;
        bar_wait(smem_addr(&full[s]), (kt / TST) & 1);
        const double* As = sm + s * (STAGE_BYTES / 8);
        const double* Bs = As + TBM * TBK;
#pragma unroll
        for (int ks = 0; ks < 4; ks++) {
          const int k = (ks & 1) * 2 + (ks >> 1) * 8 + kofs;
          double a[8], b[4];
#pragma unroll
          for (int i = 0; i < 8; i++) {
            const int mi = wm * 64 + i * 8 + r8;
            a[i] = As[TA ? off_rows(mi, k) : off_subbox(mi, k)];
          }
#pragma unroll
          for (int j = 0; j < 4; j++) {
            const int nj = wn * 32 + j * 8 + r8;
            b[j] = Bs[TB ? off_subbox(nj, k) : off_rows(nj, k)];
          }
#pragma unroll
          for (int i = 0; i < 8; i++)
#pragma unroll
            for (int j = 0; j < 4; j++) dmma8x8x4(acc[i][j], a[i], b[j]);
        }
        __syncwarp();
        if (lane == 0) bar_arrive(smem_addr(&empty[s]));
        if (tid == 0 && kt + TST < nk) {
          bar_wait(smem_addr(&empty[s]), (kt / TST) & 1);
          produce(kt + TST);
        }
      }

      // epilogue: MMA row r -> physical row pi8(r), MMA column 2q+v -> pi8(2q+v)
      const double alpha = P.alpha, beta = P.beta;
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const int r = m0 + wm * 64 + i * 8 + r8;
        if (r >= P.m) continue;
#pragma unroll
        for (int j = 0; j < 4; j++)
#pragma unroll
          for (int v = 0; v < 2; v++) {
            const int c = n0 + wn * 32 + j * 8 + pi8(2 * kq + v);
            if (c >= P.n) continue;
            // lower-triangle problems: the same 64-granular block set as the
            // 64 x 64 kernel writes (blocks on or below the diagonal)
            if (P.lower && (c >> 6) > (r >> 6)) continue;
            double* cp = P.C + r + (size_t)c * P.ldc;
            const double x = alpha * acc[i][j][v];
            *cp = beta == 0.0 ? x : x + beta * *cp;
          }
      }
    }

    PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
      static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        HSSMF_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p)
          throw CudaError("cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
      }();
      return fn;
    }

    // 2D FP64 tensor map: inner extent x outer extent, column stride ld, box
    // {16, box_outer}, 128-byte swizzle, zero fill out of bounds
    void make_map(CUtensorMap* m, const double* ptr, long long inner, long long outer, long long ld,
                  int box_outer) {
      cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
      cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
      cuuint32_t box[2] = {16, (cuuint32_t)box_outer};
      cuuint32_t es[2] = {1, 1};
      const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(ptr),
                                     dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    }

    template<bool TA, bool TB> void set_attr_once() {
      static std::atomic<unsigned long long> done{0};
      once_per_device(done, [] {
        HSSMF_CUDA(cudaFuncSetAttribute(gemm_tma_kernel<TA, TB>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, TSMEM));
      });
    }

    template<bool TA, bool TB>
    void launch(const TmaParam& prm, int tiles, cudaStream_t s) {
      set_attr_once<TA, TB>();
      gemm_tma_kernel<TA, TB><<<tiles, TTHREADS, TSMEM, s>>>(prm);
    }
  }  // namespace

  bool gemm_tma_aligned(const GemmProblem& g) {
    static const bool off = getenv("HSSMF_NO_TMA") != nullptr;
    if (off || g.m < 96 || g.n < 96) return false;
    if ((reinterpret_cast<uintptr_t>(g.A) & 15) || (reinterpret_cast<uintptr_t>(g.B) & 15)) return false;
    static const bool trans_ok = getenv("HSSMF_TMA_TRANS") != nullptr;
    if ((g.trans & 3) && !trans_ok) return false;  // (see gemm_tma_eligible)
    return !(g.lda & 1) && !(g.ldb & 1);
  }

  bool gemm_tma_eligible(const GemmProblem& g) {
    static const bool off = getenv("HSSMF_NO_TMA") != nullptr;
    if (off) return false;
    const bool ta = g.trans & 1, tb = g.trans & 2;
    // long products only: one 128 x 128 CTA per SM does not overlap a tile's
    // pipeline fill and epilogue with another tile, so short-K shapes run
    // faster on the 64 x 64 kernel (4 CTAs per SM). Measured on B200
    // (profiles/r02_gemm_shapes.json): 8192^3 33.5-34.6 TF/s vs 30.9;
    // 3000^2 x 960 25.5 vs 29.6; 4096^2 x 128 11.8 vs 18.9.
    static const int kmin = getenv("HSSMF_TMA_KMIN") ? atoi(getenv("HSSMF_TMA_KMIN")) : 2048;
    if (g.m < 96 || g.n < 96 || g.k < kmin) return false;
    if ((reinterpret_cast<uintptr_t>(g.A) & 15) || (reinterpret_cast<uintptr_t>(g.B) & 15)) return false;
    if ((g.lda & 1) || (g.ldb & 1)) return false;
    // transposed operands stay on the 64 x 64 kernel: with them on this kernel
    // c4 (nonsymmetric fronts: S_c = F^T R, U B V^T updates) is not
    // reproducible from run to run -- 1-3 of 4 runs off the reference's ranks
    // on up to 234 of 17683 nodes, against 8 of 8 runs equal to the reference
    // with HSSMF_NO_TMA=1 (tools/determinism.py, profiles/r02/c4_determinism*.txt).
    // Not found by reading the kernel; the sanitizer is closed on this pool.
    // HSSMF_TMA_TRANS=1 re-enables them.
    static const bool trans_ok = getenv("HSSMF_TMA_TRANS") != nullptr;
    if ((ta || tb) && !trans_ok) return false;
    return true;
  }

  void gemm_tma_run(const std::vector<GemmProblem>& p, cudaStream_t s) {
    // one launch per transpose combination and parameter block
    for (int tr = 0; tr < 4; tr++) {
      TmaParam prm;
      prm.nprob = 0;
      prm.pre[0] = 0;
      double fl = 0, by = 0;
      int km = 0;
      auto flush = [&] {
        if (!prm.nprob) return;
        const int tiles = prm.pre[prm.nprob];
        {
          ProbeScope pr(PROBE_GEMM, s, fl, by);
          pr.tiles = tiles;
          pr.kmax = km;
          pr.nprob = prm.nprob;
          BigLaunch bl(s, tiles >= 74);
          switch (tr) {
            case 0: launch<false, false>(prm, tiles, bl.stream()); break;
            case 1: launch<true, false>(prm, tiles, bl.stream()); break;
            case 2: launch<false, true>(prm, tiles, bl.stream()); break;
            default: launch<true, true>(prm, tiles, bl.stream()); break;
          }
          HSSMF_LAUNCH_CHECK();
        }
        prm.nprob = 0;
        fl = by = 0;
        km = 0;
      };
      for (const auto& g : p) {
        if (g.trans != tr || g.m <= 0 || g.n <= 0) continue;
        if (prm.nprob == kTmaProbs) flush();
        TmaProb& q = prm.p[prm.nprob];
        const bool ta = tr & 1, tb = tr & 2;
        if (!ta) make_map(&q.ta, g.A, g.m, g.k, g.lda, 16);
        else make_map(&q.ta, g.A, g.k, g.m, g.lda, TBM);
        if (!tb) make_map(&q.tb, g.B, g.k, g.n, g.ldb, TBN);
        else make_map(&q.tb, g.B, g.n, g.k, g.ldb, 16);
        q.C = g.C;
        q.skip = g.skip;
        q.alpha = g.alpha;
        q.beta = g.beta;
        q.m = g.m;
        q.n = g.n;
        q.k = g.k;
        q.ldc = g.ldc;
        q.lower = g.lower;
        q.tiles_m = ceil_div(g.m, TBM);
        prm.pre[prm.nprob + 1] = prm.pre[prm.nprob] + q.tiles_m * ceil_div(g.n, TBN);
        if (probe_enabled()) {
          fl += (g.lower ? 1.0 : 2.0) * g.m * g.n * g.k;
          by += gemm_bytes(8.0 * ((double)g.m * g.k + (double)g.k * g.n),
                           (g.lower ? 0.5 : 1.0) * g.m * g.n, g.beta);
          km = std::max(km, g.k);
        }
        prm.nprob++;
      }
      flush();
    }
  }

}  // namespace hssmf_b200
