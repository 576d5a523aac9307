// Grouped, variable-size FP64 GEMM on the sm_100a FP64 tensor pipe (DMMA).
//
// Replaces the reference's recursive gemm/gemm_base (kernels.hpp:25-124):
// C = alpha op(A) op(B) + beta C for a list of independent problems, each
// with its own pointers, sizes and leading dimensions, in ONE launch. Used
// for the dense-front trailing/Schur updates, the HSS sampling products and
// every batched per-level product of the HSS path.
#pragma once

#include <vector>

#include "common.cuh"

namespace hssmf_b200 {

  struct GemmProblem {
    const double* A;
    const double* B;
    double* C;
    int m, n, k;
    int lda, ldb, ldc;
    const int* skip = nullptr;  // optional device flag: problem is a no-op when *skip != 0
    int lower = 0;              // only the lower triangle of C is needed (SYRK-like)
    // per-problem operation (gemm_run_mixed): bit 0 = op(A) transposed,
    // bit 1 = op(B) transposed; C = alpha op(A) op(B) + beta C
    int trans = 0;
    double alpha = 1.0, beta = 0.0;
  };

  inline void gemm_set_op(GemmProblem& g, char ta, char tb, double alpha, double beta) {
    g.trans = (ta != 'N' ? 1 : 0) | (tb != 'N' ? 2 : 0);
    g.alpha = alpha;
    g.beta = beta;
  }

  // device-resident batch: descriptors + tile prefix (prefix[p] = first tile
  // of problem p, prefix[nprob] = total tiles)
  struct GemmBatchDev {
    const GemmProblem* probs = nullptr;
    const int* prefix = nullptr;
    int nprob = 0;
    int tiles = 0;
    double flops = 0;  // 2 m n k summed (probe accounting)
    double ab_bytes = 0;  // 8 (mk + kn) summed: A and B read once (probe accounting)
    double c_elems = 0;   // C elements touched (lower triangle only for SYRK-like problems)
  };

  constexpr int kGemmBM = 64, kGemmBN = 64;

  // tile prefix for the batched tile shape
  std::vector<int> gemm_tile_prefix(const std::vector<GemmProblem>& p);
  double gemm_flops(const std::vector<GemmProblem>& p);
  // algorithmic bytes of a batch: A and B read once, C written (beta == 0) or
  // read and written; the probe's GEMM traffic denominator
  double gemm_ab_bytes(const std::vector<GemmProblem>& p);
  double gemm_c_elems(const std::vector<GemmProblem>& p);
  inline double gemm_bytes(double ab_bytes, double c_elems, double beta) {
    return ab_bytes + c_elems * (beta == 0.0 ? 8.0 : 16.0);
  }

  // ta/tb: 'N' or 'T'. beta == 0 never reads C.
  void gemm_run(const GemmBatchDev& b, char ta, char tb, double alpha, double beta,
                cudaStream_t s);

  // dynamic batches (HSS phases, tests): the descriptors travel as kernel
  // parameters, no upload. gemm_run_host applies one op to every problem;
  // gemm_run_mixed takes each problem's own trans / alpha / beta.
  void gemm_run_host(const std::vector<GemmProblem>& p, char ta, char tb, double alpha,
                     double beta, cudaStream_t s);
  void gemm_run_mixed(const std::vector<GemmProblem>& p, cudaStream_t s);
  // TMA-fed 128 x 128 DMMA kernel (gemm_tma.cu) for big problems whose A and
  // B are 16-byte aligned with even leading dimensions; gemm_run_mixed routes
  // eligible problems there by itself
  bool gemm_tma_eligible(const GemmProblem& g);
  bool gemm_tma_aligned(const GemmProblem& g);  // alignment / size only (no K rule)
  void gemm_tma_run(const std::vector<GemmProblem>& p, cudaStream_t s);

  // one large-K problem with few output tiles: split-K over extra CTAs to fill
  // the resident-CTA waves, partial products reduced in a fixed order
  // (deterministic); falls back to a plain launch when splitting does not pay
  int gemm_splitk_factor(int m, int n, int k, bool tma = false);
  void gemm_run_splitk(const GemmProblem& p, char ta, char tb, double alpha, double beta,
                       cudaStream_t s);

}  // namespace hssmf_b200
