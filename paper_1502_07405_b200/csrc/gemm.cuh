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
  };

  // device-resident batch: descriptors + tile prefix (prefix[p] = first tile
  // of problem p, prefix[nprob] = total tiles)
  struct GemmBatchDev {
    const GemmProblem* probs = nullptr;
    const int* prefix = nullptr;
    int nprob = 0;
    int tiles = 0;
  };

  constexpr int kGemmBM = 64, kGemmBN = 64;

  // tile prefix for the batched tile shape
  std::vector<int> gemm_tile_prefix(const std::vector<GemmProblem>& p);
  double gemm_flops(const std::vector<GemmProblem>& p);

  // ta/tb: 'N' or 'T'. beta == 0 never reads C.
  void gemm_run(const GemmBatchDev& b, char ta, char tb, double alpha, double beta,
                cudaStream_t s);

  // one-off convenience: uploads descriptors synchronously into a temporary
  // device buffer (tests / dynamic HSS phases), then launches
  struct DevBuffer;
  void gemm_run_host(const std::vector<GemmProblem>& p, char ta, char tb, double alpha,
                     double beta, cudaStream_t s);

}  // namespace hssmf_b200
