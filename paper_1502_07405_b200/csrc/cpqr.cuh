// Batched tolerance-truncated column-pivoted Householder QR + interpolative
// decomposition (reference rrqr_tolerance / interpolative_decomposition,
// rrqr.hpp:32-194). One CTA per task; Y is overwritten by R (upper part) and
// Householder vectors; the ID coefficients X = R1^-1 R2 are solved by a
// second, column-tiled kernel once the ranks are known.
#pragma once

#include <vector>

#include "common.cuh"

namespace hssmf_b200 {

  struct CpqrTask {
    double* Y;     // m x n, ld ldy (overwritten)
    int m, n, ldy;
    int max_rank;  // < 0: min(m, n)
    int* perm;     // n: perm[i] = original column of pivot i
    double* X;     // rank x (n - rank), ld rank (ID coefficients)
    int* out;      // [rank, certified]
  };

  // CPQR for all tasks (device array), then the ID solve; the ranks are read
  // back to the host (one small D2H) between the two kernels.
  void cpqr_run(const CpqrTask* tasks, int ntask, int max_m, int max_n, double eps,
                double abs_tol, cudaStream_t s);
  void id_solve_run(const CpqrTask* tasks, int ntask, int max_rank, int max_cols,
                    cudaStream_t s);
  // ID coefficients for tasks with known ranks (host copies), blocked by 64:
  // X = R2; for each 64-row block from the bottom, a triangular solve of the
  // block (CTA per 128 columns) and a DMMA GEMM update of the rows above
  // (reference trsm, kernels.hpp:205-244, with the same recursion base)
  // inv_blocks: the 64 x 64 diagonal blocks are inverted first (one launch for
  // all blocks of all tasks) and each block solve becomes a DMMA GEMM with the
  // inverse (Gram route; the Householder route keeps the substitution kernel)
  void id_solve_blocked(const std::vector<CpqrTask>& tasks, const std::vector<int>& ranks,
                        cudaStream_t s, double* flops = nullptr, bool inv_blocks = false);

  // convenience: both phases with an internal rank readback
  void cpqr_id_run(const CpqrTask* tasks, int ntask, int max_m, int max_n, double eps,
                   double abs_tol, cudaStream_t s);

}  // namespace hssmf_b200
