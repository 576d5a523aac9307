// Interpolative decomposition through the Gram matrix (blocked, pivoted
// Cholesky) -- a BLAS3 restatement of the reference's tolerance-truncated
// column-pivoted Householder QR (rrqr_tolerance, rrqr.hpp:32-151).
//
// For Y (d x n) the CPQR pivot at step k is the column of largest residual
// norm after projecting out the k chosen columns; those residual norms are
// exactly the diagonal of the Schur complement of the Gram matrix G = Y^T Y
// after k steps of symmetric pivoted Cholesky, and R = L^T. Stop tests,
// tie-breaking (lowest current position), the rank cap and certification
// follow the reference verbatim; only the arithmetic route differs. G is
// accumulated incrementally across adaptive rounds (new sample columns only),
// so a round costs one rank-dd update plus the factorization, instead of a
// level-2 sweep over d x n per elimination step.
//
// Accuracy: R (hence the ID coefficients) carries kappa(R11)^2 u relative
// error; the engine uses this route only when eps >= 5e-5 (kappa(R11) <~
// 1/eps), where that is below 1e-6 relative. Smaller tolerances use the
// Householder CPQR (cpqr.cuh).
#pragma once

#include <functional>
#include <vector>

#include "common.cuh"

namespace hssmf_b200 {

  constexpr int kGramNB = 64;  // panel width (steps between trailing updates)

  struct GramTask {
    double* G;       // n x n working Gram matrix (ld n), destroyed
    double* L;       // n x kcap Cholesky columns by original index (ld n); columns
                     // below the rank are written in full (0 on pivoted rows)
    double* dg;      // n residual norms^2
    int* flag;       // n pivoted flags (zeroed)
    int* orig_at;    // n: original column at each CPQR position (the ID perm)
    int* pos_of;     // n: inverse of orig_at
    int* state;      // [k, stopped, certified]
    double* r11;     // first pivot norm
    int n, kmax_dim, kmax, kcap;
    // warm start (v2 panels, n <= 8192): the first kw (a multiple of the panel
    // width) pivots are taken, in order, from an earlier ID of the same node
    // (its final orig_at / pos_of arrays) and eliminated as blocked fixed-order
    // steps; the pivot search resumes at step kw
    const int* warm_orig = nullptr;
    const int* warm_pos = nullptr;
    int kw = 0;
    // optional: [pivot norm examined at the stop, r11] (how far from the
    // threshold an ID that hit its cap ended)
    double* pvlast = nullptr;
  };
  constexpr int kGramPanel = 48;  // panel width of the one-row-per-thread kernels

  // runs the factorization of all tasks; returns per task (rank, certified);
  // rank -1: a warm-started task whose fixed-order part broke down (repeat it
  // with kw = 0)
  // after ONE host sync; before_sync may enqueue more device->host reads
  // that the same sync then covers
  // HSSMF_GRAM_TPROBE=1: per-step segment cycles of the panel kernel
  unsigned long long* gram_tprobe();
  void gram_tprobe_report();

  void gram_cholesky_run(const std::vector<GramTask>& tasks, double eps, double abs_tol,
                         cudaStream_t s, std::vector<int>& rank, std::vector<int>& cert,
                         double* flops = nullptr,
                         const std::function<void()>& before_sync = {});

}  // namespace hssmf_b200
