// Accurate stop-test residual of the Gram-route ID (tail_check.cu).
#pragma once

#include "common.cuh"

namespace hssmf_b200 {

  // *out = max over the non-pivot rows i (not among orig[0..k)) of
  // ||P_perp s_i||^2, P_perp the projector on span(S_J)^perp, S_J the rows
  // orig[0..k) of S (mt x d, ld lds); L (mt x >= k, ld ldl) is the Gram route's
  // Cholesky factor (row = sample row, column = step). Device result.
  void gram_tail_residual2(const double* S, long long lds, int mt, int d, const double* L,
                           long long ldl, const int* orig, int k, double* out, cudaStream_t s);
  // *out = max of dg[i] over the rows with flag[i] == 0 (the Gram route's own
  // squared residual after its last step)
  void gram_dg_max(const double* dg, const int* flag, int n, double* out, cudaStream_t s);

}  // namespace hssmf_b200
