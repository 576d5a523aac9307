// Device-resident restarted GMRES and iterative refinement preconditioned by
// the multifrontal solve (reference krylov.hpp:93-232, the paper's use of the
// HSS-multifrontal factorization as a preconditioner).
//
// The algorithm is the reference's, step for step: left preconditioning,
// zero initial guess, modified Gram-Schmidt Arnoldi, Givens rotations,
// restart from the true preconditioned residual u = M^-1 (b - A x), stop at
// |u| <= atol or |u|/|u0| <= rtol, happy breakdown, non-finite Arnoldi
// entry -> KrylovDivergence; refinement x += u with stagnation (< 2x
// reduction over 3 steps) flagged. Vectors, the Krylov basis, SpMV and the
// preconditioner solves stay in HBM; only the Hessenberg scalars (one dot
// product at a time, as MGS needs them) travel to the host.
#pragma once

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>
#include <vector>

namespace hssmf_b200 {

  class Engine;

  struct KrylovDivergence : std::runtime_error {
    explicit KrylovDivergence(const std::string& m) : std::runtime_error(m) {}
  };

  struct KrylovReport {
    int iterations = 0;
    double rel_resid = 0, abs_resid = 0;
    bool converged = false, stagnated = false;
    std::vector<double> history;
  };

  // y = A x for a device CSR (n x n, int32 ptr/ind)
  struct CsrDevView {
    int n = 0;
    const int* ptr = nullptr;
    const int* ind = nullptr;
    const double* val = nullptr;
  };

  // m == nullptr: identity preconditioner (reference tests use one).
  // b, x: device vectors of length n; x is overwritten with the solution.
  KrylovReport krylov_gmres(const CsrDevView& a, Engine* m, const double* b, double* x,
                            int restart, double rtol, double atol, int maxit, cudaStream_t s);
  KrylovReport krylov_refine(const CsrDevView& a, Engine* m, const double* b, double* x,
                             double rtol, double atol, int maxit, cudaStream_t s);

}  // namespace hssmf_b200
