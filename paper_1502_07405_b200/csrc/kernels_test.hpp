// Host-buffer wrappers that run single device kernels for the parity tests
// (hssmf_dev_* entry points of include/hssmf_b200.h).
#pragma once

namespace hssmf_b200 {
  void test_random_rows(int device, int nrows, const long long* grow, int c0, int c1,
                        double* out);
  void test_gemm(int device, char ta, char tb, int m, int n, int k, double alpha,
                 const double* a, int lda, const double* b, int ldb, double beta, double* c,
                 int ldc);
  void test_id(int device, const double* y, int m, int n, double eps, int max_rank,
               double abs_tol, int* perm, int* rank, int* certified, double* coeffs);
  void test_gram_id(int device, const double* y, int m, int n, double eps, int max_rank,
                    double abs_tol, int* perm, int* rank, int* certified, double* r);
  void test_lu(int device, double* a, int m, int n, int* piv);
  double bench_gemm(int device, int m, int n, int k, int iters);
  // pivoted-Cholesky ID kernel timing: ntask tasks of an n x n Gram matrix of
  // rank min(n, d); returns ms per batch, *steps = pivots taken
  double bench_gram(int device, int n, int d, int ntask, int iters, int* steps);
}  // namespace hssmf_b200
