#include "kernels_test.hpp"

#include <cstring>

#include <cstdlib>
#include <stdexcept>
#include <vector>

#include "cpqr.cuh"
#include "engine.hpp"
#include "front.cuh"
#include "gemm.cuh"
#include "gram_id.cuh"
#include "rng.cuh"

namespace hssmf_b200 {

  namespace {
    struct Buf {
      void* p = nullptr;
      explicit Buf(size_t b) { HSSMF_CUDA(cudaMalloc(&p, b ? b : 8)); }
      ~Buf() { cudaFree(p); }
      template<typename T> T* as() { return static_cast<T*>(p); }
    };
  }  // namespace

  void test_random_rows(int device, int nrows, const long long* grow, int c0, int c1,
                        double* out) {
    HSSMF_CUDA(cudaSetDevice(device));
    Buf g(nrows * sizeof(long long)), o((size_t)nrows * (c1 - c0) * sizeof(double));
    HSSMF_CUDA(cudaMemcpy(g.p, grow, nrows * sizeof(long long), cudaMemcpyHostToDevice));
    rng_fill(g.as<long long>(), 0, nrows, c0, c1, o.as<double>(), nrows, 0);
    HSSMF_CUDA(cudaMemcpy(out, o.p, (size_t)nrows * (c1 - c0) * sizeof(double),
                          cudaMemcpyDeviceToHost));
  }

  void test_gemm(int device, char ta, char tb, int m, int n, int k, double alpha,
                 const double* a, int lda, const double* b, int ldb, double beta, double* c,
                 int ldc) {
    HSSMF_CUDA(cudaSetDevice(device));
    const size_t na = (size_t)lda * (ta == 'N' ? k : m), nb = (size_t)ldb * (tb == 'N' ? n : k),
                 nc = (size_t)ldc * n;
    Buf A(na * 8), B(nb * 8), C(nc * 8);
    HSSMF_CUDA(cudaMemcpy(A.p, a, na * 8, cudaMemcpyHostToDevice));
    HSSMF_CUDA(cudaMemcpy(B.p, b, nb * 8, cudaMemcpyHostToDevice));
    HSSMF_CUDA(cudaMemcpy(C.p, c, nc * 8, cudaMemcpyHostToDevice));
    // single problems go through the split-K path (a plain launch when
    // splitting does not pay), which is how the HSS sampling products run
    gemm_run_splitk({A.as<double>(), B.as<double>(), C.as<double>(), m, n, k, lda, ldb, ldc}, ta,
                    tb, alpha, beta, 0);
    HSSMF_CUDA(cudaMemcpy(c, C.p, nc * 8, cudaMemcpyDeviceToHost));
  }

  void test_id(int device, const double* y, int m, int n, double eps, int max_rank,
               double abs_tol, int* perm, int* rank, int* certified, double* coeffs) {
    HSSMF_CUDA(cudaSetDevice(device));
    Buf Y((size_t)m * n * 8), X((size_t)std::min(m, n) * n * 8), P(n * 4), R(16);
    HSSMF_CUDA(cudaMemcpy(Y.p, y, (size_t)m * n * 8, cudaMemcpyHostToDevice));
    CpqrTask t{Y.as<double>(), m, n, m, max_rank, P.as<int>(), X.as<double>(), R.as<int>()};
    Buf T(sizeof(CpqrTask));
    HSSMF_CUDA(cudaMemcpy(T.p, &t, sizeof(t), cudaMemcpyHostToDevice));
    cpqr_id_run(T.as<CpqrTask>(), 1, m, n, eps, abs_tol, 0);
    int rc[2];
    HSSMF_CUDA(cudaMemcpy(rc, R.p, 2 * sizeof(int), cudaMemcpyDeviceToHost));
    HSSMF_CUDA(cudaMemcpy(perm, P.p, n * 4, cudaMemcpyDeviceToHost));
    *rank = rc[0];
    *certified = rc[1];
    if (rc[0] && n > rc[0])
      HSSMF_CUDA(cudaMemcpy(coeffs, X.p, (size_t)rc[0] * (n - rc[0]) * 8,
                            cudaMemcpyDeviceToHost));
  }

  // Gram route of the ID (gram_id.cuh): G = Y^T Y (lower triangle), pivoted
  // Cholesky with the CPQR stop rules; returns the permutation, rank,
  // certification and R = L^T (rank x n, columns in position order)
  void test_gram_id(int device, const double* y, int m, int n, double eps, int max_rank,
                    double abs_tol, int* perm, int* rank, int* certified, double* r) {
    HSSMF_CUDA(cudaSetDevice(device));
    Buf Y((size_t)m * n * 8), G((size_t)n * n * 8);
    HSSMF_CUDA(cudaMemcpy(Y.p, y, (size_t)m * n * 8, cudaMemcpyHostToDevice));
    if (n && m) {
      GemmProblem g{Y.as<double>(), Y.as<double>(), G.as<double>(), n, n, m, m, m, n};
      g.lower = 1;
      gemm_run_host({g}, 'T', 'N', 1.0, 0.0, 0);
    }
    const int kdim = std::min(m, n), kmax = max_rank < 0 ? kdim : std::min(kdim, max_rank);
    const int kcap = ((kmax + kGramNB - 1) / kGramNB) * kGramNB + kGramNB;
    Buf L((size_t)n * kcap * 8), dg((size_t)n * 8), fl((size_t)n * 4), pos((size_t)n * 4),
        P((size_t)n * 4), st(12), r11(8);
    GramTask t{G.as<double>(), L.as<double>(), dg.as<double>(), fl.as<int>(), P.as<int>(),
               pos.as<int>(), st.as<int>(), r11.as<double>(), n, kdim, kmax, kcap};
    std::vector<int> rk, ce;
    gram_cholesky_run({t}, eps, abs_tol, 0, rk, ce);
    HSSMF_CUDA(cudaDeviceSynchronize());
    *rank = rk[0];
    *certified = ce[0];
    HSSMF_CUDA(cudaMemcpy(perm, P.p, (size_t)n * 4, cudaMemcpyDeviceToHost));
    const int k = rk[0];
    if (k) {
      std::vector<double> hl((size_t)n * k);
      HSSMF_CUDA(cudaMemcpy(hl.data(), L.p, hl.size() * 8, cudaMemcpyDeviceToHost));
      for (int j = 0; j < n; j++)
        for (int q = 0; q < k; q++) r[q + (size_t)j * k] = hl[perm[j] + (size_t)q * n];
    }
  }

  void test_lu(int device, double* a, int m, int n, int* piv) {
    if (m != n) throw std::invalid_argument("dev lu: square matrices only");
    HSSMF_CUDA(cudaSetDevice(device));
    Buf A((size_t)m * n * 8), I(2 * n * 4 + 16), F(sizeof(FrontDev)), S(8);
    HSSMF_CUDA(cudaMemcpy(A.p, a, (size_t)m * n * 8, cudaMemcpyHostToDevice));
    std::vector<int> id(n);
    for (int i = 0; i < n; i++) id[i] = i;
    HSSMF_CUDA(cudaMemcpy(I.as<int>() + n, id.data(), n * 4, cudaMemcpyHostToDevice));
    FrontDev f{};
    f.ns = n;
    f.nu = 0;
    f.m = n;
    f.ldu = n;
    f.ldc = 1;
    f.child0 = f.child1 = -1;
    f.P = A.as<double>();
    f.piv = I.as<int>();
    f.perm = I.as<int>() + n;
    HSSMF_CUDA(cudaMemcpy(F.p, &f, sizeof(f), cudaMemcpyHostToDevice));
    int zero = 0, neg = -1;
    HSSMF_CUDA(cudaMemcpy(S.p, &zero, 4, cudaMemcpyHostToDevice));
    HSSMF_CUDA(cudaMemcpy(S.as<int>() + 1, &neg, 4, cudaMemcpyHostToDevice));
    const int* ids = S.as<int>();
    int* status = S.as<int>() + 1;  // front id 0 -> status[0]
    for (int k = 0; k < n; k += 32) {
      DenseKernels::lu_panel(F.as<FrontDev>(), ids, 1, k, 32, status, 0);
      DenseKernels::swap_trsm(F.as<FrontDev>(), ids, 1, k, 32, n, 0);
      const int nbk = std::min(32, n - k), k1 = k + nbk;
      if (n > k1) {
        std::vector<GemmProblem> p{{f.P + k1 + (size_t)k * n, f.P + k + (size_t)k1 * n,
                                    f.P + k1 + (size_t)k1 * n, n - k1, n - k1, nbk, n, n, n}};
        gemm_run_host(p, 'N', 'N', -1.0, 1.0, 0);
      }
    }
    int st = -1;
    HSSMF_CUDA(cudaMemcpy(&st, status, 4, cudaMemcpyDeviceToHost));
    if (st >= 0) throw SolverFailure(3, 0, st, "lu_partial_pivot: exactly singular, zero pivot column " + std::to_string(st));
    HSSMF_CUDA(cudaMemcpy(a, A.p, (size_t)m * n * 8, cudaMemcpyDeviceToHost));
    HSSMF_CUDA(cudaMemcpy(piv, I.p, n * 4, cudaMemcpyDeviceToHost));
  }

  double bench_gemm(int device, int m, int n, int k, int iters) {
    HSSMF_CUDA(cudaSetDevice(device));
    Buf A((size_t)m * k * 8), B((size_t)k * n * 8), C((size_t)m * n * 8);
    HSSMF_CUDA(cudaMemset(A.p, 0, (size_t)m * k * 8));
    HSSMF_CUDA(cudaMemset(B.p, 0, (size_t)k * n * 8));
    HSSMF_CUDA(cudaMemset(C.p, 0, (size_t)m * n * 8));
    // HSSMF_BENCH_TRANS=TN|NT|TT selects the operand transposes (measurement only)
    char ta = 'N', tb = 'N';
    if (const char* e = getenv("HSSMF_BENCH_TRANS")) {
      ta = e[0];
      tb = e[1];
    }
    const int lda = ta == 'N' ? m : k, ldb = tb == 'N' ? k : n;
    std::vector<GemmProblem> p{{A.as<double>(), B.as<double>(), C.as<double>(), m, n, k, lda, ldb, m}};
    auto pre = gemm_tile_prefix(p);
    Buf D(sizeof(GemmProblem) + pre.size() * 4);
    HSSMF_CUDA(cudaMemcpy(D.p, p.data(), sizeof(GemmProblem), cudaMemcpyHostToDevice));
    HSSMF_CUDA(cudaMemcpy((char*)D.p + sizeof(GemmProblem), pre.data(), pre.size() * 4, cudaMemcpyHostToDevice));
    GemmBatchDev b{D.as<GemmProblem>(), (const int*)((char*)D.p + sizeof(GemmProblem)), 1, pre.back()};
    // HSSMF_BENCH_PATH=mixed: the dynamic-batch entry (TMA kernel for
    // eligible problems), =splitk: the split-K entry of the sampling products
    const char* path = getenv("HSSMF_BENCH_PATH");
    const int mode = !path ? 0 : !strcmp(path, "mixed") ? 1 : !strcmp(path, "splitk") ? 2 : 0;
    auto run = [&] {
      if (mode == 1) gemm_run_host(p, ta, tb, 1.0, 1.0, 0);
      else if (mode == 2) gemm_run_splitk(p[0], ta, tb, 1.0, 1.0, 0);
      else gemm_run(b, ta, tb, 1.0, 1.0, 0);
    };
    run();
    HSSMF_CUDA(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    HSSMF_CUDA(cudaEventCreate(&e0));
    HSSMF_CUDA(cudaEventCreate(&e1));
    HSSMF_CUDA(cudaEventRecord(e0, 0));
    for (int i = 0; i < iters; i++) run();
    HSSMF_CUDA(cudaEventRecord(e1, 0));
    HSSMF_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    HSSMF_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return ms / iters;
  }

  double bench_gram(int device, int n, int d, int ntask, int iters, int* steps) {
    HSSMF_CUDA(cudaSetDevice(device));
    // S: n x d pseudo-random (host LCG), G0 = S S^T (lower triangle)
    std::vector<double> hs((size_t)n * d);
    unsigned long long x = 88172645463325252ull;
    for (auto& v : hs) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      v = (double)(x >> 11) / 9007199254740992.0 - 0.5;
    }
    Buf S(hs.size() * 8), G0((size_t)n * n * 8);
    HSSMF_CUDA(cudaMemcpy(S.p, hs.data(), hs.size() * 8, cudaMemcpyHostToDevice));
    GemmProblem g{S.as<double>(), S.as<double>(), G0.as<double>(), n, n, d, n, n, n};
    g.lower = 1;
    gemm_run_host({g}, 'N', 'T', 1.0, 0.0, 0);
    const int kdim = std::min(n, d), kmax = kdim;
    const int kcap = ((kmax + kGramNB - 1) / kGramNB) * kGramNB + kGramNB;
    Buf Gw((size_t)n * n * 8 * ntask), L((size_t)n * kcap * 8 * ntask), dg((size_t)n * 8 * ntask),
        fl((size_t)n * 4 * ntask), pos((size_t)n * 4 * ntask), perm((size_t)n * 4 * ntask),
        st(12 * ntask), r11(8 * ntask);
    std::vector<GramTask> tasks(ntask);
    for (int t = 0; t < ntask; t++)
      tasks[t] = {Gw.as<double>() + (size_t)t * n * n, L.as<double>() + (size_t)t * n * kcap,
                  dg.as<double>() + (size_t)t * n, fl.as<int>() + (size_t)t * n,
                  perm.as<int>() + (size_t)t * n, pos.as<int>() + (size_t)t * n,
                  st.as<int>() + 3 * t, r11.as<double>() + t, n, kdim, kmax, kcap};
    std::vector<int> rk, ce;
    auto once = [&] {
      for (int t = 0; t < ntask; t++)
        HSSMF_CUDA(cudaMemcpyAsync(tasks[t].G, G0.p, (size_t)n * n * 8, cudaMemcpyDeviceToDevice, 0));
      gram_cholesky_run(tasks, 1e-14, 0.0, 0, rk, ce);
    };
    once();
    HSSMF_CUDA(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    HSSMF_CUDA(cudaEventCreate(&e0));
    HSSMF_CUDA(cudaEventCreate(&e1));
    HSSMF_CUDA(cudaEventRecord(e0, 0));
    for (int i = 0; i < iters; i++) once();
    HSSMF_CUDA(cudaEventRecord(e1, 0));
    HSSMF_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    HSSMF_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *steps = rk.empty() ? 0 : rk[0];
    gram_tprobe_report();
    return ms / iters;
  }

}  // namespace hssmf_b200
