// Accurate residual of the Gram-route ID at its last step (rrqr.hpp:67-77's
// stop test, evaluated without the Gram matrix's cancellation).
//
// The Gram route (gram_id.cu) reads the CPQR residual norms of the sample rows
// off the diagonal of the Schur complement of G = S S^T. Near the stop of a
// large node that diagonal is a difference of numbers about 1/eps^2 larger
// than itself, so its rounding is of the order of the stop threshold: at
// BASELINE config 5 (eps 1e-4, nodes of 6000-8000 rows) the top nodes of three
// fronts certified 1-3 adaptive rounds after the reference did. This check
// recomputes the residual after k pivots directly: with J the first k pivot
// rows, the residual of row i is the projection of s_i on the orthogonal
// complement of span(S_J) (dimension w = d - k, about p = 10 at the cap), so
//   pv(k) = max_{i not in J} || W^T s_i ||,  W = orthonormal basis of span(S_J)^perp.
// W comes from w seeded Gaussian vectors projected twice against span(S_J)
// (normal equations with the Gram route's own Cholesky factor L_JJ, whose
// error only enters relative to the projected vectors) and orthonormalised.
#include "tail_check.cuh"

#include <cmath>

#include "gemm.cuh"
#include "hss_kernels.cuh"
#include "rng.cuh"

namespace hssmf_b200 {

  namespace {
    // packed LU of G_JJ = L_JJ L_JJ^T (unit lower L_JJ D^-1, upper D L_JJ^T),
    // L_JJ(i, j) = L(orig[i], j): the layout lu_solve_vec reads
    __global__ void chol_to_lu_kernel(const double* __restrict__ L, long long ldl,
                                      const int* __restrict__ orig, int k, double* __restrict__ M) {
      const long long tot = (long long)k * k;
      for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot;
           e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e % k), j = (int)(e / k);
        double v;
        if (i > j) v = L[orig[i] + (size_t)j * ldl] / L[orig[j] + (size_t)j * ldl];
        else v = L[orig[i] + (size_t)i * ldl] * L[orig[j] + (size_t)i * ldl];
        M[e] = v;
      }
    }

    // modified Gram-Schmidt, twice, on the w columns of Z (d x w, ld d), one CTA
    __global__ void __launch_bounds__(512) mgs2_kernel(double* Z, int d, int w) {
      __shared__ double red[16];
      __shared__ double bc;
      const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
      auto dot = [&](const double* a, const double* b) {
        double s = 0.0;
        for (int i = tid; i < d; i += blockDim.x) s += a[i] * b[i];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) red[warp] = s;
        __syncthreads();
        if (tid == 0) {
          double t = 0.0;
          for (int q = 0; q < nw; q++) t += red[q];
          bc = t;
        }
        __syncthreads();
        const double r = bc;
        __syncthreads();
        return r;
      };
      for (int pass = 0; pass < 2; pass++)
        for (int j = 0; j < w; j++) {
          double* zj = Z + (size_t)j * d;
          for (int l = 0; l < j; l++) {
            const double* zl = Z + (size_t)l * d;
            const double c = dot(zl, zj);
            for (int i = tid; i < d; i += blockDim.x) zj[i] -= c * zl[i];
            __syncthreads();
          }
          const double nrm = sqrt(dot(zj, zj));
          const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
          for (int i = tid; i < d; i += blockDim.x) zj[i] *= inv;
          __syncthreads();
        }
    }

    // max over rows i not among orig[0..k) of sum_c P(i, c)^2, one CTA
    __global__ void __launch_bounds__(1024) masked_rowmax_kernel(const double* __restrict__ P,
                                                                 long long ldp, int mt, int w,
                                                                 const int* __restrict__ orig,
                                                                 int k, double* out) {
      extern __shared__ unsigned char piv[];
      __shared__ double red[32];
      const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
      for (int i = tid; i < mt; i += blockDim.x) piv[i] = 0;
      __syncthreads();
      for (int j = tid; j < k; j += blockDim.x) piv[orig[j]] = 1;
      __syncthreads();
      double m = 0.0;
      for (int i = tid; i < mt; i += blockDim.x) {
        if (piv[i]) continue;
        double s = 0.0;
        for (int c = 0; c < w; c++) {
          const double v = P[i + (size_t)c * ldp];
          s += v * v;
        }
        m = fmax(m, s);
      }
      for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) red[warp] = m;
      __syncthreads();
      if (tid == 0) {
        double t = 0.0;
        for (int q = 0; q < (int)(blockDim.x >> 5); q++) t = fmax(t, red[q]);
        *out = t;
      }
    }
    __global__ void __launch_bounds__(1024) dg_max_kernel(const double* __restrict__ dg,
                                                          const int* __restrict__ flag, int n,
                                                          double* out) {
      __shared__ double red[32];
      const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
      double m = 0.0;
      for (int i = tid; i < n; i += blockDim.x)
        if (!flag[i]) m = fmax(m, dg[i]);
      for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) red[warp] = m;
      __syncthreads();
      if (tid == 0) {
        double t = 0.0;
        for (int q = 0; q < (int)(blockDim.x >> 5); q++) t = fmax(t, red[q]);
        *out = t;
      }
    }
  }  // namespace

  void gram_dg_max(const double* dg, const int* flag, int n, double* out, cudaStream_t s) {
    dg_max_kernel<<<1, 1024, 0, s>>>(dg, flag, n, out);
    HSSMF_LAUNCH_CHECK();
  }

  void gram_tail_residual2(const double* S, long long lds, int mt, int d, const double* L,
                           long long ldl, const int* orig, int k, double* out,
                           cudaStream_t s) {
    const int w = d - k;
    if (w <= 0 || k <= 0 || mt <= k) {
      HSSMF_CUDA(cudaMemsetAsync(out, 0, sizeof(double), s));
      return;
    }
    double *M = nullptr, *Z = nullptr, *SJ = nullptr, *Y = nullptr, *P = nullptr;
    HSSMF_CUDA(cudaMallocAsync((void**)&M, (size_t)k * k * sizeof(double), s));
    HSSMF_CUDA(cudaMallocAsync((void**)&Z, (size_t)d * w * sizeof(double), s));
    HSSMF_CUDA(cudaMallocAsync((void**)&SJ, (size_t)k * d * sizeof(double), s));
    HSSMF_CUDA(cudaMallocAsync((void**)&Y, (size_t)k * w * sizeof(double), s));
    HSSMF_CUDA(cudaMallocAsync((void**)&P, (size_t)mt * w * sizeof(double), s));
    {
      const long long tot = (long long)k * k;
      chol_to_lu_kernel<<<(int)std::min<long long>((tot + 255) / 256, 148 * 16), 256, 0, s>>>(
          L, ldl, orig, k, M);
      HSSMF_LAUNCH_CHECK();
    }
    // seeded Gaussian start block (rows named 2^30 + i: streams the samples
    // never use)
    rng_fill(nullptr, 1LL << 30, d, 0, w, Z, d, s);
    // S_J = rows orig[0..k) of S (k x d)
    index_copy_run({CopyDesc{S, 1, lds, orig, nullptr, 0, 0, SJ, k, nullptr, nullptr, 0, 0, k, d,
                             1.0, 0, 0}},
                   s);
    for (int pass = 0; pass < 2; pass++) {
      // Y = S_J Z; Y <- G_JJ^-1 Y; Z <- Z - S_J^T Y
      GemmProblem g1{SJ, Z, Y, k, w, d, k, d, k};
      gemm_run_host({g1}, 'N', 'N', 1.0, 0.0, s);
      for (int c = 0; c < w; c++) lu_solve_vec(M, k, nullptr, k, Y + (size_t)c * k, s);
      GemmProblem g2{SJ, Y, Z, d, w, k, k, k, d};
      gemm_run_host({g2}, 'T', 'N', -1.0, 1.0, s);
    }
    mgs2_kernel<<<1, 512, 0, s>>>(Z, d, w);
    HSSMF_LAUNCH_CHECK();
    // P = S W (mt x w), residual norms of the non-pivot rows
    GemmProblem g3{S, Z, P, mt, w, d, (int)lds, d, mt};
    gemm_run_host({g3}, 'N', 'N', 1.0, 0.0, s);
    masked_rowmax_kernel<<<1, 1024, (size_t)mt, s>>>(P, mt, mt, w, orig, k, out);
    HSSMF_LAUNCH_CHECK();
    for (void* p : {(void*)M, (void*)Z, (void*)SJ, (void*)Y, (void*)P})
      HSSMF_CUDA(cudaFreeAsync(p, s));
  }

}  // namespace hssmf_b200
