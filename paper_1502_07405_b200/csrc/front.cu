// Dense-front kernels, batched over all fronts of one elimination-tree level.
#include "front.cuh"

#include <algorithm>
#include <stdexcept>

#include "gemm.cuh"

namespace hssmf_b200 {

  namespace {

    __device__ __forceinline__ double* front_at(const FrontDev& f, int i, int j) {
      if (j < f.ns) return f.P + i + (size_t)j * f.m;
      j -= f.ns;
      if (i < f.ns) return f.U + i + (size_t)j * f.ldu;
      return f.C + (i - f.ns) + (size_t)j * f.ldc;
    }

    __device__ __forceinline__ int lower_bound_dev(const int* a, int n, int key) {
      int lo = 0, hi = n;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1; else hi = mid;
      }
      return lo;
    }

    // ownership rule of for_front_entries (multifrontal.hpp:99-119): separator
    // rows take every column >= sep_begin, update rows take separator columns;
    // F22 gets nothing, so each entry of A lands in exactly one front
    __global__ void assemble_sparse_kernel(const FrontDev* __restrict__ fr,
                                           const int* __restrict__ ids,
                                           const int* __restrict__ ptr,
                                           const int* __restrict__ ind,
                                           const double* __restrict__ val) {
      const FrontDev f = fr[ids[blockIdx.x]];
      const int se = f.sep_begin + f.ns;
      for (int r = threadIdx.x; r < f.ns; r += blockDim.x) f.perm[r] = r;
      for (int r = threadIdx.x; r < f.m; r += blockDim.x) {
        if (r < f.ns) {
          const int g = f.sep_begin + r;
          for (int k = ptr[g]; k < ptr[g + 1]; k++) {
            const int gj = ind[k];
            if (gj < f.sep_begin) continue;
            const int lj = gj < se ? gj - f.sep_begin : f.ns + lower_bound_dev(f.upd, f.nu, gj);
            *front_at(f, r, lj) += val[k];
          }
        } else {
          const int g = f.upd[r - f.ns];
          const int b = ptr[g], e = ptr[g + 1];
          for (int k = b + lower_bound_dev(ind + b, e - b, f.sep_begin); k < e; k++) {
            const int gj = ind[k];
            if (gj >= se) break;
            *front_at(f, r, gj - f.sep_begin) += val[k];
          }
        }
      }
    }

    // extend-add (multifrontal.hpp:154-168): warp per child column, child
    // update entries scattered through the position map
    __global__ void extend_add_kernel(const FrontDev* __restrict__ fr,
                                      const int* __restrict__ ids, int nf, int slot,
                                      const long long* __restrict__ colpre, long long ncols) {
      const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
      const int lane = threadIdx.x & 31;
      if (w >= ncols) return;
      int lo = 0, hi = nf - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (colpre[mid] <= w) lo = mid; else hi = mid - 1;
      }
      const FrontDev f = fr[ids[lo]];
      const int ci = slot ? f.child1 : f.child0;
      const int* pos = slot ? f.pos1 : f.pos0;
      const FrontDev c = fr[ci];
      const int bj = (int)(w - colpre[lo]);
      const int tj = pos[bj];
      const double* src = c.C + (size_t)bj * c.ldc;
      if (tj < f.ns) {
        double* dst = f.P + (size_t)tj * f.m;
        for (int bi = lane; bi < c.nu; bi += 32) dst[pos[bi]] += src[bi];
      } else {
        const int j = tj - f.ns;
        double* du = f.U + (size_t)j * f.ldu;
        double* dc = f.C + (size_t)j * f.ldc - f.ns;
        for (int bi = lane; bi < c.nu; bi += 32) {
          const int ti = pos[bi];
          (ti < f.ns ? du : dc)[ti] += src[bi];
        }
      }
    }

    constexpr int PANEL_THREADS = 256;

    // unblocked right-looking LU of panel columns [k, k+nbk) over rows [k, m),
    // pivot search restricted to F11 rows [j, ns): lu_unblocked semantics
    // (lu.hpp:16-44) - first maximum wins, exact zero column -> singular
    __global__ void __launch_bounds__(PANEL_THREADS)
    lu_panel_kernel(const FrontDev* __restrict__ fr, const int* __restrict__ ids, int k,
                    int nb, int* __restrict__ status) {
      const int fid = ids[blockIdx.x];
      const FrontDev f = fr[fid];
      if (f.ns <= k) return;
      const int nbk = min(nb, f.ns - k);
      const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
      __shared__ double sv[PANEL_THREADS / 32];
      __shared__ int si[PANEL_THREADS / 32];
      __shared__ int sp;
      __shared__ double sd;
      double* P = f.P;
      const size_t ld = f.m;
      for (int jj = 0; jj < nbk; jj++) {
        const int j = k + jj;
        double* colj = P + (size_t)j * ld;
        double bv = -1.0;
        int bi = 0x7fffffff;
        for (int i = j + tid; i < f.ns; i += PANEL_THREADS) {
          const double v = fabs(colj[i]);
          if (v > bv) { bv = v; bi = i; }
        }
        warp_argmax(bv, bi);
        if (lane == 0) { sv[warp] = bv; si[warp] = bi; }
        __syncthreads();
        if (tid == 0) {
          double v = sv[0];
          int i = si[0];
          for (int w = 1; w < PANEL_THREADS / 32; w++)
            if (sv[w] > v || (sv[w] == v && si[w] < i)) { v = sv[w]; i = si[w]; }
          if (!(v > 0.0)) {
            // exactly singular column (reference throws SingularMatrixError)
            if (status[fid] < 0) status[fid] = j;
            i = -1;
            f.piv[j] = j;
          } else {
            f.piv[j] = i;
            if (i != j) {
              const int t = f.perm[j];
              f.perm[j] = f.perm[i];
              f.perm[i] = t;
            }
            sd = 1.0 / colj[i];
          }
          sp = i;
        }
        __syncthreads();
        const int p = sp;
        if (p < 0) continue;
        if (p != j && tid < nbk) {
          double* c = P + (size_t)(k + tid) * ld;
          const double t = c[j];
          c[j] = c[p];
          c[p] = t;
        }
        __syncthreads();
        const double d = sd;
        for (int i = j + 1 + tid; i < f.ns; i += PANEL_THREADS) colj[i] *= d;
        __syncthreads();
        // rank-1 update of the remaining panel columns (F11 rows only; the
        // L21 rows follow in l21_kernel as A21 U_kk^-1)
        for (int c = j + 1; c < k + nbk; c++) {
          double* cc = P + (size_t)c * ld;
          const double t = cc[j];
          for (int i = j + 1 + tid; i < f.ns; i += PANEL_THREADS) cc[i] -= colj[i] * t;
        }
        __syncthreads();
      }
    }

    // L21 rows of the panel: x U_kk = a  (row-wise), with the same operation
    // order as the unblocked elimination: x_j = (a_j - sum_c x_c u_cj) * (1/u_jj)
    __global__ void __launch_bounds__(128)
    l21_kernel(const FrontDev* __restrict__ fr, const int* __restrict__ ids, int k, int nb) {
      const FrontDev f = fr[ids[blockIdx.y]];
      if (f.ns <= k || f.nu == 0) return;
      const int nbk = min(nb, f.ns - k);
      __shared__ double Uk[32][33];
      __shared__ double inv[32];
      for (int e = threadIdx.x; e < nbk * nbk; e += blockDim.x) {
        const int r = e % nbk, c = e / nbk;
        Uk[r][c] = f.P[(k + r) + (size_t)(k + c) * f.m];
      }
      __syncthreads();
      if (threadIdx.x < nbk) inv[threadIdx.x] = 1.0 / Uk[threadIdx.x][threadIdx.x];
      __syncthreads();
      const int i = f.ns + blockIdx.x * blockDim.x + threadIdx.x;
      if (i >= f.m) return;
      double* row = f.P + i + (size_t)k * f.m;
      double x[32];
#pragma unroll
      for (int c = 0; c < 32; c++) x[c] = c < nbk ? row[(size_t)c * f.m] : 0.0;
#pragma unroll
      for (int j = 0; j < 32; j++) {
        if (j < nbk) {
          double v = x[j] * inv[j];
          x[j] = v;
#pragma unroll
          for (int c = j + 1; c < 32; c++) x[c] -= v * Uk[j][c];
        }
      }
#pragma unroll
      for (int c = 0; c < 32; c++)
        if (c < nbk) row[(size_t)c * f.m] = x[c];
    }

    constexpr int TRSM_COLS = 128;

    // row interchanges of the panel's pivots applied to every other column of
    // the front's F11 rows (laswp, dense_matrix.hpp:172-188), then the unit
    // lower block-row solve U12_k = L_kk^-1 X_k for trailing P and U columns
    __global__ void __launch_bounds__(TRSM_COLS)
    swap_trsm_kernel(const FrontDev* __restrict__ fr, const int* __restrict__ ids, int k,
                     int nb) {
      const FrontDev f = fr[ids[blockIdx.y]];
      if (f.ns <= k) return;
      const int nbk = min(nb, f.ns - k);
      const int total = f.m - nbk;
      __shared__ double L[32][33];
      __shared__ int pv[32];
      if (threadIdx.x < nbk) pv[threadIdx.x] = f.piv[k + threadIdx.x];
      for (int e = threadIdx.x; e < nbk * nbk; e += TRSM_COLS) {
        const int r = e % nbk, c = e / nbk;
        L[r][c] = f.P[(k + r) + (size_t)(k + c) * f.m];
      }
      __syncthreads();
      const int c = blockIdx.x * TRSM_COLS + threadIdx.x;
      if (c >= total) return;
      double* col;
      bool solve;
      if (c < k) { col = f.P + (size_t)c * f.m; solve = false; }
      else if (c < f.ns - nbk) { col = f.P + (size_t)(c + nbk) * f.m; solve = true; }
      else { col = f.U + (size_t)(c - (f.ns - nbk)) * f.ldu; solve = true; }
      for (int jj = 0; jj < nbk; jj++) {
        const int p = pv[jj], j = k + jj;
        if (p != j) {
          const double t = col[j];
          col[j] = col[p];
          col[p] = t;
        }
      }
      if (!solve) return;
      double x[32];
#pragma unroll
      for (int r = 0; r < 32; r++) x[r] = r < nbk ? col[k + r] : 0.0;
#pragma unroll
      for (int r = 1; r < 32; r++) {
        double s = x[r];
#pragma unroll
        for (int q = 0; q < r; q++) s -= L[r][q] * x[q];
        x[r] = s;
      }
#pragma unroll
      for (int r = 0; r < 32; r++)
        if (r < nbk) col[k + r] = x[r];
    }

    // ---- solve ---------------------------------------------------------------
    __global__ void fold_kernel(const FrontDev* __restrict__ fr, const int* __restrict__ ids,
                                int slot, double* __restrict__ x, int ldx) {
      const FrontDev f = fr[ids[blockIdx.y]];
      const int ci = slot ? f.child1 : f.child0;
      if (ci < 0) return;
      const FrontDev c = fr[ci];
      const int* pos = slot ? f.pos1 : f.pos0;
      const int a = blockIdx.x * blockDim.x + threadIdx.x;
      if (a >= c.nu) return;
      const int r = blockIdx.z;
      const int t = pos[a];
      const double v = c.bupd[a + (size_t)r * c.nu];
      if (t < f.ns) x[f.sep_begin + t + (size_t)r * ldx] += v;
      else f.bupd[(t - f.ns) + (size_t)r * f.nu] += v;
    }

    constexpr int TRSV_THREADS = 256;

    // b1 <- L11^-1 P b1 in shared memory, blocked by 32 (warp solves the
    // diagonal block, the CTA updates the rows below)
    __global__ void __launch_bounds__(TRSV_THREADS)
    fwd_trsv_kernel(const FrontDev* __restrict__ fr, const int* __restrict__ ids,
                    double* __restrict__ x, int ldx) {
      extern __shared__ double xs[];
      const FrontDev f = fr[ids[blockIdx.x]];
      if (!f.ns) return;
      double* xg = x + f.sep_begin + (size_t)blockIdx.y * ldx;
      for (int i = threadIdx.x; i < f.ns; i += TRSV_THREADS) xs[i] = xg[f.perm[i]];
      __syncthreads();
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      for (int jb = 0; jb < f.ns; jb += 32) {
        const int bs = min(32, f.ns - jb);
        if (warp == 0) {
          double xv = lane < bs ? xs[jb + lane] : 0.0;
          for (int c = 0; c < bs - 1; c++) {
            const double xc = __shfl_sync(0xffffffffu, xv, c);
            if (lane > c && lane < bs) xv -= f.P[(jb + lane) + (size_t)(jb + c) * f.m] * xc;
          }
          if (lane < bs) xs[jb + lane] = xv;
        }
        __syncthreads();
        for (int i = jb + bs + threadIdx.x; i < f.ns; i += TRSV_THREADS) {
          double s = xs[i];
          for (int c = 0; c < bs; c++) s -= f.P[i + (size_t)(jb + c) * f.m] * xs[jb + c];
          xs[i] = s;
        }
        __syncthreads();
      }
      for (int i = threadIdx.x; i < f.ns; i += TRSV_THREADS) xg[i] = xs[i];
    }

    // bupd -= L21 x1
    __global__ void fwd_gemv_kernel(const FrontDev* __restrict__ fr,
                                    const int* __restrict__ ids, const double* __restrict__ x,
                                    int ldx) {
      const FrontDev f = fr[ids[blockIdx.y]];
      const int r = blockIdx.x * blockDim.x + threadIdx.x;
      if (r >= f.nu || !f.ns) return;
      const double* x1 = x + f.sep_begin + (size_t)blockIdx.z * ldx;
      const double* L = f.P + f.ns + r;
      double s = 0.0;
      for (int c = 0; c < f.ns; c++) s += L[(size_t)c * f.m] * x1[c];
      f.bupd[r + (size_t)blockIdx.z * f.nu] -= s;
    }

    // x1 -= U12 x2, x2 = x(upd)
    __global__ void bwd_gemv_kernel(const FrontDev* __restrict__ fr,
                                    const int* __restrict__ ids, double* __restrict__ x,
                                    int ldx) {
      const FrontDev f = fr[ids[blockIdx.y]];
      const int r = blockIdx.x * blockDim.x + threadIdx.x;
      if (r >= f.ns || !f.nu) return;
      double* xr = x + (size_t)blockIdx.z * ldx;
      double s = 0.0;
      for (int c = 0; c < f.nu; c++) s += f.U[r + (size_t)c * f.ldu] * xr[f.upd[c]];
      xr[f.sep_begin + r] -= s;
    }

    // x1 <- U11^-1 x1
    __global__ void __launch_bounds__(TRSV_THREADS)
    bwd_trsv_kernel(const FrontDev* __restrict__ fr, const int* __restrict__ ids,
                    double* __restrict__ x, int ldx) {
      extern __shared__ double xs[];
      const FrontDev f = fr[ids[blockIdx.x]];
      if (!f.ns) return;
      double* xg = x + f.sep_begin + (size_t)blockIdx.y * ldx;
      for (int i = threadIdx.x; i < f.ns; i += TRSV_THREADS) xs[i] = xg[i];
      __syncthreads();
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      const int nblk = (f.ns + 31) / 32;
      for (int b = nblk - 1; b >= 0; b--) {
        const int jb = b * 32, bs = min(32, f.ns - jb);
        if (warp == 0) {
          double xv = lane < bs ? xs[jb + lane] : 0.0;
          for (int c = bs - 1; c >= 0; c--) {
            if (lane == c) xv = xv / f.P[(jb + c) + (size_t)(jb + c) * f.m];
            const double xc = __shfl_sync(0xffffffffu, xv, c);
            if (lane < c) xv -= f.P[(jb + lane) + (size_t)(jb + c) * f.m] * xc;
          }
          if (lane < bs) xs[jb + lane] = xv;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < jb; i += TRSV_THREADS) {
          double s = xs[i];
          for (int c = 0; c < bs; c++) s -= f.P[i + (size_t)(jb + c) * f.m] * xs[jb + c];
          xs[i] = s;
        }
        __syncthreads();
      }
      for (int i = threadIdx.x; i < f.ns; i += TRSV_THREADS) xg[i] = xs[i];
    }

    constexpr int kMaxTrsvSmem = 200 * 1024;

    void set_smem_attr() {
      static std::atomic<unsigned long long> done{0};
      once_per_device(done, [] {
      HSSMF_CUDA(cudaFuncSetAttribute(fwd_trsv_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxTrsvSmem));
      HSSMF_CUDA(cudaFuncSetAttribute(bwd_trsv_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxTrsvSmem));
      });
    }

  }  // namespace

  void DenseKernels::assemble_sparse(const FrontDev* f, const int* ids, int nf, const int* ptr,
                                     const int* ind, const double* val, cudaStream_t s) {
    if (!nf) return;
    assemble_sparse_kernel<<<nf, 128, 0, s>>>(f, ids, ptr, ind, val);
    HSSMF_LAUNCH_CHECK();
  }

  void DenseKernels::extend_add(const FrontDev* f, const int* ids, int nf, int slot,
                                const long long* colpre, long long ncols, cudaStream_t s) {
    if (!nf || !ncols) return;
    const long long threads = ncols * 32;
    extend_add_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(f, ids, nf, slot,
                                                                         colpre, ncols);
    HSSMF_LAUNCH_CHECK();
  }

  void DenseKernels::lu_panel(const FrontDev* f, const int* ids, int nf, int k, int nb,
                              int* status, cudaStream_t s) {
    if (!nf) return;
    lu_panel_kernel<<<nf, PANEL_THREADS, 0, s>>>(f, ids, k, nb, status);
    HSSMF_LAUNCH_CHECK();
  }

  void DenseKernels::l21(const FrontDev* f, const int* ids, int nf, int k, int nb, int max_nu,
                         cudaStream_t s) {
    if (!nf || max_nu <= 0) return;
    l21_kernel<<<dim3(ceil_div(max_nu, 128), nf), 128, 0, s>>>(f, ids, k, nb);
    HSSMF_LAUNCH_CHECK();
  }

  void DenseKernels::swap_trsm(const FrontDev* f, const int* ids, int nf, int k, int nb,
                               int max_cols, cudaStream_t s) {
    if (!nf || max_cols <= 0) return;
    dim3 grid(ceil_div(max_cols, TRSM_COLS), nf);
    swap_trsm_kernel<<<grid, TRSM_COLS, 0, s>>>(f, ids, k, nb);
    HSSMF_LAUNCH_CHECK();
  }

  void DenseKernels::fold_children(const FrontDev* f, const int* ids, int nf, int slot,
                                   double* x, int ldx, int nrhs, int max_nu, cudaStream_t s) {
    if (!nf || max_nu <= 0) return;
    dim3 grid(ceil_div(max_nu, 256), nf, nrhs);
    fold_kernel<<<grid, 256, 0, s>>>(f, ids, slot, x, ldx);
    HSSMF_LAUNCH_CHECK();
  }

  void DenseKernels::fwd_trsv(const FrontDev* f, const int* ids, int nf, double* x, int ldx,
                              int nrhs, int max_ns, cudaStream_t s) {
    if (!nf || max_ns <= 0) return;
    if ((size_t)max_ns * 8 > (size_t)kMaxTrsvSmem)
      throw std::runtime_error("dense front separator too large for the smem solve");
    set_smem_attr();
    fwd_trsv_kernel<<<dim3(nf, nrhs), TRSV_THREADS, max_ns * 8, s>>>(f, ids, x, ldx);
    HSSMF_LAUNCH_CHECK();
  }

  void DenseKernels::fwd_gemv(const FrontDev* f, const int* ids, int nf, double* x, int ldx,
                              int nrhs, int max_nu, cudaStream_t s) {
    if (!nf || max_nu <= 0) return;
    fwd_gemv_kernel<<<dim3(ceil_div(max_nu, 128), nf, nrhs), 128, 0, s>>>(f, ids, x, ldx);
    HSSMF_LAUNCH_CHECK();
  }

  void DenseKernels::bwd_gemv(const FrontDev* f, const int* ids, int nf, double* x, int ldx,
                              int nrhs, int max_ns, cudaStream_t s) {
    if (!nf || max_ns <= 0) return;
    bwd_gemv_kernel<<<dim3(ceil_div(max_ns, 128), nf, nrhs), 128, 0, s>>>(f, ids, x, ldx);
    HSSMF_LAUNCH_CHECK();
  }

  void DenseKernels::bwd_trsv(const FrontDev* f, const int* ids, int nf, double* x, int ldx,
                              int nrhs, int max_ns, cudaStream_t s) {
    if (!nf || max_ns <= 0) return;
    if ((size_t)max_ns * 8 > (size_t)kMaxTrsvSmem)
      throw std::runtime_error("dense front separator too large for the smem solve");
    set_smem_attr();
    bwd_trsv_kernel<<<dim3(nf, nrhs), TRSV_THREADS, max_ns * 8, s>>>(f, ids, x, ldx);
    HSSMF_LAUNCH_CHECK();
  }

  namespace {
    __global__ void init_perm_kernel(const FrontDev* __restrict__ fr) {
      const FrontDev f = fr[blockIdx.x];
      for (int r = threadIdx.x; r < f.ns; r += blockDim.x) f.perm[r] = r;
    }
  }  // namespace

  std::vector<int> partial_lu_dynamic(const std::vector<FrontDev>& fronts, cudaStream_t s,
                                      double* flops) {
    const int nf = (int)fronts.size();
    std::vector<int> st(nf, -1);
    if (!nf) return st;
    int max_ns = 0, max_nu = 0;
    for (const auto& h : fronts) {
      max_ns = std::max(max_ns, h.ns);
      max_nu = std::max(max_nu, h.nu);
    }
    std::vector<int> ids(nf);
    for (int i = 0; i < nf; i++) ids[i] = i;
    const size_t fb = nf * sizeof(FrontDev), ib = nf * sizeof(int);
    char* d = nullptr;
    HSSMF_CUDA(cudaMallocAsync((void**)&d, fb + 2 * ib, s));
    FrontDev* F = reinterpret_cast<FrontDev*>(d);
    int* dids = reinterpret_cast<int*>(d + fb);
    int* dst = reinterpret_cast<int*>(d + fb + ib);
    HSSMF_CUDA(cudaMemcpyAsync(F, fronts.data(), fb, cudaMemcpyHostToDevice, s));
    HSSMF_CUDA(cudaMemcpyAsync(dids, ids.data(), ib, cudaMemcpyHostToDevice, s));
    HSSMF_CUDA(cudaMemsetAsync(dst, 0xff, ib, s));
    init_perm_kernel<<<nf, 128, 0, s>>>(F);
    HSSMF_LAUNCH_CHECK();
    const int NB = 32;
    double fl = 0;
    for (int k = 0; k < max_ns; k += NB) {
      int max_cols = 0;
      std::vector<GemmProblem> probs;
      for (const auto& h : fronts) {
        if (h.ns <= k) continue;
        const int nbk = std::min(NB, h.ns - k), k1 = k + nbk;
        max_cols = std::max(max_cols, h.m - nbk);
        if (h.ns > k1) {
          probs.push_back({h.P + k1 + (size_t)k * h.m, h.P + k + (size_t)k1 * h.m,
                           h.P + k1 + (size_t)k1 * h.m, h.m - k1, h.ns - k1, nbk, h.m, h.m, h.m});
          if (h.nu)
            probs.push_back({h.P + k1 + (size_t)k * h.m, h.U + k, h.U + k1, h.ns - k1, h.nu, nbk,
                             h.m, h.ldu, h.ldu});
        }
      }
      DenseKernels::lu_panel(F, dids, nf, k, NB, dst, s);
      DenseKernels::l21(F, dids, nf, k, NB, max_nu, s);
      DenseKernels::swap_trsm(F, dids, nf, k, NB, max_cols, s);
      fl += gemm_flops(probs);
      gemm_run_host(probs, 'N', 'N', -1.0, 1.0, s);
    }
    std::vector<GemmProblem> probs;
    for (const auto& h : fronts)
      if (h.ns && h.nu) probs.push_back({h.P + h.ns, h.U, h.C, h.nu, h.nu, h.ns, h.m, h.ldu, h.ldc});
    fl += gemm_flops(probs);
    gemm_run_host(probs, 'N', 'N', -1.0, 1.0, s);
    HSSMF_CUDA(cudaMemcpyAsync(st.data(), dst, ib, cudaMemcpyDeviceToHost, s));
    HSSMF_CUDA(cudaFreeAsync(d, s));
    HSSMF_CUDA(cudaStreamSynchronize(s));
    if (flops) *flops += fl;
    return st;
  }

}  // namespace hssmf_b200
