#include "hss_kernels.cuh"

#include <algorithm>

#include "staging.cuh"

namespace hssmf_b200 {

  namespace {
    constexpr int CPB = 1024;  // elements per block for index_copy

    constexpr int kParamCopies = 64;
    struct CopyParam {
      int nd;
      long long pre[kParamCopies + 1];
      CopyDesc d[kParamCopies];
    };

    // descriptors in a __grid_constant__ parameter block (no upload)
    __global__ void index_copy_kernel(const __grid_constant__ CopyParam P) {
      const CopyDesc* ds = P.d;
      const long long* pre = P.pre;
      const int nd = P.nd;
      int lo = 0, hi = nd - 1;
      const long long b = blockIdx.x;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (pre[mid] <= b) lo = mid; else hi = mid - 1;
      }
      const CopyDesc d = ds[lo];
      const long long base = (b - pre[lo]) * CPB;
      const long long tot = d.diag ? d.nr : (long long)d.nr * d.nc;
      for (long long e = base + threadIdx.x; e < base + CPB && e < tot; e += blockDim.x) {
        const int i = d.diag ? (int)e : (int)(e % d.nr), j = d.diag ? (int)e : (int)(e / d.nr);
        const long long si = d.sr ? d.sr[i] : d.sr_off + i;
        const long long sj = d.sc ? d.sc[j] : d.sc_off + j;
        const long long di = d.dr ? d.dr[i] : d.dr_off + i;
        const long long dj = d.dc ? d.dc[j] : d.dc_off + j;
        const double v = d.alpha * d.src[si * d.srs + sj * d.scs];
        double* o = d.dst + di + dj * d.ldd;
        *o = d.accumulate ? *o + v : v;
      }
    }

    constexpr int kParamSegs = 128;
    struct SegParam {
      int ns;
      IntSeg g[kParamSegs];
    };
    __global__ void int_gather_kernel(const __grid_constant__ SegParam P, int* __restrict__ dst) {
      const IntSeg& g = P.g[blockIdx.y];
      for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += gridDim.x * blockDim.x)
        dst[g.off + i] = g.src[i];
    }

    __global__ void maxabs_kernel(const double* __restrict__ a, long long lda, int m, int n,
                                  unsigned long long* out) {
      double mx = 0;
      const long long tot = (long long)m * n;
      for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < tot;
           e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e % m), j = (int)(e / m);
        mx = fmax(mx, fabs(a[i + j * lda]));
      }
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      __shared__ double sm[32];
      if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = mx;
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); w++) mx = fmax(mx, sm[w]);
        atomicMax(out, (unsigned long long)__double_as_longlong(mx));
      }
    }

    constexpr int UT = 256;

    // forward ULV step of one node (fwd, hss_ulv.hpp:226-248)
    __global__ void __launch_bounds__(UT)
    ulv_fwd_kernel(const UlvSolveNode* __restrict__ nodes) {
      extern __shared__ double sm[];
      const UlvSolveNode N = nodes[blockIdx.x];
      const int m = N.m, r = N.r, k = N.k;
      double* y = sm;
      double* o = sm + m;
      for (int i = threadIdx.x; i < m; i += UT) y[i] = i < N.n0 ? N.in0[i] : N.in1[i - N.n0];
      __syncthreads();
      // omega: [y_rest - E y_skel ; y_skel]
      for (int j = threadIdx.x; j < m; j += UT) {
        if (j < k) {
          double s = y[N.uperm[r + j]];
          for (int i = 0; i < r; i++) s -= N.Eu[j + (size_t)i * k] * y[N.uperm[i]];
          o[j] = s;
        } else {
          o[j] = y[N.uperm[j - k]];
        }
      }
      __syncthreads();
      if (k == 0) {
        for (int i = threadIdx.x; i < r; i += UT) N.fout[i] = o[i];
        return;
      }
      // z = L^-1 P o[0:k]  (y reused as z)
      for (int i = threadIdx.x; i < k; i += UT) y[i] = o[N.lperm[i]];
      __syncthreads();
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      const double* G = N.G;
      for (int jb = 0; jb < k; jb += 32) {
        const int bs = min(32, k - jb);
        if (warp == 0) {
          double xv = lane < bs ? y[jb + lane] : 0.0;
          for (int c = 0; c < bs - 1; c++) {
            const double xc = __shfl_sync(0xffffffffu, xv, c);
            if (lane > c && lane < bs) xv -= G[(jb + lane) + (size_t)(jb + c) * m] * xc;
          }
          if (lane < bs) y[jb + lane] = xv;
        }
        __syncthreads();
        for (int i = jb + bs + threadIdx.x; i < k; i += UT) {
          double s = y[i];
          for (int c = 0; c < bs; c++) s -= G[i + (size_t)(jb + c) * m] * y[jb + c];
          y[i] = s;
        }
        __syncthreads();
      }
      for (int i = threadIdx.x; i < k; i += UT) N.ws[i] = y[i];
      // ret = o[k:m] - L21 z
      for (int i = threadIdx.x; i < r; i += UT) {
        double s = o[k + i];
        for (int c = 0; c < k; c++) s -= G[(k + i) + (size_t)c * m] * y[c];
        N.fout[i] = s;
      }
    }

    // backward ULV step of one node (bwd, hss_ulv.hpp:250-276)
    __global__ void __launch_bounds__(UT)
    ulv_bwd_kernel(const UlvSolveNode* __restrict__ nodes) {
      extern __shared__ double sm[];
      const UlvSolveNode N = nodes[blockIdx.x];
      const int m = N.m, r = N.r, k = N.k;
      double* xh = sm;
      for (int i = threadIdx.x; i < r; i += UT) xh[k + i] = N.xkeep[i];
      __syncthreads();
      const double* G = N.G;
      if (k) {
        for (int i = threadIdx.x; i < k; i += UT) {
          double s = N.ws[i];
          for (int c = 0; c < r; c++) s -= G[i + (size_t)(k + c) * m] * xh[k + c];
          xh[i] = s;
        }
        __syncthreads();
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const int nblk = (k + 31) / 32;
        for (int b = nblk - 1; b >= 0; b--) {
          const int jb = b * 32, bs = min(32, k - jb);
          if (warp == 0) {
            double xv = lane < bs ? xh[jb + lane] : 0.0;
            for (int c = bs - 1; c >= 0; c--) {
              if (lane == c) xv = xv / G[(jb + c) + (size_t)(jb + c) * m];
              const double xc = __shfl_sync(0xffffffffu, xv, c);
              if (lane < c) xv -= G[(jb + lane) + (size_t)(jb + c) * m] * xc;
            }
            if (lane < bs) xh[jb + lane] = xv;
          }
          __syncthreads();
          for (int i = threadIdx.x; i < jb; i += UT) {
            double s = xh[i];
            for (int c = 0; c < bs; c++) s -= G[i + (size_t)(jb + c) * m] * xh[jb + c];
            xh[i] = s;
          }
          __syncthreads();
        }
      }
      __syncthreads();
      // psi: x(vperm[i<r]) = xh[k+i] - (Ev^T xh[0:k])(i); x(vperm[r+j]) = xh[j]
      for (int t = threadIdx.x; t < m; t += UT) {
        double v;
        int dst;
        if (t < r) {
          v = xh[k + t];
          for (int j = 0; j < k; j++) v -= N.Ev[j + (size_t)t * k] * xh[j];
          dst = N.vperm[t];
        } else {
          v = xh[t - r];
          dst = N.vperm[t];
        }
        if (dst < N.n0) N.out0[dst] = v; else N.out1[dst - N.n0] = v;
      }
    }

    __global__ void __launch_bounds__(UT)
    lu_solve_vec_kernel(const double* __restrict__ lu, int ld, const int* __restrict__ perm,
                        int n, double* __restrict__ x) {
      extern __shared__ double y[];
      for (int i = threadIdx.x; i < n; i += UT) y[i] = x[perm[i]];
      __syncthreads();
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      for (int jb = 0; jb < n; jb += 32) {
        const int bs = min(32, n - jb);
        if (warp == 0) {
          double xv = lane < bs ? y[jb + lane] : 0.0;
          for (int c = 0; c < bs - 1; c++) {
            const double xc = __shfl_sync(0xffffffffu, xv, c);
            if (lane > c && lane < bs) xv -= lu[(jb + lane) + (size_t)(jb + c) * ld] * xc;
          }
          if (lane < bs) y[jb + lane] = xv;
        }
        __syncthreads();
        for (int i = jb + bs + threadIdx.x; i < n; i += UT) {
          double s = y[i];
          for (int c = 0; c < bs; c++) s -= lu[i + (size_t)(jb + c) * ld] * y[jb + c];
          y[i] = s;
        }
        __syncthreads();
      }
      const int nblk = (n + 31) / 32;
      for (int b = nblk - 1; b >= 0; b--) {
        const int jb = b * 32, bs = min(32, n - jb);
        if (warp == 0) {
          double xv = lane < bs ? y[jb + lane] : 0.0;
          for (int c = bs - 1; c >= 0; c--) {
            if (lane == c) xv = xv / lu[(jb + c) + (size_t)(jb + c) * ld];
            const double xc = __shfl_sync(0xffffffffu, xv, c);
            if (lane < c) xv -= lu[(jb + lane) + (size_t)(jb + c) * ld] * xc;
          }
          if (lane < bs) y[jb + lane] = xv;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < jb; i += UT) {
          double s = y[i];
          for (int c = 0; c < bs; c++) s -= lu[i + (size_t)(jb + c) * ld] * y[jb + c];
          y[i] = s;
        }
        __syncthreads();
      }
      for (int i = threadIdx.x; i < n; i += UT) x[i] = y[i];
    }

    __global__ void gemv_n_kernel(int m, int n, double alpha, const double* __restrict__ A,
                                  int lda, const double* __restrict__ x, double beta,
                                  double* __restrict__ y) {
      const int i = blockIdx.x * blockDim.x + threadIdx.x;
      if (i >= m) return;
      double s = 0;
      for (int c = 0; c < n; c++) s += A[i + (size_t)c * lda] * x[c];
      y[i] = (beta == 0.0 ? 0.0 : beta * y[i]) + alpha * s;
    }

    __global__ void gemv_t_kernel(int m, int n, double alpha, const double* __restrict__ A,
                                  int lda, const double* __restrict__ x, double beta,
                                  double* __restrict__ y) {
      // y(i) for i < n: column i of A dotted with x (m entries); warp per output
      const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
      if (w >= n) return;
      double s = 0;
      for (int r = lane; r < m; r += 32) s += A[r + (size_t)w * lda] * x[r];
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) y[w] = (beta == 0.0 ? 0.0 : beta * y[w]) + alpha * s;
    }

    void set_attr() {
      static bool done = false;
      if (done) return;
      HSSMF_CUDA(cudaFuncSetAttribute(ulv_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      HSSMF_CUDA(cudaFuncSetAttribute(ulv_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      HSSMF_CUDA(cudaFuncSetAttribute(lu_solve_vec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      done = true;
    }

    // device copy of a host array: through the thread's staging ring when it
    // serves this stream (no free needed), else a stream-ordered allocation
    template<typename T> struct Up {
      T* p;
      bool owned;
    };
    template<typename T> Up<T> upload_async(const std::vector<T>& v, cudaStream_t s) {
      if (Staging* st = current_staging(s))
        if (!v.empty())
          if (void* p = st->put(v.data(), v.size() * sizeof(T)))
            return {static_cast<T*>(p), false};
      T* d = nullptr;
      HSSMF_CUDA(cudaMallocAsync((void**)&d, std::max<size_t>(v.size() * sizeof(T), 16), s));
      HSSMF_CUDA(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
      return {d, true};
    }
    template<typename T> void release_async(const Up<T>& u, cudaStream_t s) {
      if (u.owned) HSSMF_CUDA(cudaFreeAsync(u.p, s));
    }
  }  // namespace

  void index_copy_run(const std::vector<CopyDesc>& d0, cudaStream_t s) {
    CopyParam P;
    P.nd = 0;
    P.pre[0] = 0;
    auto flush = [&] {
      if (!P.nd) return;
      index_copy_kernel<<<(unsigned)P.pre[P.nd], 256, 0, s>>>(P);
      HSSMF_LAUNCH_CHECK();
      P.nd = 0;
    };
    // descriptors of one call write disjoint outputs: long lists are split
    for (const auto& x : d0) {
      if (x.nr <= 0 || (x.nc <= 0 && !x.diag)) continue;
      if (P.nd == kParamCopies) flush();
      P.d[P.nd] = x;
      P.pre[P.nd + 1] =
          P.pre[P.nd] + ((x.diag ? (long long)x.nr : (long long)x.nr * x.nc) + CPB - 1) / CPB;
      P.nd++;
    }
    flush();
  }

  void int_gather_run(const std::vector<IntSeg>& segs, int* dst, cudaStream_t s) {
    SegParam P;
    P.ns = 0;
    int maxn = 0;
    auto flush = [&] {
      if (!P.ns) return;
      int_gather_kernel<<<dim3(std::min(ceil_div(maxn, 256), 64), P.ns), 256, 0, s>>>(P, dst);
      HSSMF_LAUNCH_CHECK();
      P.ns = 0;
      maxn = 0;
    };
    for (const auto& g : segs) {
      if (g.n <= 0) continue;
      if (P.ns == kParamSegs) flush();
      P.g[P.ns++] = g;
      maxn = std::max(maxn, g.n);
    }
    flush();
  }

  void maxabs_run(const double* a, long long lda, int m, int n, double* out, cudaStream_t s) {
    if (m <= 0 || n <= 0) return;
    const long long tot = (long long)m * n;
    const int blocks = (int)std::min<long long>((tot + 255) / 256, 148 * 8);
    maxabs_kernel<<<blocks, 256, 0, s>>>(a, lda, m, n, (unsigned long long*)out);
    HSSMF_LAUNCH_CHECK();
  }

  void ulv_fwd_level(const std::vector<UlvSolveNode>& nodes, int, cudaStream_t s) {
    if (nodes.empty()) return;
    set_attr();
    int mmax = 0;
    for (auto& n : nodes) mmax = std::max(mmax, n.m);
    if ((size_t)mmax * 16 > 200 * 1024) throw CudaError("ulv solve: node too large for smem");
    auto d = upload_async(nodes, s);
    ulv_fwd_kernel<<<(unsigned)nodes.size(), UT, (size_t)mmax * 16, s>>>(d.p);
    HSSMF_LAUNCH_CHECK();
    release_async(d, s);
  }

  void ulv_bwd_level(const std::vector<UlvSolveNode>& nodes, cudaStream_t s) {
    if (nodes.empty()) return;
    set_attr();
    int mmax = 0;
    for (auto& n : nodes) mmax = std::max(mmax, n.m);
    if ((size_t)mmax * 8 > 200 * 1024) throw CudaError("ulv solve: node too large for smem");
    auto d = upload_async(nodes, s);
    ulv_bwd_kernel<<<(unsigned)nodes.size(), UT, (size_t)mmax * 8, s>>>(d.p);
    HSSMF_LAUNCH_CHECK();
    release_async(d, s);
  }

  void lu_solve_vec(const double* lu, int ld, const int* perm, int n, double* x, cudaStream_t s) {
    if (n <= 0) return;
    set_attr();
    if ((size_t)n * 8 > 200 * 1024) throw CudaError("lu solve: block too large for smem");
    lu_solve_vec_kernel<<<1, UT, (size_t)n * 8, s>>>(lu, ld, perm, n, x);
    HSSMF_LAUNCH_CHECK();
  }

  void gemv_run(char ta, int m, int n, double alpha, const double* A, int lda, const double* x,
                double beta, double* y, cudaStream_t s) {
    if (ta == 'N') {
      if (m <= 0) return;
      gemv_n_kernel<<<ceil_div(m, 128), 128, 0, s>>>(m, n, alpha, A, lda, x, beta, y);
    } else {
      if (n <= 0) return;
      gemv_t_kernel<<<ceil_div((long long)n * 32, 256), 256, 0, s>>>(m, n, alpha, A, lda, x,
                                                                      beta, y);
    }
    HSSMF_LAUNCH_CHECK();
  }

}  // namespace hssmf_b200
