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

    __global__ void diag_gather_kernel(const double* __restrict__ L, int n, const int* __restrict__ perm,
                                       int k, double* __restrict__ out) {
      const int j = blockIdx.x * blockDim.x + threadIdx.x;
      if (j < k) out[j] = L[perm[j] + (size_t)j * n];
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

    // asymmetry of a dense front: out[0] = max_{i>j} |a(i,j) - a(j,i)|,
    // out[1] = max |a(i,j)| (non-negative doubles compare as their bits)
    __global__ void asymmetry_kernel(const double* __restrict__ a, long long lda, int m,
                                     unsigned long long* out) {
      const long long tot = (long long)m * m;
      double da = 0.0, mx = 0.0;
      for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < tot;
           e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e % m), j = (int)(e / m);
        const double x = a[i + j * lda];
        mx = fmax(mx, fabs(x));
        if (i > j) da = fmax(da, fabs(x - a[j + i * lda]));
      }
      for (int o = 16; o > 0; o >>= 1) {
        da = fmax(da, __shfl_xor_sync(0xffffffffu, da, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      }
      if ((threadIdx.x & 31) == 0) {
        atomicMax(out, (unsigned long long)__double_as_longlong(da));
        atomicMax(out + 1, (unsigned long long)__double_as_longlong(mx));
      }
    }

    // strict upper triangle of the n x n matrix a (ld) := transpose of its
    // strict lower triangle, 32 x 32 tiles through shared memory
    __global__ void mirror_lower_kernel(double* a, long long ld, int n) {
      __shared__ double t[32][33];
      const int bi = blockIdx.y, bj = blockIdx.x;  // destination tile (bi < bj or diagonal)
      if (bi > bj) return;
      const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
      // source tile (bj, bi) of the lower triangle
      for (int r = ty; r < 32; r += 8) {
        const int i = bj * 32 + tx, j = bi * 32 + r;
        t[r][tx] = (i < n && j < n) ? a[i + (size_t)j * ld] : 0.0;
      }
      __syncthreads();
      for (int r = ty; r < 32; r += 8) {
        const int i = bi * 32 + tx, j = bj * 32 + r;  // destination (i, j), i < j
        if (i < n && j < n && i < j) a[i + (size_t)j * ld] = t[tx][r];
      }
    }

    constexpr int UT = 256;

    // ---- batched ULV sweep phases (see ulv_fwd_level / ulv_bwd_level) -------
    // omega: o[j<k] = y[uperm[r+j]] - sum_i Eu(j,i) y[uperm[i]], o[k+i] =
    // y[uperm[i]], y = [in0[0:n0]; in1]; the skeleton values are staged in
    // shared memory in chunks. k == 0: fout = o directly.
    __global__ void __launch_bounds__(256) ulv_fwd_omega_kernel(const UlvSolveNode* __restrict__ nodes) {
      const UlvSolveNode& N = nodes[blockIdx.y];
      const int m = N.m, r = N.r, k = N.k;
      const int j = blockIdx.x * 256 + threadIdx.x;
      if ((int)(blockIdx.x * 256) >= m) return;
      auto y = [&](int q) { return q < N.n0 ? N.in0[q] : N.in1[q - N.n0]; };
      __shared__ double ys[1024];
      double s0 = 0.0, s1 = 0.0;
      if (j < k) s0 = y(N.uperm[r + j]);
      for (int i0 = 0; i0 < r && (int)(blockIdx.x * 256) < k; i0 += 1024) {
        const int nc = min(1024, r - i0);
        __syncthreads();
        for (int i = threadIdx.x; i < nc; i += 256) ys[i] = y(N.uperm[i0 + i]);
        __syncthreads();
        if (j < k) {
          const double* E = N.Eu + j + (size_t)i0 * k;
          int i = 0;
          for (; i + 1 < nc; i += 2) {
            s0 -= E[(size_t)i * k] * ys[i];
            s1 -= E[(size_t)(i + 1) * k] * ys[i + 1];
          }
          if (i < nc) s0 -= E[(size_t)i * k] * ys[i];
        }
      }
      if (j >= m) return;
      const double v = j < k ? s0 + s1 : y(N.uperm[j - k]);
      if (k == 0) N.fout[j] = v;
      else N.scr[j] = v;
    }

    // z = L11^-1 P o[0:k] in shared memory, one CTA per node (k <= kmax_cta)
    __global__ void __launch_bounds__(UT) ulv_fwd_lsolve_kernel(const UlvSolveNode* __restrict__ nodes,
                                                                int kmax_cta) {
      extern __shared__ double z[];
      const UlvSolveNode& N = nodes[blockIdx.x];
      const int m = N.m, k = N.k;
      if (k == 0 || k > kmax_cta) return;
      for (int i = threadIdx.x; i < k; i += UT) z[i] = N.scr[N.lperm[i]];
      __syncthreads();
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      const double* G = N.G;
      for (int jb = 0; jb < k; jb += 32) {
        const int bs = min(32, k - jb);
        if (warp == 0) {
          double xv = lane < bs ? z[jb + lane] : 0.0;
          for (int c = 0; c < bs - 1; c++) {
            const double xc = __shfl_sync(0xffffffffu, xv, c);
            if (lane > c && lane < bs) xv -= G[(jb + lane) + (size_t)(jb + c) * m] * xc;
          }
          if (lane < bs) z[jb + lane] = xv;
        }
        __syncthreads();
        for (int i = jb + bs + threadIdx.x; i < k; i += UT) {
          double s = z[i];
          for (int c = 0; c < bs; c++) s -= G[i + (size_t)(jb + c) * m] * z[jb + c];
          z[i] = s;
        }
        __syncthreads();
      }
      for (int i = threadIdx.x; i < k; i += UT) N.ws[i] = z[i];
    }

    // fout = o[k:m] - L21 z
    __global__ void __launch_bounds__(256) ulv_fwd_l21_kernel(const UlvSolveNode* __restrict__ nodes) {
      const UlvSolveNode& N = nodes[blockIdx.y];
      const int m = N.m, r = N.r, k = N.k;
      const int i = blockIdx.x * 256 + threadIdx.x;
      if (k == 0 || i >= r) return;
      const double* G = N.G + (k + i);
      const double* z = N.ws;
      double s0 = N.scr[k + i], s1 = 0.0;
      int c = 0;
      for (; c + 1 < k; c += 2) {
        s0 -= G[(size_t)c * m] * z[c];
        s1 -= G[(size_t)(c + 1) * m] * z[c + 1];
      }
      if (c < k) s0 -= G[(size_t)c * m] * z[c];
      N.fout[i] = s0 + s1;
    }

    // rhs = ws - U12 xkeep  -> scr[0:k]
    __global__ void __launch_bounds__(256) ulv_bwd_u12_kernel(const UlvSolveNode* __restrict__ nodes) {
      const UlvSolveNode& N = nodes[blockIdx.y];
      const int m = N.m, r = N.r, k = N.k;
      const int i = blockIdx.x * 256 + threadIdx.x;
      if (i >= k) return;
      const double* G = N.G + i + (size_t)k * m;
      double s0 = N.ws[i], s1 = 0.0;
      int c = 0;
      for (; c + 1 < r; c += 2) {
        s0 -= G[(size_t)c * m] * N.xkeep[c];
        s1 -= G[(size_t)(c + 1) * m] * N.xkeep[c + 1];
      }
      if (c < r) s0 -= G[(size_t)c * m] * N.xkeep[c];
      N.scr[i] = s0 + s1;
    }

    // sol = U11^-1 rhs -> scr[k:2k], one CTA per node (k <= kmax_cta)
    __global__ void __launch_bounds__(UT) ulv_bwd_usolve_kernel(const UlvSolveNode* __restrict__ nodes,
                                                                int kmax_cta) {
      extern __shared__ double xh[];
      const UlvSolveNode& N = nodes[blockIdx.x];
      const int m = N.m, k = N.k;
      if (k == 0 || k > kmax_cta) return;
      for (int i = threadIdx.x; i < k; i += UT) xh[i] = N.scr[i];
      __syncthreads();
      const double* G = N.G;
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
      for (int i = threadIdx.x; i < k; i += UT) N.scr[k + i] = xh[i];
    }

    // psi: x(vperm[t<r]) = xkeep[t] - (Ev^T sol)(t), x(vperm[r+j]) = sol[j];
    // one warp per output entry
    __global__ void __launch_bounds__(256) ulv_bwd_psi_kernel(const UlvSolveNode* __restrict__ nodes) {
      const UlvSolveNode& N = nodes[blockIdx.y];
      const int m = N.m, r = N.r, k = N.k;
      const int t = (int)((blockIdx.x * 256 + threadIdx.x) >> 5), lane = threadIdx.x & 31;
      if (t >= m) return;
      const double* sol = N.scr + k;
      double v;
      if (t < r) {
        double s = 0.0;
        const double* E = N.Ev + (size_t)t * k;
        for (int j = lane; j < k; j += 32) s += E[j] * sol[j];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        v = N.xkeep[t] - s;
      } else {
        v = sol[t - r];
      }
      if (lane == 0) {
        const int dst = N.vperm[t];
        if (dst < N.n0) N.out0[dst] = v;
        else N.out1[dst - N.n0] = v;
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

    // ---- chained blocked triangular solve (large factors) ------------------
    // x = T^-1 rhs over the n x n diagonal block of A (ld): T unit lower
    // (LOWER, rows top-down) or non-unit upper (rows bottom-up). One CTA per
    // TB-row block; blocks are claimed in dependency order through an atomic
    // ticket and finish in that order, so a single completion counter tells a
    // block which solution blocks it may already subtract. Each block folds in
    // the finished blocks as they appear (the bulk of the matrix traffic
    // overlaps the chain), then solves its diagonal block in one warp (two rows
    // per lane) and publishes. rhs[i] = in[gperm ? gperm[i] : i]; out != in.
    // sync[0] = ticket, sync[1] = finished blocks (zeroed by the caller).
    constexpr int TB = 64;
    __device__ __forceinline__ int ld_acquire(const int* p) {
      int v;
      asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
      return v;
    }
    template <bool LOWER>
    __global__ void __launch_bounds__(256)
    trsv_chain_kernel(const double* __restrict__ A, int ld, int n, const double* in,
                      const int* __restrict__ gperm, double* out, int* sync) {
      __shared__ int s_t, s_avail;
      __shared__ double red[4][TB];
      __shared__ double D[TB][TB + 1];
      const int nb = (n + TB - 1) / TB;
      if (threadIdx.x == 0) s_t = atomicAdd(sync, 1);
      __syncthreads();
      const int t = s_t;
      const int b = LOWER ? t : nb - 1 - t;
      const int r0 = b * TB, rows = min(TB, n - r0);
      const int row = threadIdx.x & (TB - 1), part = threadIdx.x / TB;
      // own diagonal block into shared memory (column-major tile, padded)
      for (int e = threadIdx.x; e < TB * TB; e += blockDim.x) {
        const int i = e % TB, c = e / TB;
        D[i][c] = (i < rows && c < rows) ? A[(r0 + i) + (size_t)(r0 + c) * ld] : 0.0;
      }
      double acc = 0.0;
      int done = 0;
      while (done < t) {
        if (threadIdx.x == 0) {
          int a;
          while ((a = ld_acquire(sync + 1)) <= done) __nanosleep(32);
          s_avail = a < t ? a : t;
        }
        __syncthreads();
        const int avail = s_avail;
        if (row < rows)
          for (int q = done; q < avail; q++) {
            const int j = LOWER ? q : nb - 1 - q;
            const int c0 = j * TB, cols = min(TB, n - c0);
            const double* Ar = A + (r0 + row) + (size_t)c0 * ld;
            for (int c = part; c < cols; c += 4) acc += Ar[(size_t)c * ld] * __ldcg(out + c0 + c);
          }
        done = avail;
        __syncthreads();
      }
      red[part][row] = acc;
      __syncthreads();
      if (threadIdx.x < 32) {
        const int lane = threadIdx.x, i0 = lane, i1 = lane + 32;
        auto rhs = [&](int i) {
          const int gi = r0 + i;
          return in[gperm ? gperm[gi] : gi] - (red[0][i] + red[1][i] + red[2][i] + red[3][i]);
        };
        double y0 = i0 < rows ? rhs(i0) : 0.0, y1 = i1 < rows ? rhs(i1) : 0.0;
        if (LOWER) {
          for (int c = 0; c < rows - 1; c++) {
            const double xc = __shfl_sync(0xffffffffu, c < 32 ? y0 : y1, c & 31);
            if (i0 > c && i0 < rows) y0 -= D[i0][c] * xc;
            if (i1 > c && i1 < rows) y1 -= D[i1][c] * xc;
          }
        } else {
          for (int c = rows - 1; c >= 0; c--) {
            if (lane == (c & 31)) {
              if (c < 32) y0 /= D[c][c];
              else y1 /= D[c][c];
            }
            const double xc = __shfl_sync(0xffffffffu, c < 32 ? y0 : y1, c & 31);
            if (i0 < c) y0 -= D[i0][c] * xc;
            if (i1 < c) y1 -= D[i1][c] * xc;
          }
        }
        if (i0 < rows) out[r0 + i0] = y0;
        if (i1 < rows) out[r0 + i1] = y1;
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(sync + 1, 1);
      }
    }

    // ---- GEMV y = beta y + alpha A x split over column chunks: partial sums
    // per chunk, then one deterministic reduction in chunk order ------------
    constexpr int GV_ROWS = 256, GV_COLS = 256;
    __global__ void gemv_n_part_kernel(int m, int n, const double* __restrict__ A, int lda,
                                       const double* __restrict__ x, double* __restrict__ part) {
      const int i = blockIdx.x * GV_ROWS + threadIdx.x;
      const int c0 = blockIdx.y * GV_COLS, c1 = min(n, c0 + GV_COLS);
      __shared__ double xs[GV_COLS];
      for (int c = c0 + threadIdx.x; c < c1; c += blockDim.x) xs[c - c0] = x[c];
      __syncthreads();
      if (i >= m) return;
      const double* Ar = A + i + (size_t)c0 * lda;
      double s0 = 0.0, s1 = 0.0;
      int c = 0;
      for (; c + 1 < c1 - c0; c += 2) {
        s0 += Ar[(size_t)c * lda] * xs[c];
        s1 += Ar[(size_t)(c + 1) * lda] * xs[c + 1];
      }
      if (c < c1 - c0) s0 += Ar[(size_t)c * lda] * xs[c];
      part[(size_t)blockIdx.y * m + i] = s0 + s1;
    }
    __global__ void gemv_n_reduce_kernel(int m, int nchunk, double alpha,
                                         const double* __restrict__ part, double beta,
                                         double* __restrict__ y) {
      const int i = blockIdx.x * blockDim.x + threadIdx.x;
      if (i >= m) return;
      double s = 0.0;
      for (int q = 0; q < nchunk; q++) s += part[(size_t)q * m + i];
      y[i] = (beta == 0.0 ? 0.0 : beta * y[i]) + alpha * s;
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
      static std::atomic<unsigned long long> done{0};
      once_per_device(done, [] {
      HSSMF_CUDA(cudaFuncSetAttribute(ulv_fwd_lsolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      HSSMF_CUDA(cudaFuncSetAttribute(ulv_bwd_usolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      HSSMF_CUDA(cudaFuncSetAttribute(lu_solve_vec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      });
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

  void diag_gather_run(const double* L, int n, const int* perm, int k, double* out, cudaStream_t s) {
    if (k <= 0) return;
    diag_gather_kernel<<<ceil_div(k, 256), 256, 0, s>>>(L, n, perm, k, out);
    HSSMF_LAUNCH_CHECK();
  }

  void maxabs_run(const double* a, long long lda, int m, int n, double* out, cudaStream_t s) {
    if (m <= 0 || n <= 0) return;
    const long long tot = (long long)m * n;
    const int blocks = (int)std::min<long long>((tot + 255) / 256, 148 * 8);
    maxabs_kernel<<<blocks, 256, 0, s>>>(a, lda, m, n, (unsigned long long*)out);
    HSSMF_LAUNCH_CHECK();
  }

  // ULV solve sweeps, one tree level per call, batched over the level's
  // nodes in three phases each so that the matrix-vector parts of a node
  // spread over many CTAs (fwd, hss_ulv.hpp:226-248):
  //   omega: o = [y_rest - Eu y_skel; y_skel]          (rows over CTAs)
  //   z = L11^-1 P o[0:k] -> ws  (one CTA per node; chained blocked solve over
  //                               many CTAs when k > kUlvChainK)
  //   fout = o[k:m] - L21 z                              (rows over CTAs)
  // and (bwd, hss_ulv.hpp:250-276):
  //   rhs = ws - U12 xkeep; sol = U11^-1 rhs; x(vperm) = psi(sol, xkeep)
  constexpr int kUlvChainK = 1024;

  void ulv_fwd_level(const std::vector<UlvSolveNode>& all, int, cudaStream_t s) {
    if (all.empty()) return;
    set_attr();
    std::vector<UlvSolveNode> nodes(all);
    size_t tot = 0;
    int mmax = 0, rmax = 0, ksm = 0;
    for (auto& n : nodes) {
      tot += (size_t)n.m + 1;
      mmax = std::max(mmax, n.m);
      rmax = std::max(rmax, n.r);
      if (n.k <= kUlvChainK) ksm = std::max(ksm, n.k);
    }
    double* scr = nullptr;
    HSSMF_CUDA(cudaMallocAsync((void**)&scr, tot * sizeof(double) + 64 * nodes.size(), s));
    int* sync = reinterpret_cast<int*>(scr + tot);
    HSSMF_CUDA(cudaMemsetAsync(sync, 0, 16 * nodes.size(), s));
    size_t off = 0;
    for (auto& n : nodes) {
      n.scr = scr + off;
      off += (size_t)n.m + 1;
    }
    auto d = upload_async(nodes, s);
    const int nn = (int)nodes.size();
    if (mmax > 0) {
      ulv_fwd_omega_kernel<<<dim3(ceil_div(mmax, 256), nn), 256, 0, s>>>(d.p);
      HSSMF_LAUNCH_CHECK();
    }
    if (ksm > 0) {
      ulv_fwd_lsolve_kernel<<<nn, UT, (size_t)ksm * 8, s>>>(d.p, kUlvChainK);
      HSSMF_LAUNCH_CHECK();
    }
    for (int q = 0; q < nn; q++) {
      const auto& n = nodes[q];
      if (n.k <= kUlvChainK) continue;
      trsv_chain_kernel<true><<<ceil_div(n.k, TB), 256, 0, s>>>(n.G, n.m, n.k, n.scr, n.lperm,
                                                               n.ws, sync + 4 * q);
      HSSMF_LAUNCH_CHECK();
    }
    if (rmax > 0) {
      ulv_fwd_l21_kernel<<<dim3(ceil_div(rmax, 256), nn), 256, 0, s>>>(d.p);
      HSSMF_LAUNCH_CHECK();
    }
    release_async(d, s);
    HSSMF_CUDA(cudaFreeAsync(scr, s));
  }

  void ulv_bwd_level(const std::vector<UlvSolveNode>& all, cudaStream_t s) {
    if (all.empty()) return;
    set_attr();
    std::vector<UlvSolveNode> nodes(all);
    size_t tot = 0;
    int mmax = 0, kmax = 0, ksm = 0;
    for (auto& n : nodes) {
      tot += 2 * (size_t)n.k + 1;
      mmax = std::max(mmax, n.m);
      kmax = std::max(kmax, n.k);
      if (n.k <= kUlvChainK) ksm = std::max(ksm, n.k);
    }
    double* scr = nullptr;
    HSSMF_CUDA(cudaMallocAsync((void**)&scr, tot * sizeof(double) + 64 * nodes.size(), s));
    int* sync = reinterpret_cast<int*>(scr + tot);
    HSSMF_CUDA(cudaMemsetAsync(sync, 0, 16 * nodes.size(), s));
    size_t off = 0;
    for (auto& n : nodes) {
      n.scr = scr + off;
      off += 2 * (size_t)n.k + 1;
    }
    auto d = upload_async(nodes, s);
    const int nn = (int)nodes.size();
    if (kmax > 0) {
      ulv_bwd_u12_kernel<<<dim3(ceil_div(kmax, 256), nn), 256, 0, s>>>(d.p);
      HSSMF_LAUNCH_CHECK();
    }
    if (ksm > 0) {
      ulv_bwd_usolve_kernel<<<nn, UT, (size_t)ksm * 8, s>>>(d.p, kUlvChainK);
      HSSMF_LAUNCH_CHECK();
    }
    for (int q = 0; q < nn; q++) {
      const auto& n = nodes[q];
      if (n.k <= kUlvChainK) continue;
      trsv_chain_kernel<false><<<ceil_div(n.k, TB), 256, 0, s>>>(n.G, n.m, n.k, n.scr, nullptr,
                                                                n.scr + n.k, sync + 4 * q);
      HSSMF_LAUNCH_CHECK();
    }
    if (mmax > 0) {
      ulv_bwd_psi_kernel<<<dim3(ceil_div((long long)mmax * 32, 256), nn), 256, 0, s>>>(d.p);
      HSSMF_LAUNCH_CHECK();
    }
    release_async(d, s);
    HSSMF_CUDA(cudaFreeAsync(scr, s));
  }

  void asymmetry_async(const double* a, long long lda, int m, double* dout, cudaStream_t s) {
    HSSMF_CUDA(cudaMemsetAsync(dout, 0, 2 * sizeof(double), s));
    if (m > 0) {
      asymmetry_kernel<<<std::min(ceil_div((long long)m * m, 256), 148 * 8), 256, 0, s>>>(
          a, lda, m, reinterpret_cast<unsigned long long*>(dout));
      HSSMF_LAUNCH_CHECK();
    }
  }

  void mirror_lower_run(double* a, long long ld, int n, cudaStream_t s) {
    if (n <= 1) return;
    const int nb = ceil_div(n, 32);
    mirror_lower_kernel<<<dim3(nb, nb), dim3(32, 8), 0, s>>>(a, ld, n);
    HSSMF_LAUNCH_CHECK();
  }

  void lu_solve_vec(const double* lu, int ld, const int* perm, int n, double* x, cudaStream_t s) {
    if (n <= 0) return;
    set_attr();
    if (n > 256) {
      // large factors: chained blocked L and U solves over many SMs
      double* y = nullptr;
      int* sync = nullptr;
      HSSMF_CUDA(cudaMallocAsync((void**)&y, (size_t)n * sizeof(double) + 64, s));
      sync = reinterpret_cast<int*>(y + n);
      HSSMF_CUDA(cudaMemsetAsync(sync, 0, 4 * sizeof(int), s));
      const int nb = ceil_div(n, TB);
      trsv_chain_kernel<true><<<nb, 256, 0, s>>>(lu, ld, n, x, perm, y, sync);
      HSSMF_LAUNCH_CHECK();
      trsv_chain_kernel<false><<<nb, 256, 0, s>>>(lu, ld, n, y, nullptr, x, sync + 2);
      HSSMF_LAUNCH_CHECK();
      HSSMF_CUDA(cudaFreeAsync(y, s));
      return;
    }
    if ((size_t)n * 8 > 200 * 1024) throw CudaError("lu solve: block too large for smem");
    lu_solve_vec_kernel<<<1, UT, (size_t)n * 8, s>>>(lu, ld, perm, n, x);
    HSSMF_LAUNCH_CHECK();
  }

  void gemv_run(char ta, int m, int n, double alpha, const double* A, int lda, const double* x,
                double beta, double* y, cudaStream_t s) {
    if (ta == 'N' && m > 0 && n > 2 * GV_COLS) {
      // long rows: column chunks over a second grid dimension
      const int nch = ceil_div(n, GV_COLS);
      double* part = nullptr;
      HSSMF_CUDA(cudaMallocAsync((void**)&part, (size_t)nch * m * sizeof(double), s));
      gemv_n_part_kernel<<<dim3(ceil_div(m, GV_ROWS), nch), GV_ROWS, 0, s>>>(m, n, A, lda, x, part);
      HSSMF_LAUNCH_CHECK();
      gemv_n_reduce_kernel<<<ceil_div(m, 256), 256, 0, s>>>(m, nch, alpha, part, beta, y);
      HSSMF_LAUNCH_CHECK();
      HSSMF_CUDA(cudaFreeAsync(part, s));
      return;
    }
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
