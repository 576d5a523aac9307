#include "cpqr.cuh"
#include "staging.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "gemm.cuh"

namespace hssmf_b200 {

  namespace {
    constexpr int CT = 256, NW = CT / 32;

    __device__ __forceinline__ double warp_sum(double v) {
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      return v;
    }

    // dynamic smem: nrm2[n], last[n] (double), v[m] (double), perm[n] (int)
    __global__ void __launch_bounds__(CT)
    cpqr_kernel(const CpqrTask* __restrict__ tasks, double eps, double abs_tol) {
      extern __shared__ double sm[];
      const CpqrTask T = tasks[blockIdx.x];
      const int m = T.m, n = T.n, ld = T.ldy;
      double* Y = T.Y;
      double* nrm2 = sm;
      double* last = nrm2 + n;
      double* v = last + n;
      int* perm = reinterpret_cast<int*>(v + m);
      __shared__ double rv[NW];
      __shared__ int ri[NW];
      __shared__ int s_p, s_stop, s_cert;
      __shared__ double s_tk, s_r11;
      const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
      const int kmax_dim = min(m, n);
      const int kmax = T.max_rank < 0 ? kmax_dim : min(kmax_dim, T.max_rank);

      if (m == 0 || n == 0) {
        for (int j = tid; j < n; j += CT) T.perm[j] = j;
        if (tid == 0) { T.out[0] = 0; T.out[1] = 1; }
        return;
      }
      // exact squared column norms (rrqr.hpp:49-53)
      for (int j = warp; j < n; j += NW) {
        const double* c = Y + (size_t)j * ld;
        double s = 0;
        for (int i = lane; i < m; i += 32) s += c[i] * c[i];
        s = warp_sum(s);
        if (lane == 0) { nrm2[j] = s; last[j] = s; }
      }
      for (int j = tid; j < n; j += CT) perm[j] = j;
      if (tid == 0) { s_r11 = 0; s_cert = 0; }
      __syncthreads();
      int k = 0;
      while (true) {
        // pivot: largest downdated norm, lowest index on ties
        double bv = -1.0;
        int bi = 0x7fffffff;
        for (int j = k + tid; j < n; j += CT)
          if (nrm2[j] > bv) { bv = nrm2[j]; bi = j; }
        warp_argmax(bv, bi);
        if (lane == 0) { rv[warp] = bv; ri[warp] = bi; }
        __syncthreads();
        if (tid == 0) {
          double b = rv[0];
          int p = ri[0];
          for (int w = 1; w < NW; w++)
            if (rv[w] > b || (rv[w] == b && ri[w] < p)) { b = rv[w]; p = ri[w]; }
          const double pv = nrm2[p] > 0.0 ? sqrt(nrm2[p]) : 0.0;
          int stop = 0;
          if (k == 0) {
            s_r11 = pv;
            if (pv == 0.0 || pv <= abs_tol) { stop = 1; s_cert = 1; }
          } else if (pv <= eps * s_r11 || pv <= abs_tol) {
            stop = 1;
            s_cert = 1;
          }
          if (!stop && k == kmax) {
            stop = 1;
            s_cert = (k == kmax_dim);
          }
          if (!stop && p != k) {
            double t = nrm2[k]; nrm2[k] = nrm2[p]; nrm2[p] = t;
            t = last[k]; last[k] = last[p]; last[p] = t;
            const int q = perm[k]; perm[k] = perm[p]; perm[p] = q;
          }
          s_p = p;
          s_stop = stop;
        }
        __syncthreads();
        if (s_stop) break;
        const int p = s_p;
        double* ck = Y + (size_t)k * ld;
        if (p != k) {
          double* cp = Y + (size_t)p * ld;
          for (int i = tid; i < m; i += CT) {
            const double t = ck[i];
            ck[i] = cp[i];
            cp[i] = t;
          }
          __syncthreads();
        }
        // Householder reflector (rrqr.hpp:85-103)
        double s = 0;
        for (int i = k + 1 + tid; i < m; i += CT) s += ck[i] * ck[i];
        s = warp_sum(s);
        if (lane == 0) rv[warp] = s;
        __syncthreads();
        if (tid == 0) {
          double xs = 0;
          for (int w = 0; w < NW; w++) xs += rv[w];
          const double xn = sqrt(xs);
          const double alpha = ck[k];
          double tk = 0, sc = 0;
          if (xn != 0.0 || fabs(alpha) != 0.0) {
            double beta = hypot(fabs(alpha), xn);
            if (alpha > 0.0) beta = -beta;
            if (beta != 0.0) {
              tk = (beta - alpha) / beta;
              sc = 1.0 / (alpha - beta);
              ck[k] = beta;
            }
          }
          s_tk = tk;
          rv[0] = sc;
        }
        __syncthreads();
        const double tk = s_tk, sc = rv[0];
        for (int i = k + 1 + tid; i < m; i += CT) {
          const double x = tk != 0.0 ? ck[i] * sc : ck[i];
          if (tk != 0.0) ck[i] = x;
          v[i] = x;
        }
        __syncthreads();
        // apply the reflector to the trailing columns and downdate norms
        for (int j = k + 1 + warp; j < n; j += NW) {
          double* cj = Y + (size_t)j * ld;
          if (tk != 0.0) {
            double w = 0;
            for (int i = k + 1 + lane; i < m; i += 32) w += v[i] * cj[i];
            w = warp_sum(w) + cj[k];
            w *= tk;
            if (lane == 0) cj[k] -= w;
            for (int i = k + 1 + lane; i < m; i += 32) cj[i] -= w * v[i];
          }
          __syncwarp();
          const double rk = cj[k];
          double nj = nrm2[j] - rk * rk;
          if (nj < 0.0) nj = 0.0;
          if (nj < 0.1 * last[j]) {
            double q = 0;
            for (int i = k + 1 + lane; i < m; i += 32) q += cj[i] * cj[i];
            q = warp_sum(q);
            if (lane == 0) { nrm2[j] = q; last[j] = q; }
          } else if (lane == 0) {
            nrm2[j] = nj;
          }
        }
        __syncthreads();
        k++;
        if (k == kmax_dim) {
          if (tid == 0) s_cert = 1;
          break;
        }
      }
      __syncthreads();
      for (int j = tid; j < n; j += CT) T.perm[j] = perm[j];
      if (tid == 0) { T.out[0] = k; T.out[1] = s_cert; }
    }

    // X = R1^-1 R2 (upper TRSM, rrqr.hpp:187-192), CPC columns per CTA held in
    // smem, backward column sweep over R1
    __global__ void id_solve_kernel(const CpqrTask* __restrict__ tasks, int cpc) {
      extern __shared__ double xs[];
      const CpqrTask T = tasks[blockIdx.y];
      const int k = T.out[0], n = T.n, ld = T.ldy;
      const int c0 = blockIdx.x * cpc;
      if (k == 0 || c0 >= n - k) return;
      const int nc = min(cpc, n - k - c0);
      const double* R = T.Y;
      for (int e = threadIdx.x; e < k * nc; e += blockDim.x) {
        const int i = e % k, c = e / k;
        xs[i + c * k] = R[i + (size_t)(k + c0 + c) * ld];
      }
      __syncthreads();
      for (int i = k - 1; i >= 0; i--) {
        const double d = R[i + (size_t)i * ld];
        if (threadIdx.x < nc) xs[i + threadIdx.x * k] /= d;
        __syncthreads();
        for (int e = threadIdx.x; e < i * nc; e += blockDim.x) {
          const int l = e % i, c = e / i;
          xs[l + c * k] -= R[l + (size_t)i * ld] * xs[i + c * k];
        }
        __syncthreads();
      }
      for (int e = threadIdx.x; e < k * nc; e += blockDim.x) {
        const int i = e % k, c = e / k;
        T.X[i + (size_t)(c0 + c) * k] = xs[i + c * k];
      }
    }

    // ---- cluster CPQR: one thread-block cluster (CL CTAs) per task --------
    // Columns are dealt cyclically to the CTAs of the cluster (column j lives
    // in CTA j % CL, its norms in that CTA's shared memory). Per elimination
    // step: local pivot candidates -> cluster barrier -> every CTA reduces
    // the CL candidates over DSMEM (identical decision everywhere) -> the
    // owner of column k swaps, builds the reflector -> cluster barrier ->
    // every CTA applies it to its own trailing columns and downdates norms.
    // The matrix stays in global memory and is only accessed with L2-coherent
    // (.cg) loads, since columns migrate between CTAs on pivot swaps.
    struct ClPub {
      double bv;
      int bi;
      int pad;
      double tau;
    };

    __global__ void __launch_bounds__(CT)
    cpqr_cluster_kernel(const CpqrTask* __restrict__ tasks, double eps, double abs_tol,
                        int CL) {
      namespace cg = cooperative_groups;
      cg::cluster_group cl = cg::this_cluster();
      const int rank = (int)cl.block_rank();
      extern __shared__ double sm[];
      const CpqrTask T = tasks[blockIdx.x / CL];
      const int m = T.m, n = T.n, ld = T.ldy;
      double* Y = T.Y;
      const int nloc = (n + CL - 1) / CL;
      double* nrm2 = sm;
      double* last = nrm2 + nloc;
      double* v = last + nloc;
      __shared__ ClPub pub;
      __shared__ double rv[NW];
      __shared__ int ri[NW];
      __shared__ int s_p, s_stop, s_cert;
      __shared__ double s_r11, s_tau;
      const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
      const int kmax_dim = min(m, n);
      const int kmax = T.max_rank < 0 ? kmax_dim : min(kmax_dim, T.max_rank);
      if (m == 0 || n == 0) {
        if (rank == 0) {
          for (int j = tid; j < n; j += CT) T.perm[j] = j;
          if (tid == 0) { T.out[0] = 0; T.out[1] = 1; }
        }
        return;
      }
      // own columns: j = rank + CL * jl
      for (int jl = warp; jl < nloc; jl += NW) {
        const int j = rank + CL * jl;
        if (j >= n) break;
        const double* c = Y + (size_t)j * ld;
        double s = 0;
        for (int i = lane; i < m; i += 32) {
          const double x = __ldcg(c + i);
          s += x * x;
        }
        s = warp_sum(s);
        if (lane == 0) { nrm2[jl] = s; last[jl] = s; }
      }
      if (rank == 0)
        for (int j = tid; j < n; j += CT) T.perm[j] = j;
      if (tid == 0) { s_r11 = 0; s_cert = 0; }
      __syncthreads();
      int k = 0;
      while (true) {
        // 1. local pivot candidate among own columns j >= k
        double bv = -1.0;
        int bi = 0x7fffffff;
        for (int jl = tid; jl < nloc; jl += CT) {
          const int j = rank + CL * jl;
          if (j >= k && j < n && nrm2[jl] > bv) { bv = nrm2[jl]; bi = j; }
        }
        warp_argmax(bv, bi);
        if (lane == 0) { rv[warp] = bv; ri[warp] = bi; }
        __syncthreads();
        if (tid == 0) {
          double b = rv[0];
          int p = ri[0];
          for (int w = 1; w < NW; w++)
            if (rv[w] > b || (rv[w] == b && ri[w] < p)) { b = rv[w]; p = ri[w]; }
          pub.bv = b;
          pub.bi = p;
        }
        cl.sync();
        // 2. global decision (identical in every CTA); one lane per peer CTA
        double gb = -1.0;
        int gp = 0x7fffffff;
        if (tid < 32) {
          if (tid < CL) {
            const ClPub* q = cl.map_shared_rank(&pub, tid);
            gb = q->bv;
            gp = q->bi;
          }
          warp_argmax(gb, gp);
        }
        if (tid == 0) {
          const double b = gb;
          const int p = gp;
          const double pv = b > 0.0 ? sqrt(b) : 0.0;
          int stop = 0;
          if (k == 0) {
            s_r11 = pv;
            if (pv == 0.0 || pv <= abs_tol) { stop = 1; s_cert = 1; }
          } else if (pv <= eps * s_r11 || pv <= abs_tol) {
            stop = 1;
            s_cert = 1;
          }
          if (!stop && k == kmax) {
            stop = 1;
            s_cert = (k == kmax_dim);
          }
          s_p = p;
          s_stop = stop;
        }
        __syncthreads();
        if (s_stop) break;
        const int p = s_p;
        const int ok = k % CL;
        double* ck = Y + (size_t)k * ld;
        if (rank == ok) {
          if (p != k) {
            double* cp = Y + (size_t)p * ld;
            for (int i = tid; i < m; i += CT) {
              const double t = __ldcg(ck + i);
              __stcg(ck + i, __ldcg(cp + i));
              __stcg(cp + i, t);
            }
            if (tid == 0) {
              double* nk = cl.map_shared_rank(nrm2, ok) + k / CL;
              double* np = cl.map_shared_rank(nrm2, p % CL) + p / CL;
              double* lk = cl.map_shared_rank(last, ok) + k / CL;
              double* lp = cl.map_shared_rank(last, p % CL) + p / CL;
              double t = *nk; *nk = *np; *np = t;
              t = *lk; *lk = *lp; *lp = t;
              const int q = T.perm[k]; T.perm[k] = T.perm[p]; T.perm[p] = q;
            }
            __syncthreads();
          }
          // 3. Householder reflector of column k (rrqr.hpp:85-103)
          double s = 0;
          for (int i = k + 1 + tid; i < m; i += CT) {
            const double x = __ldcg(ck + i);
            s += x * x;
          }
          s = warp_sum(s);
          if (lane == 0) rv[warp] = s;
          __syncthreads();
          if (tid == 0) {
            double xs = 0;
            for (int w = 0; w < NW; w++) xs += rv[w];
            const double xn = sqrt(xs);
            const double alpha = __ldcg(ck + k);
            double tk = 0, sc = 0;
            if (xn != 0.0 || fabs(alpha) != 0.0) {
              double beta = hypot(fabs(alpha), xn);
              if (alpha > 0.0) beta = -beta;
              if (beta != 0.0) {
                tk = (beta - alpha) / beta;
                sc = 1.0 / (alpha - beta);
                __stcg(ck + k, beta);
              }
            }
            pub.tau = tk;
            rv[0] = sc;
          }
          __syncthreads();
          const double sc = rv[0];
          if (pub.tau != 0.0)
            for (int i = k + 1 + tid; i < m; i += CT) __stcg(ck + i, __ldcg(ck + i) * sc);
        }
        cl.sync();
        // 4. apply the reflector to own trailing columns, downdate norms
        if (tid == 0) s_tau = cl.map_shared_rank(&pub, ok)->tau;
        for (int i = k + 1 + tid; i < m; i += CT) v[i] = __ldcg(ck + i);
        __syncthreads();
        const double tk = s_tau;
        int jl0 = (k + 1 - rank + CL - 1) / CL;
        if (jl0 < 0) jl0 = 0;
        for (int jl = jl0 + warp; jl < nloc; jl += NW) {
          const int j = rank + CL * jl;
          if (j >= n) break;
          double* cj = Y + (size_t)j * ld;
          if (tk != 0.0) {
            double w = 0;
            for (int i = k + 1 + lane; i < m; i += 32) w += v[i] * __ldcg(cj + i);
            w = warp_sum(w) + __ldcg(cj + k);
            w *= tk;
            if (lane == 0) __stcg(cj + k, __ldcg(cj + k) - w);
            for (int i = k + 1 + lane; i < m; i += 32) __stcg(cj + i, __ldcg(cj + i) - w * v[i]);
          }
          __syncwarp();
          const double rk = __ldcg(cj + k);
          double nj = nrm2[jl] - rk * rk;
          if (nj < 0.0) nj = 0.0;
          if (nj < 0.1 * last[jl]) {
            double q = 0;
            for (int i = k + 1 + lane; i < m; i += 32) {
              const double x = __ldcg(cj + i);
              q += x * x;
            }
            q = warp_sum(q);
            if (lane == 0) { nrm2[jl] = q; last[jl] = q; }
          } else if (lane == 0) {
            nrm2[jl] = nj;
          }
        }
        __syncthreads();
        k++;
        if (k == kmax_dim) {
          if (tid == 0) s_cert = 1;
          break;
        }
      }
      cl.sync();  // keep peers' shared memory alive until every CTA is done
      if (rank == 0 && tid == 0) { T.out[0] = k; T.out[1] = s_cert; }
    }

    void set_attr() {
      static std::atomic<unsigned long long> done{0};
      once_per_device(done, [] {
      HSSMF_CUDA(cudaFuncSetAttribute(cpqr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      220 * 1024));
      HSSMF_CUDA(cudaFuncSetAttribute(cpqr_cluster_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      HSSMF_CUDA(cudaFuncSetAttribute(cpqr_cluster_kernel,
                                      cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      HSSMF_CUDA(cudaFuncSetAttribute(id_solve_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      });
    }
  }  // namespace

  void cpqr_run(const CpqrTask* tasks, int ntask, int max_m, int max_n, double eps,
                double abs_tol, cudaStream_t s) {
    if (!ntask) return;
    set_attr();
    // cluster width: enough CTAs that each owns ~32 columns, at most 16
    int CL = 1;
    while (CL < 16 && (long long)max_n * max_m > (long long)CL * 32 * 512) CL *= 2;
    const char* env = getenv("HSSMF_CPQR_CLUSTER");
    if (env) CL = std::max(1, std::min(16, atoi(env)));
    if (CL == 1) {
      const size_t smem = (size_t)max_n * 20 + (size_t)max_m * 8 + 64;
      if (smem > 220 * 1024) throw CudaError("cpqr: task too large for shared memory");
      cpqr_kernel<<<ntask, CT, smem, s>>>(tasks, eps, abs_tol);
      HSSMF_LAUNCH_CHECK();
      return;
    }
    const int nloc = (max_n + CL - 1) / CL;
    const size_t smem = (size_t)nloc * 16 + (size_t)max_m * 8 + 64;
    if (smem > 200 * 1024) throw CudaError("cpqr: task too large for shared memory");
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ntask * CL);
    cfg.blockDim = dim3(CT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    HSSMF_CUDA(cudaLaunchKernelEx(&cfg, cpqr_cluster_kernel, tasks, eps, abs_tol, CL));
    HSSMF_LAUNCH_CHECK();
  }

  void id_solve_run(const CpqrTask* tasks, int ntask, int max_rank, int max_cols,
                    cudaStream_t s) {
    if (!ntask || max_rank <= 0 || max_cols <= 0) return;
    set_attr();
    int cpc = (int)std::min<long long>(8, (200LL * 1024) / (8LL * max_rank));
    if (cpc < 1) throw CudaError("id solve: rank too large");
    dim3 grid(ceil_div(max_cols, cpc), ntask);
    id_solve_kernel<<<grid, 256, (size_t)cpc * max_rank * 8, s>>>(tasks, cpc);
    HSSMF_LAUNCH_CHECK();
  }

  namespace {
    constexpr int TB = 64, TC = 128;

    struct TriStep {
      const double* R;   // R1 block origin: R + i0 + i0*ldr
      int ldr;
      double* X;         // X rows [i0, i0+bs), ld ldx
      int ldx, bs, ncols;
    };

    constexpr int kParamSteps = 128;
    struct TriParam {
      TriStep st[kParamSteps];
    };

    // X[i0:i0+bs, :] <- R1[i0:i0+bs, i0:i0+bs]^-1 X[i0:i0+bs, :] (upper, non-unit)
    __global__ void __launch_bounds__(TC) tri_block_kernel(const __grid_constant__ TriParam P) {
      const TriStep S = P.st[blockIdx.y];
      __shared__ double Rb[TB][TB + 1];
      for (int e = threadIdx.x; e < S.bs * S.bs; e += TC) {
        const int r = e % S.bs, c = e / S.bs;
        Rb[r][c] = S.R[r + (size_t)c * S.ldr];
      }
      __syncthreads();
      const int c = blockIdx.x * TC + threadIdx.x;
      if (c >= S.ncols) return;
      double* col = S.X + (size_t)c * S.ldx;
      double x[TB];
#pragma unroll
      for (int r = 0; r < TB; r++) x[r] = r < S.bs ? col[r] : 0.0;
#pragma unroll
      for (int i = TB - 1; i >= 0; i--) {
        if (i < S.bs) {
          double s = x[i];
#pragma unroll
          for (int l = i + 1; l < TB; l++)
            if (l < S.bs) s -= Rb[i][l] * x[l];
          x[i] = s / Rb[i][i];
        }
      }
#pragma unroll
      for (int r = 0; r < TB; r++)
        if (r < S.bs) col[r] = x[r];
    }

    // inverse of an upper-triangular diagonal block (bs <= 64): thread j solves
    // R x = e_j by back substitution from the shared copy of the block;
    // out is 64 x 64 (ld 64), zero below the diagonal and beyond bs
    struct InvStep {
      const double* R;
      int ldr, bs;
      double* out;
    };
    __global__ void __launch_bounds__(TB) tri_inv_kernel(const InvStep* __restrict__ st) {
      const InvStep S = st[blockIdx.x];
      __shared__ double Rb[TB][TB + 1];
      for (int e = threadIdx.x; e < S.bs * S.bs; e += TB) {
        const int r = e % S.bs, c = e / S.bs;
        Rb[r][c] = S.R[r + (size_t)c * S.ldr];
      }
      __syncthreads();
      const int j = threadIdx.x;
      double* o = S.out + (size_t)j * TB;
      if (j >= S.bs) {
        for (int i = 0; i < TB; i++) o[i] = 0.0;
        return;
      }
      double x[TB];
#pragma unroll
      for (int i = 0; i < TB; i++) x[i] = 0.0;
#pragma unroll
      for (int i = TB - 1; i >= 0; i--) {
        if (i <= j) {
          double sacc = (i == j) ? 1.0 : 0.0;
#pragma unroll
          for (int l = i + 1; l < TB; l++)
            if (l <= j) sacc -= Rb[i][l] * x[l];
          x[i] = sacc / Rb[i][i];
        }
      }
#pragma unroll
      for (int i = 0; i < TB; i++) o[i] = x[i];
    }
  }  // namespace

  void id_solve_blocked(const std::vector<CpqrTask>& tasks, const std::vector<int>& ranks,
                        cudaStream_t s, double* flops, bool inv_blocks) {
    if (inv_blocks) {
      // X = R2; all diagonal blocks inverted in one launch; per block from the
      // bottom: W = inv(R_bb) X_b (GEMM), X[0:i0] -= R[0:i0, b] W (GEMM), X_b = W
      std::vector<InvStep> inv;
      std::vector<size_t> first(tasks.size(), 0);
      int maxb = 0;
      size_t wtot = 0;
      std::vector<size_t> woff(tasks.size(), 0);
      for (size_t t = 0; t < tasks.size(); t++) {
        const int k = ranks[t], nc = tasks[t].n - k;
        if (k <= 0 || nc <= 0) continue;
        HSSMF_CUDA(cudaMemcpy2DAsync(tasks[t].X, (size_t)k * sizeof(double),
                                     tasks[t].Y + (size_t)k * tasks[t].ldy,
                                     (size_t)tasks[t].ldy * sizeof(double), (size_t)k * sizeof(double),
                                     nc, cudaMemcpyDeviceToDevice, s));
        const int nb = (k + TB - 1) / TB;
        maxb = std::max(maxb, nb);
        first[t] = inv.size();
        for (int j = 0; j < nb; j++) {
          const int i1 = k - j * TB, i0 = std::max(0, i1 - TB);
          inv.push_back({tasks[t].Y + i0 + (size_t)i0 * tasks[t].ldy, tasks[t].ldy, i1 - i0, nullptr});
        }
        woff[t] = wtot;
        wtot += (size_t)TB * nc;
      }
      if (inv.empty()) return;
      char* buf = nullptr;
      const size_t inv_bytes = inv.size() * (size_t)TB * TB * sizeof(double);
      const size_t st_bytes = inv.size() * sizeof(InvStep);
      HSSMF_CUDA(cudaMallocAsync((void**)&buf, inv_bytes + wtot * sizeof(double) + st_bytes, s));
      double* invs = reinterpret_cast<double*>(buf);
      double* W = invs + inv.size() * (size_t)TB * TB;
      InvStep* dst = reinterpret_cast<InvStep*>(buf + inv_bytes + wtot * sizeof(double));
      for (size_t q = 0; q < inv.size(); q++) inv[q].out = invs + q * (size_t)TB * TB;
      h2d(dst, inv.data(), st_bytes, s);  // (copied out of the vector before returning)
      tri_inv_kernel<<<(unsigned)inv.size(), TB, 0, s>>>(dst);
      HSSMF_LAUNCH_CHECK();
      for (int j = 0; j < maxb; j++) {
        std::vector<GemmProblem> solve, up;
        struct Back { double* x; int ldx, bs, nc; const double* w; };
        std::vector<Back> back;
        for (size_t t = 0; t < tasks.size(); t++) {
          const auto& T = tasks[t];
          const int k = ranks[t], nc = T.n - k;
          if (k <= 0 || nc <= 0) continue;
          const int i1 = k - j * TB;
          if (i1 <= 0) continue;
          const int i0 = std::max(0, i1 - TB), bs = i1 - i0;
          double* Wt = W + woff[t];
          solve.push_back({inv[first[t] + j].out, T.X + i0, Wt, bs, nc, bs, TB, k, TB});
          if (i0 > 0) {
            up.push_back({T.Y + (size_t)i0 * T.ldy, Wt, T.X, i0, nc, bs, T.ldy, TB, k});
            if (flops) *flops += 2.0 * i0 * nc * bs;
          }
          back.push_back({T.X + i0, k, bs, nc, Wt});
          if (flops) *flops += (double)bs * bs * nc;
        }
        gemm_run_host(solve, 'N', 'N', 1.0, 0.0, s);
        gemm_run_host(up, 'N', 'N', -1.0, 1.0, s);
        for (const auto& b : back)
          HSSMF_CUDA(cudaMemcpy2DAsync(b.x, (size_t)b.ldx * sizeof(double), b.w, (size_t)TB * sizeof(double),
                                       (size_t)b.bs * sizeof(double), b.nc, cudaMemcpyDeviceToDevice, s));
      }
      HSSMF_CUDA(cudaFreeAsync(buf, s));
      return;
    }
    // X = R2 (copies), then blocks from the bottom
    int maxb = 0;
    for (size_t t = 0; t < tasks.size(); t++) {
      const int k = ranks[t], nc = tasks[t].n - k;
      if (k <= 0 || nc <= 0) continue;
      HSSMF_CUDA(cudaMemcpy2DAsync(tasks[t].X, (size_t)k * sizeof(double),
                                   tasks[t].Y + (size_t)k * tasks[t].ldy,
                                   (size_t)tasks[t].ldy * sizeof(double), (size_t)k * sizeof(double),
                                   nc, cudaMemcpyDeviceToDevice, s));
      maxb = std::max(maxb, (k + TB - 1) / TB);
    }
    for (int j = 0; j < maxb; j++) {
      std::vector<TriStep> steps;
      std::vector<GemmProblem> up;
      int maxc = 0;
      for (size_t t = 0; t < tasks.size(); t++) {
        const auto& T = tasks[t];
        const int k = ranks[t], nc = T.n - k;
        if (k <= 0 || nc <= 0) continue;
        const int i1 = k - j * TB;
        if (i1 <= 0) continue;
        const int i0 = std::max(0, i1 - TB), bs = i1 - i0;
        steps.push_back({T.Y + i0 + (size_t)i0 * T.ldy, T.ldy, T.X + i0, k, bs, nc});
        maxc = std::max(maxc, nc);
        if (i0 > 0) {  // X[0:i0, :] -= R1[0:i0, i0:i1] X[i0:i1, :]
          up.push_back({T.Y + (size_t)i0 * T.ldy, T.X + i0, T.X, i0, nc, bs, T.ldy, k, k});
          if (flops) *flops += 2.0 * i0 * nc * bs;
        }
        if (flops) *flops += (double)bs * bs * nc;
      }
      for (size_t b0 = 0; b0 < steps.size(); b0 += kParamSteps) {
        TriParam P;
        const int nb = (int)std::min<size_t>(kParamSteps, steps.size() - b0);
        for (int q = 0; q < nb; q++) P.st[q] = steps[b0 + q];
        tri_block_kernel<<<dim3(ceil_div(maxc, TC), (unsigned)nb), TC, 0, s>>>(P);
        HSSMF_LAUNCH_CHECK();
      }
      gemm_run_host(up, 'N', 'N', -1.0, 1.0, s);
    }
  }

  void cpqr_id_run(const CpqrTask* tasks, int ntask, int max_m, int max_n, double eps,
                   double abs_tol, cudaStream_t s) {
    cpqr_run(tasks, ntask, max_m, max_n, eps, abs_tol, s);
    std::vector<CpqrTask> h(ntask);
    HSSMF_CUDA(cudaMemcpyAsync(h.data(), tasks, ntask * sizeof(CpqrTask), cudaMemcpyDeviceToHost, s));
    HSSMF_CUDA(cudaStreamSynchronize(s));
    int max_rank = 0, max_cols = 0;
    for (auto& t : h) {
      int o[2];
      HSSMF_CUDA(cudaMemcpy(o, t.out, sizeof(o), cudaMemcpyDeviceToHost));
      max_rank = std::max(max_rank, o[0]);
      max_cols = std::max(max_cols, t.n - o[0]);
    }
    id_solve_run(tasks, ntask, max_rank, max_cols, s);
  }

}  // namespace hssmf_b200
