#include "krylov.hpp"

#include <cmath>

#include "common.cuh"
#include "engine.hpp"

namespace hssmf_b200 {

  namespace {
    constexpr int KT = 256, KB = 296;  // 2 CTAs per SM for the reductions

    __global__ void spmv_kernel(CsrDevView a, const double* __restrict__ x, double* __restrict__ y) {
      const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
      if (row >= a.n) return;
      double s = 0;
      for (int k = a.ptr[row] + lane; k < a.ptr[row + 1]; k += 32) s += a.val[k] * x[a.ind[k]];
      for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
      if (lane == 0) y[row] = s;
    }

    // partial dot products in a fixed order (deterministic)
    __global__ void __launch_bounds__(KT) dot_partial(const double* __restrict__ a,
                                                      const double* __restrict__ b, long long n,
                                                      double* __restrict__ part) {
      double s = 0;
      for (long long i = (long long)blockIdx.x * KT + threadIdx.x; i < n; i += (long long)KB * KT)
        s += a[i] * b[i];
      __shared__ double sm[KT];
      sm[threadIdx.x] = s;
      __syncthreads();
      for (int w = KT / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
        __syncthreads();
      }
      if (threadIdx.x == 0) part[blockIdx.x] = sm[0];
    }
    __global__ void dot_final(const double* __restrict__ part, double* __restrict__ out) {
      __shared__ double sm[512];
      sm[threadIdx.x] = threadIdx.x < KB ? part[threadIdx.x] : 0.0;
      __syncthreads();
      for (int w = 256; w > 0; w >>= 1) {
        if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
        __syncthreads();
      }
      if (threadIdx.x == 0) *out = sm[0];
    }

    __global__ void axpy_kernel(long long n, double alpha, const double* __restrict__ x,
                                double* __restrict__ y) {
      for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
           i += (long long)gridDim.x * blockDim.x)
        y[i] += alpha * x[i];
    }
    __global__ void div_kernel(long long n, double beta, const double* __restrict__ x,
                               double* __restrict__ y) {
      for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
           i += (long long)gridDim.x * blockDim.x)
        y[i] = x[i] / beta;
    }
    __global__ void sub_kernel(long long n, const double* __restrict__ b, double* __restrict__ y) {
      for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
           i += (long long)gridDim.x * blockDim.x)
        y[i] = b[i] - y[i];
    }

    struct Dev {
      double* p = nullptr;
      explicit Dev(size_t n) { HSSMF_CUDA(cudaMalloc((void**)&p, std::max<size_t>(n, 1) * 8)); }
      ~Dev() { cudaFree(p); }
    };

    struct Ops {
      const CsrDevView& a;
      Engine* m;
      cudaStream_t s;
      int n;
      Dev part, res;
      double* hres = nullptr;
      Ops(const CsrDevView& aa, Engine* mm, cudaStream_t ss)
          : a(aa), m(mm), s(ss), n(aa.n), part(KB), res(1) {
        HSSMF_CUDA(cudaMallocHost((void**)&hres, sizeof(double)));
      }
      ~Ops() { cudaFreeHost(hres); }
      int grid() const { return std::min(ceil_div(n, 256), 148 * 8); }
      void spmv(const double* x, double* y) {
        spmv_kernel<<<ceil_div((long long)n * 32, 256), 256, 0, s>>>(a, x, y);
        HSSMF_LAUNCH_CHECK();
      }
      double dot(const double* x, const double* y) {
        dot_partial<<<KB, KT, 0, s>>>(x, y, n, part.p);
        HSSMF_LAUNCH_CHECK();
        dot_final<<<1, 512, 0, s>>>(part.p, res.p);
        HSSMF_LAUNCH_CHECK();
        HSSMF_CUDA(cudaMemcpyAsync(hres, res.p, sizeof(double), cudaMemcpyDeviceToHost, s));
        HSSMF_CUDA(cudaStreamSynchronize(s));
        return *hres;
      }
      double nrm2(const double* x) { return std::sqrt(dot(x, x)); }
      void axpy(double alpha, const double* x, double* y) {
        axpy_kernel<<<grid(), 256, 0, s>>>(n, alpha, x, y);
        HSSMF_LAUNCH_CHECK();
      }
      void div(double beta, const double* x, double* y) {
        div_kernel<<<grid(), 256, 0, s>>>(n, beta, x, y);
        HSSMF_LAUNCH_CHECK();
      }
      void copy(const double* x, double* y) {
        HSSMF_CUDA(cudaMemcpyAsync(y, x, (size_t)n * 8, cudaMemcpyDeviceToDevice, s));
      }
      // y = M^-1 x (identity without factors)
      void minv(const double* x, double* y) {
        copy(x, y);
        if (m) {
          HSSMF_CUDA(cudaStreamSynchronize(s));
          m->solve(y, n, 1, true);
        }
      }
      // u = M^-1 (b - A x)  (detail::precond_residual, krylov.hpp:62-72)
      void precond_residual(const double* b, const double* x, double* u, double* tmp) {
        spmv(x, tmp);
        sub_kernel<<<grid(), 256, 0, s>>>(n, b, tmp);
        HSSMF_LAUNCH_CHECK();
        minv(tmp, u);
      }
    };
  }  // namespace

  KrylovReport krylov_gmres(const CsrDevView& a, Engine* m, const double* b, double* x,
                            int restart, double rtol, double atol, int maxit, cudaStream_t s0) {
    if (restart < 1) throw SolverFailure(1, -1, -1, "gmres: restart must be >= 1");
    const cudaStream_t s = m ? m->stream() : s0;
    Ops op(a, m, s);
    const int n = a.n;
    Dev u(n), tmp(n), w(n), V((size_t)n * (restart + 1));
    HSSMF_CUDA(cudaMemsetAsync(x, 0, (size_t)n * 8, s));
    KrylovReport rep;
    op.precond_residual(b, x, u.p, tmp.p);
    const double u0 = op.nrm2(u.p);
    double resid = u0;
    rep.history.push_back(resid);
    auto done = [&](double r) { return r <= atol || (u0 > 0 && r / u0 <= rtol); };
    std::vector<double> h((size_t)(restart + 1) * restart), cs(restart), sn(restart),
        g(restart + 1);
    auto hij = [&](int i, int j) -> double& { return h[(size_t)j * (restart + 1) + i]; };
    auto vcol = [&](int j) { return V.p + (size_t)j * n; };
    rep.converged = done(resid);
    while (!rep.converged && rep.iterations < maxit) {
      const double beta = op.nrm2(u.p);
      if (beta == 0.0) {
        rep.converged = true;
        break;
      }
      op.div(beta, u.p, vcol(0));
      std::fill(g.begin(), g.end(), 0.0);
      g[0] = beta;
      int j = 0;
      bool breakdown = false;
      for (; j < restart && rep.iterations < maxit; j++) {
        op.spmv(vcol(j), tmp.p);
        op.minv(tmp.p, w.p);
        for (int i = 0; i <= j; i++) {  // modified Gram-Schmidt
          hij(i, j) = op.dot(vcol(i), w.p);
          op.axpy(-hij(i, j), vcol(i), w.p);
        }
        const double wn = op.nrm2(w.p);
        hij(j + 1, j) = wn;
        bool finite = std::isfinite(wn);
        for (int i = 0; i <= j && finite; i++) finite = std::isfinite(std::fabs(hij(i, j)));
        if (!finite)
          throw KrylovDivergence("gmres: non-finite Arnoldi entry at iteration " +
                                 std::to_string(rep.iterations + 1));
        for (int i = 0; i < j; i++) {
          const double t = cs[i] * hij(i, j) + sn[i] * hij(i + 1, j);
          hij(i + 1, j) = -sn[i] * hij(i, j) + cs[i] * hij(i + 1, j);
          hij(i, j) = t;
        }
        // rotg (krylov.hpp:76-82), real case
        const double d = hij(j, j), sj = hij(j + 1, j), ad = std::fabs(d);
        double c, sg;
        if (ad == 0.0) {
          c = 0.0;
          sg = 1.0;
        } else {
          const double den = std::sqrt(ad * ad + std::fabs(sj) * std::fabs(sj));
          c = ad / den;
          sg = (d / ad) * sj / den;
        }
        cs[j] = c;
        sn[j] = sg;
        hij(j, j) = c * hij(j, j) + sg * hij(j + 1, j);
        hij(j + 1, j) = 0.0;
        g[j + 1] = -sg * g[j];
        g[j] = c * g[j];
        resid = std::fabs(g[j + 1]);
        rep.iterations++;
        rep.history.push_back(resid);
        if (wn == 0.0) {  // happy breakdown: the solution is exact
          breakdown = true;
          j++;
          break;
        }
        op.div(wn, w.p, vcol(j + 1));
        if (done(resid)) {
          j++;
          break;
        }
      }
      std::vector<double> y(j);
      for (int i = j - 1; i >= 0; i--) {
        double t = g[i];
        for (int l = i + 1; l < j; l++) t -= hij(i, l) * y[l];
        y[i] = t / hij(i, i);
      }
      for (int i = 0; i < j; i++) op.axpy(y[i], vcol(i), x);
      op.precond_residual(b, x, u.p, tmp.p);
      resid = op.nrm2(u.p);
      rep.converged = breakdown || done(resid);
    }
    rep.abs_resid = resid;
    rep.rel_resid = u0 > 0 ? resid / u0 : 0.0;
    HSSMF_CUDA(cudaStreamSynchronize(s));
    return rep;
  }

  KrylovReport krylov_refine(const CsrDevView& a, Engine* m, const double* b, double* x,
                             double rtol, double atol, int maxit, cudaStream_t s0) {
    const cudaStream_t s = m ? m->stream() : s0;
    Ops op(a, m, s);
    const int n = a.n;
    Dev u(n), tmp(n);
    HSSMF_CUDA(cudaMemsetAsync(x, 0, (size_t)n * 8, s));
    KrylovReport rep;
    op.precond_residual(b, x, u.p, tmp.p);
    const double u0 = op.nrm2(u.p);
    double resid = u0;
    rep.history.push_back(resid);
    auto done = [&](double r) { return r <= atol || (u0 > 0 && r / u0 <= rtol); };
    rep.converged = done(resid);
    while (!rep.converged && rep.iterations < maxit) {
      if (!std::isfinite(resid))
        throw KrylovDivergence("refinement: non-finite residual at iteration " +
                               std::to_string(rep.iterations));
      op.axpy(1.0, u.p, x);
      rep.iterations++;
      op.precond_residual(b, x, u.p, tmp.p);
      resid = op.nrm2(u.p);
      rep.history.push_back(resid);
      rep.converged = done(resid);
      const size_t k = rep.history.size();
      if (!rep.converged && k >= 4 && rep.history[k - 4] < 2 * rep.history[k - 1])
        rep.stagnated = true;
    }
    rep.abs_resid = resid;
    rep.rel_resid = u0 > 0 ? resid / u0 : 0.0;
    HSSMF_CUDA(cudaStreamSynchronize(s));
    return rep;
  }

}  // namespace hssmf_b200
