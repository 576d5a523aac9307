#include "rng.cuh"

namespace hssmf_b200 {

  namespace {
    constexpr unsigned long long kMod = 2147483647ull, kMul = 48271ull;

    __device__ __forceinline__ unsigned long long mulmod(unsigned long long a,
                                                         unsigned long long b) {
      return (a * b) % kMod;
    }
    __device__ __forceinline__ unsigned long long powmod(unsigned long long b,
                                                         unsigned long long e) {
      unsigned long long r = 1;
      while (e) {
        if (e & 1) r = mulmod(r, b);
        b = mulmod(b, b);
        e >>= 1;
      }
      return r;
    }

    // thread per row; walks the row's stream from pair c0/2 and writes
    // column-major (coalesced across rows)
    __global__ void rng_kernel(const long long* __restrict__ grow, long long row0, int nrows,
                               int c0, int c1, double* __restrict__ out, long long ldo) {
      const int l = blockIdx.x * blockDim.x + threadIdx.x;
      if (l >= nrows) return;
      const long long g = grow ? grow[l] : row0 + l;
      unsigned long long x = (unsigned long long)(g + 1) % kMod;
      if (x == 0) x = 1;
      const int q0 = c0 / 2;
      x = mulmod(x, powmod(kMul, 2ull * q0));
      for (int q = q0; 2 * q < c1; q++) {
        x = mulmod(x, kMul);
        const double u1 = (double)x / (double)kMod;
        x = mulmod(x, kMul);
        const double u2 = (double)x / (double)kMod;
        const double rad = sqrt(-2.0 * log(u1));
        const double ang = 2.0 * 3.14159265358979323846 * u2;
        double sn, cs;
        sincos(ang, &sn, &cs);
        const int c = 2 * q;
        if (c >= c0) out[l + (c - c0) * ldo] = rad * cs;
        if (c + 1 >= c0 && c + 1 < c1) out[l + (c + 1 - c0) * ldo] = rad * sn;
      }
    }
  }  // namespace

  void rng_fill(const long long* grow, long long row0, int nrows, int c0, int c1, double* out,
                long long ldo, cudaStream_t s) {
    if (nrows <= 0 || c1 <= c0) return;
    rng_kernel<<<ceil_div(nrows, 128), 128, 0, s>>>(grow, row0, nrows, c0, c1, out, ldo);
    HSSMF_LAUNCH_CHECK();
  }

}  // namespace hssmf_b200
