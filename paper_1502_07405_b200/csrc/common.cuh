// Shared device helpers for the sm_100a kernels of the HSS-multifrontal path.
#pragma once

#include <cuda_runtime.h>

#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace hssmf_b200 {

  struct CudaError : std::runtime_error {
    explicit CudaError(const std::string& s) : std::runtime_error(s) {}
  };

#define HSSMF_CUDA(call)                                                              \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      throw ::hssmf_b200::CudaError(std::string(#call) + ": " + cudaGetErrorString(e_) + \
                                    " at " __FILE__ ":" + std::to_string(__LINE__));  \
  } while (0)

  // host-side count of kernel launches issued by this library (bench.py
  // reports it as gpu_launches)
  std::atomic<long long>& launch_counter();
#define HSSMF_LAUNCH_CHECK()                 \
  do {                                       \
    ++::hssmf_b200::launch_counter();        \
    HSSMF_CUDA(cudaGetLastError());          \
  } while (0)

  // NVTX range for timeline tools (nsys / ncu --nvtx); header-only NVTX 3,
  // a no-op pointer check when no tool is attached
  struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
  };

  inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

  // Runs f once per CUDA device for one call site (`done` is that site's device
  // bitmask). Function attributes (dynamic shared memory, non-portable cluster
  // sizes) are per device, and the factor entry points run on worker threads,
  // so a plain static flag is both racy and wrong for a second device.
  template <class F>
  void once_per_device(std::atomic<unsigned long long>& done, F&& f) {
    int dev = 0;
    HSSMF_CUDA(cudaGetDevice(&dev));
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    f();  // idempotent: two threads racing here both set the same attributes
    done.fetch_or(bit, std::memory_order_acq_rel);
  }

  // host time the calling thread spent blocked in stream_sync (seconds) and the
  // number of such waits: HSSMF_DEBUG splits a front's wall time into host work
  // and GPU waits with it
  struct SyncClock {
    double wait_s = 0;
    long long n = 0;
  };
  SyncClock& sync_clock();
  void stream_sync(cudaStream_t s);

  // ---- device-side ----------------------------------------------------------
#ifdef __CUDACC__
  // one FP64 tensor-core MMA: D(8x8) += A(8x4) * B(4x8).
  // lane layout (PTX m8n8k4 .f64): a = A[lane>>2][lane&3], b = B[lane&3][lane>>2],
  // c[v] = C[lane>>2][2*(lane&3)+v]
  __device__ __forceinline__ void dmma8x8x4(double (&c)[2], double a, double b) {
    asm volatile(
        "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c[0]), "+d"(c[1])
        : "d"(a), "d"(b));
  }

  __device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int sz = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
  }
  __device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;\n" ::);
  }
  template<int N> __device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
  }

  // block-wide argmax of |v| with the lowest index winning ties
  // (partial pivoting rule, reference lu.hpp:22-26). blockDim multiple of 32.
  __device__ __forceinline__ void warp_argmax(double& v, int& i) {
    for (int o = 16; o > 0; o >>= 1) {
      const double v2 = __shfl_down_sync(0xffffffffu, v, o);
      const int i2 = __shfl_down_sync(0xffffffffu, i, o);
      if (v2 > v || (v2 == v && i2 < i)) {
        v = v2;
        i = i2;
      }
    }
  }
#endif

}  // namespace hssmf_b200

namespace hssmf_b200 {
  // ---- per-kernel device-time probes (bench.py's roofline entries) ----------
  // When enabled, the launchers of the probed kernels bracket every launch with
  // CUDA events on the launching stream and record the launch's algorithmic
  // flops / bytes; probe_read() synchronizes the device, sums and resets.
  enum ProbeKind { PROBE_GEMM = 0, PROBE_GRAM_PANEL = 1, PROBE_GRAM_SYRK = 2, PROBE_KINDS = 3 };
  struct ProbeStat {
    long long launches;
    double ms, flops, bytes;
  };
  bool probe_enabled();
  void probe_enable(bool on);
  void probe_read(ProbeStat out[PROBE_KINDS]);
  // device counter the Gram SYRK kernel adds its live tasks' algorithmic bytes
  // to (stopped tasks are skipped on the device, so the host cannot count them)
  unsigned long long* probe_device_bytes();
  // HSS phase tag of the calling thread (recorded with each probed launch)
  int& probe_phase();
  struct ProbeScope {
    int kind;
    cudaStream_t s;
    double flops, bytes;
    cudaEvent_t a = nullptr;
    int tiles = 0, kmax = 0, nprob = 0;  // GEMM shape summary (HSSMF_PROBE_DUMP)
    int phase = -1;                      // HSS phase of the launching thread
    ProbeScope(int k, cudaStream_t st, double f, double b);
    ~ProbeScope();
  };
}  // namespace hssmf_b200
