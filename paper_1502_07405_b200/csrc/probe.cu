#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace hssmf_b200 {

  namespace {
    struct Rec {
      int kind;
      cudaEvent_t a, b;
      double flops, bytes;
      int tiles, kmax, nprob, phase;
    };
    std::mutex g_mu;
    std::vector<Rec> g_recs;
    std::atomic<bool> g_on{false};
    unsigned long long* g_dev_bytes = nullptr;
  }  // namespace

  bool probe_enabled() { return g_on.load(std::memory_order_relaxed); }
  int& probe_phase() {
    static thread_local int ph = -1;
    return ph;
  }

  unsigned long long* probe_device_bytes() {
    std::lock_guard<std::mutex> l(g_mu);
    if (!g_dev_bytes) {
      HSSMF_CUDA(cudaMalloc(&g_dev_bytes, sizeof(unsigned long long)));
      HSSMF_CUDA(cudaMemset(g_dev_bytes, 0, sizeof(unsigned long long)));
    }
    return g_dev_bytes;
  }

  void probe_enable(bool on) {
    if (on) probe_device_bytes();
    g_on = on;
  }

  void probe_read(ProbeStat out[PROBE_KINDS]) {
    HSSMF_CUDA(cudaDeviceSynchronize());
    std::lock_guard<std::mutex> l(g_mu);
    for (int k = 0; k < PROBE_KINDS; k++) out[k] = {0, 0.0, 0.0, 0.0};
    // HSSMF_PROBE_DUMP=<path>: one CSV line per probed launch (shape study)
    FILE* dump = nullptr;
    if (const char* pth = getenv("HSSMF_PROBE_DUMP")) dump = fopen(pth, "w");
    if (dump) fprintf(dump, "kind,ms,flops,bytes,tiles,kmax,nprob,phase\n");
    for (auto& r : g_recs) {
      float ms = 0;
      cudaEventElapsedTime(&ms, r.a, r.b);
      if (dump)
        fprintf(dump, "%d,%.4f,%.6g,%.6g,%d,%d,%d,%d\n", r.kind, ms, r.flops, r.bytes, r.tiles,
                r.kmax, r.nprob, r.phase);
      auto& o = out[r.kind];
      o.launches++;
      o.ms += ms;
      o.flops += r.flops;
      o.bytes += r.bytes;
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    g_recs.clear();
    if (dump) fclose(dump);
    if (g_dev_bytes) {
      unsigned long long b = 0;
      HSSMF_CUDA(cudaMemcpy(&b, g_dev_bytes, sizeof(b), cudaMemcpyDeviceToHost));
      HSSMF_CUDA(cudaMemset(g_dev_bytes, 0, sizeof(b)));
      out[PROBE_GRAM_SYRK].bytes += (double)b;
    }
  }

  ProbeScope::ProbeScope(int k, cudaStream_t st, double f, double b)
      : kind(k), s(st), flops(f), bytes(b) {
    if (!probe_enabled()) return;
    HSSMF_CUDA(cudaEventCreate(&a));
    HSSMF_CUDA(cudaEventRecord(a, s));
  }

  ProbeScope::~ProbeScope() {
    if (!a) return;
    cudaEvent_t b;
    if (cudaEventCreate(&b) != cudaSuccess || cudaEventRecord(b, s) != cudaSuccess) return;
    std::lock_guard<std::mutex> l(g_mu);
    g_recs.push_back({kind, a, b, flops, bytes, tiles, kmax, nprob, probe_phase()});
  }

}  // namespace hssmf_b200
