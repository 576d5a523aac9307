// Pinned host -> device staging ring for small per-launch descriptor arrays.
//
// The dynamic (HSS) phases upload a few hundred bytes of descriptors before
// almost every launch. A ring of pinned chunks makes each upload one truly
// asynchronous cudaMemcpyAsync, with no per-launch device allocation; a chunk
// is reused only after an event recorded behind its last consumer has
// completed. A Staging is bound to one stream and made current for the
// calling thread with StagingScope; gemm_run_host / index_copy_run / the ULV
// solve launchers use it when the stream matches.
#pragma once

#include <vector>

#include "common.cuh"

namespace hssmf_b200 {

  class Staging {
   public:
    explicit Staging(cudaStream_t s, size_t chunk_bytes = 256 << 10, int chunks = 64);
    ~Staging();
    Staging(const Staging&) = delete;
    Staging& operator=(const Staging&) = delete;
    cudaStream_t stream() const { return s_; }
    // device copy of n host bytes, stream-ordered; nullptr if n exceeds a chunk
    void* put(const void* src, size_t n);
    // stream-ordered copy of n host bytes to the device address dst through a
    // pinned chunk (false if n exceeds a chunk)
    bool copy_to(void* dst, const void* src, size_t n);
    // device -> host read of n bytes into dst, staged through pinned memory
    // and delivered to dst by complete() (stream_sync calls it); false if the
    // pinned buffer cannot take it now
    bool d2h(void* dst, const void* src, size_t n);
    void complete();
    // drop the pending reads without delivering them (their destinations may
    // be gone): waits for the stream, then clears the landing area
    void discard();

   private:
    char* stage(const void* src, size_t n, char** dev);
    cudaStream_t s_;
    size_t chunk_;
    int nchunks_, cur_ = 0;
    size_t head_ = 0;
    char* h_ = nullptr;
    char* d_ = nullptr;
    std::vector<cudaEvent_t> ev_;
    std::vector<char> armed_;
    // pinned landing area of the pending device -> host reads
    struct Pending {
      void* dst;
      size_t off, n;
    };
    char* hr_ = nullptr;
    size_t hr_cap_ = 0, hr_used_ = 0;
    std::vector<Pending> pend_;
  };

  // host -> device copy through the current staging ring of s when there is
  // one (pinned, truly asynchronous), else a plain cudaMemcpyAsync
  void h2d(void* dst, const void* src, size_t n, cudaStream_t s);
  // device -> host read that the next stream_sync(s) completes (a pageable
  // cudaMemcpyAsync blocks inside the driver and serialises the other front
  // threads' CUDA calls; a pinned one does not)
  void d2h(void* dst, const void* src, size_t n, cudaStream_t s);

  // Low-priority lane of a high-priority worker stream. The fronts of one tree
  // level run concurrently, each a chain of small, latency-bound launches
  // (pivot panels, index copies, small GEMMs) interleaved with full-device
  // kernels (big GEMMs, Gram trailing updates). At equal priority a small
  // kernel queues behind every CTA the other fronts' big grids still have to
  // dispatch. Worker streams therefore run at the highest priority and send
  // their big kernels through a lowest-priority lane: BigLaunch orders the
  // lane after everything enqueued on the worker stream (fork event) and the
  // worker stream after the kernel (join event), so the stream's order of
  // operations is unchanged; only the CTA dispatch priority differs.
  // The priorities alone are the default; the lanes are opt-in (HSSMF_LANES=1,
  // measured slower, see low_lane_for). HSSMF_NO_PRIO=1: every stream at the
  // default priority.
  struct LowLane {
    cudaStream_t lo = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
  };
  LowLane* low_lane_for(cudaStream_t s);  // nullptr unless s is a high-priority stream
  struct BigLaunch {
    cudaStream_t s;
    LowLane* lane;
    BigLaunch(cudaStream_t st, bool big);
    ~BigLaunch();
    cudaStream_t stream() const { return lane ? lane->lo : s; }
    BigLaunch(const BigLaunch&) = delete;
    BigLaunch& operator=(const BigLaunch&) = delete;
  };

  // process-wide ring per stream (created on first use)
  Staging* staging_for(cudaStream_t s);
  // thread-local current staging ring
  Staging* current_staging(cudaStream_t s);
  // Binds st for the calling thread. Leaving the scope by an exception
  // discards st's pending device -> host reads: their destinations are stack or
  // local buffers of the unwound frames, and the ring is pooled with its stream,
  // so the next stream_sync would otherwise write into freed memory.
  struct StagingScope {
    Staging* prev;
    Staging* cur;
    int exc;
    explicit StagingScope(Staging* st);
    ~StagingScope();
  };

}  // namespace hssmf_b200
