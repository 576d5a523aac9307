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
