#include "staging.cuh"

#include <algorithm>
#include <cstring>
#include <exception>
#include <map>
#include <memory>
#include <mutex>

namespace hssmf_b200 {

  namespace {
    thread_local Staging* g_cur = nullptr;
  }

  Staging::Staging(cudaStream_t s, size_t chunk_bytes, int chunks)
      : s_(s), chunk_(chunk_bytes), nchunks_(chunks), ev_(chunks), armed_(chunks, 0) {
    HSSMF_CUDA(cudaMallocHost((void**)&h_, chunk_ * nchunks_));
    HSSMF_CUDA(cudaMalloc((void**)&d_, chunk_ * nchunks_));
    for (auto& e : ev_) HSSMF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }

  Staging::~Staging() {
    cudaStreamSynchronize(s_);
    for (auto& e : ev_) cudaEventDestroy(e);
    cudaFreeHost(h_);
    cudaFree(d_);
    if (hr_) cudaFreeHost(hr_);
  }

  bool Staging::d2h(void* dst, const void* src, size_t n) {
    const size_t a = (n + 255) & ~size_t(255);
    if (hr_used_ + a > hr_cap_) {
      if (!pend_.empty()) return false;
      if (hr_) HSSMF_CUDA(cudaFreeHost(hr_));
      hr_cap_ = std::max<size_t>(2 * hr_cap_, std::max<size_t>(a, 1 << 20));
      HSSMF_CUDA(cudaMallocHost((void**)&hr_, hr_cap_));
    }
    HSSMF_CUDA(cudaMemcpyAsync(hr_ + hr_used_, src, n, cudaMemcpyDeviceToHost, s_));
    pend_.push_back({dst, hr_used_, n});
    hr_used_ += a;
    return true;
  }

  void Staging::complete() {
    for (const auto& p : pend_) std::memcpy(p.dst, hr_ + p.off, p.n);
    pend_.clear();
    hr_used_ = 0;
  }

  void Staging::discard() {
    cudaStreamSynchronize(s_);  // no throw: may run during unwinding
    pend_.clear();
    hr_used_ = 0;
  }

  void d2h(void* dst, const void* src, size_t n, cudaStream_t s) {
    if (!n) return;
    if (Staging* st = current_staging(s))
      if (st->d2h(dst, src, n)) return;
    HSSMF_CUDA(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, s));
  }

  char* Staging::stage(const void* src, size_t n, char** dev) {
    const size_t a = (n + 255) & ~size_t(255);
    if (a > chunk_) return nullptr;
    if (head_ + a > chunk_) {
      // leave the current chunk: mark it busy until the stream passes this point
      HSSMF_CUDA(cudaEventRecord(ev_[cur_], s_));
      armed_[cur_] = 1;
      cur_ = (cur_ + 1) % nchunks_;
      head_ = 0;
      if (armed_[cur_]) {
        HSSMF_CUDA(cudaEventSynchronize(ev_[cur_]));
        armed_[cur_] = 0;
      }
    }
    char* h = h_ + (size_t)cur_ * chunk_ + head_;
    *dev = d_ + (size_t)cur_ * chunk_ + head_;
    std::memcpy(h, src, n);
    head_ += a;
    return h;
  }

  void* Staging::put(const void* src, size_t n) {
    char* d = nullptr;
    char* h = stage(src, n, &d);
    if (!h) return nullptr;
    HSSMF_CUDA(cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, s_));
    return d;
  }

  bool Staging::copy_to(void* dst, const void* src, size_t n) {
    char* d = nullptr;
    char* h = stage(src, n, &d);
    if (!h) return false;
    HSSMF_CUDA(cudaMemcpyAsync(dst, h, n, cudaMemcpyHostToDevice, s_));
    return true;
  }

  void h2d(void* dst, const void* src, size_t n, cudaStream_t s) {
    if (!n) return;
    if (Staging* st = current_staging(s))
      if (st->copy_to(dst, src, n)) return;
    HSSMF_CUDA(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, s));
  }

  LowLane* low_lane_for(cudaStream_t s) {
    // opt-in (HSSMF_LANES=1): measured on c5 at 7.61-7.66 s per step against
    // 7.32 s with the priorities alone (and 7.99 s without either): the two
    // event edges per big launch cost more than the earlier dispatch returns
    static const bool off = getenv("HSSMF_NO_PRIO") != nullptr || getenv("HSSMF_LANES") == nullptr;
    if (off || !s) return nullptr;
    static std::mutex mu;
    static std::map<cudaStream_t, std::unique_ptr<LowLane>>* reg =
        new std::map<cudaStream_t, std::unique_ptr<LowLane>>();  // never destroyed
    std::lock_guard<std::mutex> lk(mu);
    auto it = reg->find(s);
    if (it != reg->end()) return it->second.get();
    int least = 0, greatest = 0, prio = 0;
    HSSMF_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    HSSMF_CUDA(cudaStreamGetPriority(s, &prio));
    std::unique_ptr<LowLane> L;
    if (prio == greatest && greatest != least) {
      L.reset(new LowLane());
      HSSMF_CUDA(cudaStreamCreateWithPriority(&L->lo, cudaStreamNonBlocking, least));
      HSSMF_CUDA(cudaEventCreateWithFlags(&L->fork, cudaEventDisableTiming));
      HSSMF_CUDA(cudaEventCreateWithFlags(&L->join, cudaEventDisableTiming));
    }
    LowLane* p = L.get();
    (*reg)[s] = std::move(L);
    return p;
  }

  BigLaunch::BigLaunch(cudaStream_t st, bool big) : s(st), lane(big ? low_lane_for(st) : nullptr) {
    if (!lane) return;
    HSSMF_CUDA(cudaEventRecord(lane->fork, s));
    HSSMF_CUDA(cudaStreamWaitEvent(lane->lo, lane->fork, 0));
  }
  BigLaunch::~BigLaunch() {
    if (!lane) return;
    cudaEventRecord(lane->join, lane->lo);
    cudaStreamWaitEvent(s, lane->join, 0);
  }

  Staging* staging_for(cudaStream_t s) {
    static std::mutex mu;
    static std::map<cudaStream_t, std::unique_ptr<Staging>>* reg =
        new std::map<cudaStream_t, std::unique_ptr<Staging>>();  // never destroyed
    std::lock_guard<std::mutex> lk(mu);
    auto& p = (*reg)[s];
    if (!p) p.reset(new Staging(s));
    return p.get();
  }

  Staging* current_staging(cudaStream_t s) {
    return (g_cur && g_cur->stream() == s) ? g_cur : nullptr;
  }

  StagingScope::StagingScope(Staging* st)
      : prev(g_cur), cur(st), exc(std::uncaught_exceptions()) {
    g_cur = st;
  }
  StagingScope::~StagingScope() {
    if (cur && std::uncaught_exceptions() > exc) cur->discard();
    g_cur = prev;
  }

}  // namespace hssmf_b200
