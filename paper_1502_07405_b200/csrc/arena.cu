#include "arena.cuh"

namespace hssmf_b200 {

  namespace {
    thread_local DevArena* g_arena = nullptr;
    thread_local DevArena* g_keep = nullptr;
  }  // namespace

  DevArena::~DevArena() {
    for (auto& sl : slabs_) cudaFreeAsync(sl.base, s_);
  }

  int DevArena::order_of(size_t bytes) {
    int o = 0;
    while ((kMinBlock << o) < bytes) o++;
    return o;
  }

  void DevArena::new_slab() {
    Slab sl;
    HSSMF_CUDA(cudaMallocAsync((void**)&sl.base, kSlabBytes, s_));
    slabs_.push_back(sl);
    insert_free(sl.base, kMaxOrder);
  }

  void DevArena::insert_free(char* p, int o) {
    free_[o].insert(p);
    free_order_[p] = o;
  }

  void DevArena::erase_free(char* p, int o) {
    free_[o].erase(p);
    free_order_.erase(p);
  }

  int DevArena::slab_of(const char* p) const {
    for (size_t i = 0; i < slabs_.size(); i++)
      if (p >= slabs_[i].base && p < slabs_[i].base + kSlabBytes) return (int)i;
    return -1;
  }

  void* DevArena::get(size_t bytes, size_t* cls) {
    if (bytes > kArenaMaxBlock) {
      *cls = 0;
      void* p = nullptr;
      HSSMF_CUDA(cudaMallocAsync(&p, bytes, s_));
      if (meter_) *meter_ += (long long)bytes;
      return p;
    }
    const int want = order_of(bytes);
    int o = want;
    while (o <= kMaxOrder && free_[o].empty()) o++;
    if (o > kMaxOrder) {
      new_slab();
      o = kMaxOrder;
    }
    char* p = *free_[o].begin();
    erase_free(p, o);
    // split down to the wanted order, the upper halves stay free
    while (o > want) {
      o--;
      insert_free(p + (kMinBlock << o), o);
    }
    *cls = (size_t)want + 1;
    slabs_[slab_of(p)].live++;
    live_bytes_ += kMinBlock << want;
    if (meter_) *meter_ += (long long)(kMinBlock << want);
    return p;
  }

  void DevArena::put(void* vp, size_t cls, size_t bytes) {
    if (!vp) return;
    if (cls == 0) {
      cudaFreeAsync(vp, s_);
      if (meter_) *meter_ -= (long long)bytes;
      return;
    }
    char* p = static_cast<char*>(vp);
    int o = (int)cls - 1;
    if (meter_) *meter_ -= (long long)(kMinBlock << o);
    const int si = slab_of(p);
    Slab& sl = slabs_[si];
    sl.live--;
    live_bytes_ -= kMinBlock << o;
    // merge with free buddies
    while (o < kMaxOrder) {
      const size_t off = (size_t)(p - sl.base);
      char* buddy = sl.base + (off ^ (kMinBlock << o));
      auto it = free_order_.find(buddy);
      if (it == free_order_.end() || it->second != o) break;
      erase_free(buddy, o);
      p = std::min(p, buddy);
      o++;
    }
    insert_free(p, o);
  }

  void DevArena::trim() {
    std::vector<Slab> keep;
    for (auto& sl : slabs_) {
      if (sl.live == 0) {
        erase_free(sl.base, kMaxOrder);
        cudaFreeAsync(sl.base, s_);
      } else {
        keep.push_back(sl);
      }
    }
    slabs_.swap(keep);
  }

  size_t DevArena::slab_bytes() const { return slabs_.size() * kSlabBytes; }

  void DevArena::rebind(cudaStream_t s) {
    if (s == s_) return;
    stream_sync(s_);
    s_ = s;
  }

  std::atomic<long long>*& current_meter() {
    static thread_local std::atomic<long long>* m = nullptr;
    return m;
  }

  DevArena* current_arena(cudaStream_t s) {
    return (g_arena && g_arena->stream() == s) ? g_arena : nullptr;
  }
  DevArena* current_keep_arena(cudaStream_t s) {
    return (g_keep && g_keep->stream() == s) ? g_keep : nullptr;
  }
  ArenaScope::ArenaScope(DevArena* a, DevArena* keep) : prev(g_arena), prev_keep(g_keep) {
    g_arena = a;
    g_keep = keep;
  }
  ArenaScope::~ArenaScope() {
    g_arena = prev;
    g_keep = prev_keep;
  }

}  // namespace hssmf_b200
