#include "arena.cuh"

namespace hssmf_b200 {

  namespace {
    thread_local DevArena* g_arena = nullptr;

    // 4 classes per power of two, 256 B minimum
    size_t size_class(size_t b) {
      if (b <= 256) return 256;
      size_t p = 256;
      while (p * 2 < b) p *= 2;
      const size_t q = p / 4;
      return (b + q - 1) / q * q;
    }
  }  // namespace

  DevArena::~DevArena() {
    for (auto& sl : slabs_) cudaFreeAsync(sl.base, s_);
  }

  void* DevArena::get(size_t bytes, size_t* cls) {
    if (bytes > kArenaMaxBlock) {
      *cls = 0;
      void* p = nullptr;
      HSSMF_CUDA(cudaMallocAsync(&p, bytes, s_));
      return p;
    }
    const size_t c = size_class(bytes);
    *cls = c;
    auto it = free_.find(c);
    if (it != free_.end() && !it->second.empty()) {
      void* p = it->second.back();
      it->second.pop_back();
      slabs_[owner_[p]].live++;
      return p;
    }
    if (slabs_.empty() || slabs_.back().used + c > slabs_.back().size) {
      Slab sl;
      sl.size = kSlabBytes;
      HSSMF_CUDA(cudaMallocAsync((void**)&sl.base, sl.size, s_));
      slabs_.push_back(sl);
    }
    Slab& sl = slabs_.back();
    void* p = sl.base + sl.used;
    sl.used += c;
    sl.live++;
    owner_[p] = (int)slabs_.size() - 1;
    return p;
  }

  void DevArena::put(void* p, size_t cls) {
    if (!p) return;
    if (cls == 0) {
      cudaFreeAsync(p, s_);
      return;
    }
    slabs_[owner_[p]].live--;
    free_[cls].push_back(p);
  }

  void DevArena::trim() {
    // slabs without a live block go back to the stream-ordered pool
    bool any = false;
    for (auto& sl : slabs_) any |= sl.live == 0;
    if (!any) return;
    std::vector<int> remap(slabs_.size(), -1);
    std::vector<Slab> keep;
    for (size_t i = 0; i < slabs_.size(); i++) {
      if (slabs_[i].live == 0) {
        cudaFreeAsync(slabs_[i].base, s_);
      } else {
        remap[i] = (int)keep.size();
        keep.push_back(slabs_[i]);
      }
    }
    for (auto& kv : free_) {
      std::vector<void*> v;
      for (void* p : kv.second)
        if (remap[owner_[p]] >= 0) v.push_back(p);
      kv.second.swap(v);
    }
    for (auto it = owner_.begin(); it != owner_.end();) {
      if (remap[it->second] < 0) {
        it = owner_.erase(it);
      } else {
        it->second = remap[it->second];
        ++it;
      }
    }
    slabs_.swap(keep);
    // a partially used last slab keeps taking new blocks; a fresh one starts
    // after a retained one only when that is full
  }

  size_t DevArena::slab_bytes() const {
    size_t b = 0;
    for (const auto& sl : slabs_) b += sl.size;
    return b;
  }

  void DevArena::rebind(cudaStream_t s) {
    if (s == s_) return;
    stream_sync(s_);
    s_ = s;
  }

  DevArena* current_arena(cudaStream_t s) {
    return (g_arena && g_arena->stream() == s) ? g_arena : nullptr;
  }
  ArenaScope::ArenaScope(DevArena* a) : prev(g_arena) { g_arena = a; }
  ArenaScope::~ArenaScope() { g_arena = prev; }

}  // namespace hssmf_b200
