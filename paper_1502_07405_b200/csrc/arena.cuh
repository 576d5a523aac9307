// Per-stream device block cache for the dynamic (HSS) phases.
//
// One HSS front issues hundreds of thousands of small, short-lived device
// allocations (per-node samples, bases, index lists, GEMM scratch). Served by
// cudaMallocAsync / cudaFreeAsync each costs 10-20 us of host time and the
// calls contend across the concurrent front threads, so the host, not the
// GPU, bounded the HSS phases. A DevArena carves power-of-two blocks from
// 32 MB slabs with a binary buddy allocator (freed buddies merge back), so
// the steady state makes no driver call. Reuse is stream-ordered: every
// block of an arena is only touched by work on the arena's stream, so a block
// returned to the cache may be handed to a later launch on the same stream at
// once. Blocks above kArenaMaxBlock go straight to the stream-ordered pool;
// trim() returns slabs without live blocks to it.
#pragma once

#include <atomic>
#include <set>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace hssmf_b200 {

  class DevArena {
   public:
    static constexpr size_t kMinBlock = 256;
    static constexpr int kMaxOrder = 17;  // 256 B << 17 = 32 MB slabs
    static constexpr size_t kSlabBytes = kMinBlock << kMaxOrder;
    static constexpr size_t kArenaMaxBlock = 4u << 20;

    explicit DevArena(cudaStream_t s) : s_(s) {}
    ~DevArena();
    DevArena(const DevArena&) = delete;
    DevArena& operator=(const DevArena&) = delete;

    cudaStream_t stream() const { return s_; }
    // block of >= bytes; *cls receives the block's class (0: not from a slab)
    void* get(size_t bytes, size_t* cls);
    void put(void* p, size_t cls, size_t bytes);
    // optional usage meter (bytes handed out and not yet returned), read by
    // the engine's memory admission while the front runs
    void set_meter(std::atomic<long long>* m) { meter_ = m; }
    // return slabs without live blocks to the stream-ordered pool
    void trim();
    // move to another stream: the old one is drained first
    void rebind(cudaStream_t s);
    size_t slab_bytes() const;
    size_t live_bytes() const { return live_bytes_; }

   private:
    struct Slab {
      char* base = nullptr;
      long long live = 0;
    };
    static int order_of(size_t bytes);
    void new_slab();
    void insert_free(char* p, int o);
    void erase_free(char* p, int o);
    int slab_of(const char* p) const;

    cudaStream_t s_;
    std::vector<Slab> slabs_;
    // binary buddy free lists (power-of-two blocks, merged on release)
    std::set<char*> free_[kMaxOrder + 1];
    std::unordered_map<char*, int> free_order_;
    size_t live_bytes_ = 0;
    std::atomic<long long>* meter_ = nullptr;
  };

  // meter picked up by the arenas of HSS objects created on this thread
  std::atomic<long long>*& current_meter();

  // thread-local current arenas (set by ArenaScope): scratch blocks and blocks
  // that outlive the compression (the factor data); nullptr if none or bound
  // to another stream
  DevArena* current_arena(cudaStream_t s);
  DevArena* current_keep_arena(cudaStream_t s);
  struct ArenaScope {
    DevArena* prev;
    DevArena* prev_keep;
    ArenaScope(DevArena* a, DevArena* keep);
    ~ArenaScope();
  };

}  // namespace hssmf_b200
