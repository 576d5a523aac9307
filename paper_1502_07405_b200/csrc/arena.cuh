// Per-stream device block cache for the dynamic (HSS) phases.
//
// One HSS front issues hundreds of thousands of small, short-lived device
// allocations (per-node samples, bases, index lists, GEMM scratch). Served by
// cudaMallocAsync / cudaFreeAsync each costs 10-20 us of host time and the
// calls contend across the concurrent front threads, so the host, not the
// GPU, bounded the HSS phases. A DevArena carves blocks from 32 MB slabs and recycles freed blocks by size class,
// so the steady state makes no driver call. Reuse is stream-ordered: every
// block of an arena is only touched by work on the arena's stream, so a block
// returned to the cache may be handed to a later launch on the same stream at
// once. Blocks above kArenaMaxBlock go straight to the stream-ordered pool;
// trim() returns slabs without live blocks to it.
#pragma once

#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace hssmf_b200 {

  class DevArena {
   public:
    static constexpr size_t kArenaMaxBlock = 4u << 20;
    static constexpr size_t kSlabBytes = 32u << 20;

    explicit DevArena(cudaStream_t s) : s_(s) {}
    ~DevArena();
    DevArena(const DevArena&) = delete;
    DevArena& operator=(const DevArena&) = delete;

    cudaStream_t stream() const { return s_; }
    // block of >= bytes; *cls receives the size class (0: not cached)
    void* get(size_t bytes, size_t* cls);
    void put(void* p, size_t cls);
    // return slabs without live blocks to the stream-ordered pool
    void trim();
    // move to another stream: the old one is drained first
    void rebind(cudaStream_t s);
    size_t slab_bytes() const;

   private:
    struct Slab {
      char* base = nullptr;
      size_t size = 0, used = 0;
      long long live = 0;
    };
    cudaStream_t s_;
    std::vector<Slab> slabs_;
    std::unordered_map<void*, int> owner_;  // block -> slab
    std::unordered_map<size_t, std::vector<void*>> free_;
  };

  // thread-local current arena (set by ArenaScope); nullptr if none or if it
  // is bound to another stream
  DevArena* current_arena(cudaStream_t s);
  struct ArenaScope {
    DevArena* prev;
    explicit ArenaScope(DevArena* a);
    ~ArenaScope();
  };

}  // namespace hssmf_b200
