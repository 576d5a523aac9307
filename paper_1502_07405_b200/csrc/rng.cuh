// Counter-based restatement of the reference's seeded row sampler
// (SeededRowSampler, random_sampler.hpp:19-68): row g owns the minstd stream
// x <- 48271 x mod (2^31-1) seeded (g+1) mod (2^31-1) (0 -> 1); consecutive
// uniform pairs (u1, u2) give Box-Muller variates cos then sin. Entry (l, c)
// only depends on (global row, c), so the device jumps straight to pair c/2
// with a modular power instead of replaying the stream.
#pragma once

#include "common.cuh"

namespace hssmf_b200 {

  // out(l, c - c0) for l < nrows, c in [c0, c1); rows named by grow (device)
  // either as an explicit list or, if grow == nullptr, as row0 + l
  void rng_fill(const long long* grow, long long row0, int nrows, int c0, int c1, double* out,
                long long ldo, cudaStream_t s);

}  // namespace hssmf_b200
