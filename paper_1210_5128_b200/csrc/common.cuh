// Shared device helpers for the bnmc B200 hot path (sm_100a).
//
// Reference semantics are cited as file:line relative to /root/reference/proj.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

namespace bnmc_dev {

constexpr int kMaxNodes = 64;  // types.hpp:14

// Pascal table C(n,k), n,k <= 64 (combinatorics.hpp:14-24), in constant memory.
// Single translation unit (bnmc_gpu.cu) includes this header: defined here.
__constant__ uint64_t c_binom[65][65];

__device__ __forceinline__ uint64_t binom(int n, int k) {
  return (k < 0 || n < 0 || k > n) ? 0ull : c_binom[n][k];
}

// Candidate position q of row v -> node id (index_of inverse, scoring.hpp:133-139).
__device__ __forceinline__ int cand_node(int q, int v) { return q < v ? q : q + 1; }

// Candidate-position mask -> node mask for row v.
// Bit select with a constant shift (two LOP3 + a funnel shift): identical to
// (cm & lm) | ((cm >> v) << (v + 1)) for every v in [0, 63].
__device__ __forceinline__ uint64_t cand_to_nodes(uint64_t cm, int v) {
  const uint64_t lm = (1ull << v) - 1ull;
  const uint64_t lm2 = (lm << 1) | 1ull;  // bits 0..v
  return (cm & lm) | ((cm << 1) & ~lm2);
}

// Node mask -> candidate-position mask for row v (ScoreCache::index_of,
// scoring.hpp:135-137).
// Identical to (pm & lm) | ((pm >> (v + 1)) << v) for every v in [0, 63]
// (bit v of pm is dropped either way), as a bit select.
__device__ __host__ __forceinline__ uint64_t nodes_to_cand(uint64_t pm, int v) {
  const uint64_t lm = (1ull << v) - 1ull;
  return (pm & lm) | ((pm >> 1) & ~lm);
}

// PpfTable::sum (scoring.hpp:103-107): ascending parents, starting from 0.0.
__device__ __forceinline__ double ppf_sum(const double* __restrict__ w, int n, int v,
                                          uint64_t node_mask) {
  double t = 0.0;
  for (uint64_t m = node_mask; m; m &= m - 1) t += w[v * n + __ffsll((long long)m) - 1];
  return t;
}

// Exact x % d for a fixed divisor 2 <= d < 2^32 without a 64-bit division
// (the generic one is ~100 instructions, issued every iteration by
// propose_swap): m = floor((2^64 - 1) / d), q = umulhi(x, m) is floor(x / d)
// minus at most 2, so at most two corrections. thr = (0 - d) % d is
// next_below's rejection threshold (rng.hpp:31-38).
struct FastDiv {
  uint64_t d, m, thr;
  __device__ __host__ static FastDiv make(uint64_t d) {
    return FastDiv{d, ~0ull / d, (0 - d) % d};
  }
  __device__ __host__ uint64_t mod(uint64_t x) const {
#ifdef __CUDA_ARCH__
    const uint64_t q = __umul64hi(x, m);
#else
    const uint64_t q = (uint64_t)(((unsigned __int128)x * m) >> 64);
#endif
    uint64_t r = x - q * d;
    if (r >= d) r -= d;
    if (r >= d) r -= d;
    return r;
  }
};

// splitmix64 Rng (rng.hpp:14-45)
struct Rng {
  uint64_t s;
  __device__ __host__ static uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  __device__ __host__ Rng split(uint64_t tag) const {
    return Rng{mix(s + 0x9E3779B97F4A7C15ull * (tag + 1))};
  }
  __device__ __host__ uint64_t next_u64() {
    s += 0x9E3779B97F4A7C15ull;
    return mix(s);
  }
  __device__ __host__ uint64_t next_below(uint64_t bound) {
    const uint64_t threshold = (0 - bound) % bound;
    uint64_t x;
    do {
      x = next_u64();
    } while (x < threshold);
    return x % bound;
  }
  // next_below with a precomputed divisor (FastDiv): same draws, same results
  template <class Div>
  __device__ __host__ uint64_t next_below(const Div& d) {
    uint64_t x;
    do {
      x = next_u64();
    } while (x < d.thr);
    return d.mod(x);
  }
  __device__ __host__ double next_unit_open() {
    return ((double)(next_u64() >> 11) + 0.5) * 0x1.0p-53;
  }
};

}  // namespace bnmc_dev
