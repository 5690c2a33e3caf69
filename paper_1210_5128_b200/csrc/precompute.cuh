// K1 — local-score precompute (sm_100a): ScoreCache::build on the device.
//
// Replaces ScoreCache::build -> count_statistics -> local_score_from_counts
// (scoring.cpp:162-192, 82-135). Counting is done on sample BITPLANES: for
// every variable i and state x, bit t of plane (i,x) is set iff row t has
// state x in column i. The count of a joint configuration is then the
// popcount of the AND of the member planes — integer-exact, no atomics on the
// sample stream, every count bit-identical to the reference's CountTable.
//
// Work is organised by joint sets U (|U| <= s+1): the joint histogram of U
// serves all |U| entries (v, U - v), v in U, because N_ijk of (v, pi) is the
// joint count over pi + {v}. A CTA owns one "prefix" P (any set |P| <= s); its
// U's are P + {u} for every u > max(P), so the AND-planes of P's
// configurations are built once in shared memory and reused for every
// extension u; only states x < card(u)-1 are popcounted, the last state is
// the prefix count minus the others.
//
// The score of an entry follows local_score_from_counts exactly: configs of
// pi ascending (mixed radix, lowest parent least significant, scoring.cpp:
// 99-105), empty configs skipped (scoring.hpp:55-67), per config
// inner = sum_{c>0} (lG(c + a_cell) - lG(a_cell)) in state order, then
// score += (lG(a_row) - lG(a_row + N_ik)) + inner, starting from
// |pi| * log10(gamma). lG values come from a host-built glibc-lgamma LUT
// per distinct (r_i, card) pair (log10_gamma, scoring.hpp:16-18), so the fp64
// adds reproduce the reference bits (the TU is built with -fmad=false).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <set>
#include <vector>

#include "common.cuh"
#include "host_util.hpp"

namespace bnmc_dev {

constexpr int kHMax = 4096;   // max joint cells of a set U (dense counter bound)
constexpr int kRPMax = 1024;  // max configurations of a prefix P
#ifndef BNMC_K1_THREADS
#define BNMC_K1_THREADS 256
#endif
constexpr int kK1Threads = BNMC_K1_THREADS;
constexpr int kMaxPrefix = 8;  // members of a prefix P (|P| <= s <= 8)

struct K1Args {
  const uint32_t* __restrict__ bits;  // bitplanes
  const uint32_t* __restrict__ boff;  // [n] word offset of plane (i, 0); plane x at +x*W
  const int* __restrict__ cards;      // [n]
  int n, s, W;
  uint32_t last_mask;                 // valid bits of the last word
  int cmax;                           // max cardinality
  const uint64_t* __restrict__ pair_keys;  // sorted r*512 + card
  int n_pairs;
  const double* __restrict__ lut;     // [pair][2*(m+1)]: lG(c + a_cell), then lG(a_row + N)
  uint64_t lut_stride;                // 2*(m+1)
  uint64_t m;
  double log10_gamma;
  double* ls;                          // [n][S]
  uint64_t S;
  int row_begin, row_end;
  int rp_dense;                        // prefixes with more configurations go to K1W
  int WT, EG;
  int* error;
};

// Subset of {0..c-1} at global index j in the (size desc, lexicographic) order.
__device__ __forceinline__ uint64_t unrank_global(uint64_t j, int c, int s, int* size_out) {
  int k = s < c ? s : c;
  for (; k >= 0; --k) {
    const uint64_t block = binom(c, k);
    if (j < block) break;
    j -= block;
  }
  uint64_t mask = 0;
  int x = 0;
  for (int i = 0; i < k; ++i) {
    for (;;) {
      const uint64_t cnt = binom(c - x - 1, k - i - 1);
      if (j < cnt) {
        mask |= 1ull << x;
        ++x;
        break;
      }
      j -= cnt;
      ++x;
    }
  }
  *size_out = k;
  return mask;
}

// global_index (combinatorics.cpp:61-76)
__device__ __forceinline__ uint64_t global_index_dev(uint64_t mask, int c, int s) {
  const int k = __popcll(mask);
  uint64_t offset = 0;
  for (int j = k + 1; j <= s; ++j) offset += binom(c, j);
  uint64_t rank = 0;
  int prev = 0, pos = 1;
  for (uint64_t m = mask; m != 0; m &= m - 1, ++pos) {
    const int a = __ffsll((long long)m);  // 1-based element
    rank += binom(c - prev, k - pos + 1) - binom(c - a + 1, k - pos + 1);
    prev = a;
  }
  return offset + rank;
}

__device__ __forceinline__ int find_pair(const K1Args& a, uint64_t key) {
  int lo = 0, hi = a.n_pairs - 1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const uint64_t k = a.pair_keys[mid];
    if (k == key) return mid;
    if (k < key) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

template <bool TILED>
__global__ void __launch_bounds__(kK1Threads) k1_kernel(K1Args a, uint64_t prefix_base) {
  extern __shared__ uint32_t smem[];
  __shared__ int s_p[9];
  __shared__ int s_rad[10];
  __shared__ int s_k, s_rP, s_ext0;
  __shared__ double s_term[kK1Threads];  // per-warp scoring terms
  const int tid = threadIdx.x;
  const int n = a.n, W = a.W;
  if (tid == 0) {
    int k;
    const uint64_t P = unrank_global(prefix_base + blockIdx.x, n, a.s, &k);
    int i = 0;
    uint64_t r = 1;  // saturates: wide prefixes (r > rp_dense) leave below
    for (uint64_t m = P; m; m &= m - 1) {
      s_p[i] = __ffsll((long long)m) - 1;
      s_rad[i] = (int)min(r, (uint64_t)0x7fffffff);
      r = min(r * (uint64_t)a.cards[s_p[i]], (uint64_t)1 << 40);
      ++i;
    }
    s_rad[i] = (int)min(r, (uint64_t)0x7fffffff);
    s_k = k;
    s_rP = (int)min(r, (uint64_t)0x7fffffff);
    s_ext0 = k ? s_p[k - 1] + 1 : 0;
  }
  __syncthreads();
  const int k = s_k, rP = s_rP, ext0 = s_ext0;
  const int n_ext = n - ext0;
  if (n_ext <= 0) return;
  // Skip prefixes none of whose entries fall in this shard's row range.
  bool any = ext0 < a.row_end && n > a.row_begin;
  for (int i = 0; i < k; ++i) any |= (s_p[i] >= a.row_begin && s_p[i] < a.row_end);
  if (!any) return;
  if (rP > a.rp_dense) return;  // wide prefix: its joint sets are counted by K1W
  const int cmax = a.cmax;
  const int WT = TILED ? a.WT : 0;             // AND-plane tiles in smem, or formed on the fly
  const int WTP = WT | 1;                      // odd row stride: lanes over cfgs hit distinct banks
  uint32_t* NP = smem;                         // [rP]
  uint32_t* CNT = NP + rP;                     // [EG][rP][cmax]
  uint32_t* PB = CNT + (size_t)a.EG * rP * cmax;  // [rP][WTP] (tiled mode)
  uint32_t* PO = PB + (size_t)rP * WTP;        // [rP][kMaxPrefix] member plane offsets (tiled)
  const int warp = tid >> 5, lane = tid & 31;
  const int nx = cmax - 1;
  const int ncg = (rP + 31) / 32;

  // Member plane rows of configuration cfg of P (mixed radix, lowest member
  // least significant, scoring.cpp:99-105).
  auto member_rows = [&](int cfg, const uint32_t** mp) {
    int rem = cfg < rP ? cfg : 0;
#pragma unroll
    for (int i = 0; i < kMaxPrefix; ++i) {
      if (i < k) {
        const int ci = a.cards[s_p[i]];
        mp[i] = a.bits + a.boff[s_p[i]] + (uint32_t)(rem % ci) * W;
        rem /= ci;
      } else {
        mp[i] = nullptr;
      }
    }
  };

  if constexpr (TILED) {
    for (int cfg = tid; cfg < rP; cfg += kK1Threads) {
      const uint32_t* mp[kMaxPrefix];
      member_rows(cfg, mp);
      for (int i = 0; i < k; ++i) PO[cfg * kMaxPrefix + i] = (uint32_t)(mp[i] - a.bits);
    }
  }

  for (int e0 = 0; e0 < n_ext; e0 += a.EG) {
    const int ne = min(a.EG, n_ext - e0);
    for (int i = tid; i < ne * rP * cmax; i += kK1Threads) CNT[i] = 0;
    if (e0 == 0)
      for (int i = tid; i < rP; i += kK1Threads) NP[i] = 0;
    __syncthreads();
    // Counting as a popcount "product": a lane owns one configuration of P,
    // a warp unit owns 32 configurations x 4 (extension, state) planes read as
    // warp-broadcast loads; every output belongs to one lane (no atomics). The
    // configuration's AND-plane comes from a shared-memory tile (tiled mode)
    // or is formed word by word from its member planes (WT == 0; few distinct
    // addresses per warp load). The last state of u comes by difference below.
    const int nex = ne * nx;
    const int units = ncg * ((nex + 3) / 4) + (e0 == 0 ? ncg : 0);
    const int tile = WT > 0 ? WT : W;
    for (int w0 = 0; w0 < W; w0 += tile) {
      const int wt = min(tile, W - w0);
      if constexpr (TILED) {
        for (int idx = tid; idx < rP * wt; idx += kK1Threads) {
          const int cfg = idx / wt, w = idx - cfg * wt;
          uint32_t word = (w0 + w == W - 1) ? a.last_mask : 0xFFFFFFFFu;
          for (int i = 0; i < k; ++i) word &= __ldg(a.bits + PO[cfg * kMaxPrefix + i] + w0 + w);
          PB[cfg * WTP + w] = word;
        }
        __syncthreads();
      }
      for (int un = warp; un < units; un += kK1Threads / 32) {
        const int cg = un % ncg, blk = un / ncg;
        const int cfg = cg * 32 + lane;
        const uint32_t* mp[kMaxPrefix];
        if constexpr (!TILED) member_rows(cfg, mp);
        const uint32_t* pb = PB + (cfg < rP ? cfg : 0) * WTP;
        auto plane_word = [&](int w) -> uint32_t {
          if constexpr (TILED) return pb[w];
          uint32_t pw = w0 + w == W - 1 ? a.last_mask : 0xFFFFFFFFu;
#pragma unroll
          for (int i = 0; i < kMaxPrefix; ++i)
            if (i < k) pw &= __ldg(mp[i] + w0 + w);
          return pw;
        };
        if (blk * 4 >= nex) {  // prefix counts (first extension group only)
          uint32_t acc = 0;
          for (int w = 0; w < wt; ++w) acc += __popc(plane_word(w));
          if (cfg < rP) NP[cfg] += acc;
          continue;
        }
        const uint32_t* bp[4];
        int slot[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int ex = blk * 4 + q;
          const int e = ex / nx, x = ex - e * nx;
          const int u = ext0 + e0 + (e < ne ? e : 0);
          const bool ok = ex < nex && x < a.cards[u] - 1;
          slot[q] = ok ? (e * rP + cfg) * cmax + x : -1;
          bp[q] = a.bits + a.boff[u] + (uint32_t)(ok ? x : 0) * W + w0;
        }
        uint32_t acc[4] = {0, 0, 0, 0};
        for (int w = 0; w < wt; ++w) {
          const uint32_t pw = plane_word(w);
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[q] += __popc(pw & __ldg(bp[q] + w));
        }
        if (cfg < rP) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (slot[q] >= 0) CNT[slot[q]] += acc[q];
        }
      }
      __syncthreads();
    }
    // Last state of u by difference with the prefix count.
    for (int idx = tid; idx < ne * rP; idx += kK1Threads) {
      const int e = idx / rP, cfg = idx - e * rP;
      const int cu = a.cards[ext0 + e0 + e];
      uint32_t* c = CNT + (e * rP + cfg) * cmax;
      uint32_t sum = 0;
      for (int x = 0; x < cu - 1; ++x) sum += c[x];
      c[cu - 1] = NP[cfg] - sum;
    }
    __syncthreads();
    // Score the |U| entries (v, U - v) of every U = P + {u}: one warp per
    // entry, lanes over the configurations of pi (their terms are
    // independent), then lane 0 folds the terms in configuration order — the
    // reference's serial summation (scoring.cpp:111-135) bit for bit, with
    // the gathers of 32 configurations in flight instead of one.
    for (int idx = warp; idx < ne * (k + 1); idx += kK1Threads / 32) {
      const int e = idx / (k + 1), d = idx - e * (k + 1);
      const int u = ext0 + e0 + e;
      const int v = d < k ? s_p[d] : u;
      if (v < a.row_begin || v >= a.row_end) continue;
      const int cu = a.cards[u];
      const int cv = a.cards[v];
      uint64_t pmask = 1ull << u;
      for (int i = 0; i < k; ++i) pmask |= 1ull << s_p[i];
      pmask &= ~(1ull << v);
      const uint64_t r_pi = (uint64_t)rP * cu / cv;
      const int pair = find_pair(a, r_pi * 512 + cv);
      if (pair < 0) {
        if (lane == 0) atomicExch(a.error, 2);
        continue;
      }
      const double* lgc = a.lut + (uint64_t)pair * a.lut_stride;
      const double* lgr = lgc + a.m + 1;
      const double lg_cell = lgc[0], lg_row = lgr[0];
      double score = (double)k * a.log10_gamma;  // |pi| = k, int * double first
      const uint32_t* H = CNT + e * rP * cmax;    // H[cfgP * cmax + x_u]
      // child = u: configs of pi = P, H[cfg * cmax + x]; child = p_d: configs
      // of pi = (P - p_d) + {u}, k' = low + R*(mid + Q*x_u), H[(low + R*(y +
      // cd*mid)) * cmax + x_u]
      const int R = d < k ? s_rad[d] : 1, Q = d < k ? rP / (R * cv) : 1;
      const int rpi = (int)r_pi;
      double* term = s_term + warp * 32;
      for (int c0 = 0; c0 < rpi; c0 += 32) {
        const int kk = c0 + lane;
        uint32_t n_ik = 0;
        double inner = 0.0;
        if (kk < rpi) {
          int base, stride;
          if (d == k) {
            base = kk * cmax;
            stride = 1;
          } else {
            const int low = kk % R, rest = kk / R;
            const int mid = rest % Q, xu = rest / Q;
            base = (low + R * cv * mid) * cmax + xu;
            stride = R * cmax;
          }
          for (int y = 0; y < cv; ++y) {
            const uint32_t c = H[base + y * stride];
            if (c > 0) {
              inner += lgc[c] - lg_cell;
              n_ik += c;
            }
          }
          if (n_ik > 0) term[lane] = lg_row - lgr[n_ik] + inner;
        }
        const unsigned has = __ballot_sync(0xffffffffu, n_ik > 0);
        __syncwarp();
        if (lane == 0) {
          const int cnt = min(32, rpi - c0);
          if (has == (cnt == 32 ? 0xffffffffu : (1u << cnt) - 1u)) {
            // every configuration of the chunk is non-empty (the common case):
            // loads batched ahead of the serial add chain
#pragma unroll 8
            for (int j = 0; j < cnt; ++j) score += term[j];
          } else {
            for (unsigned b = has; b; b &= b - 1) score += term[__ffs(b) - 1];
          }
        }
        __syncwarp();
      }
      if (lane != 0) continue;
      const uint64_t g = global_index_dev(nodes_to_cand(pmask, v), n - 1, a.s);
      a.ls[(uint64_t)v * a.S + g] = score;
    }
    __syncthreads();
  }
}

// Bitplanes from row-major cells: one thread per (variable, word).
__global__ void bitplane_kernel(const uint8_t* __restrict__ cells, const int* __restrict__ cards,
                                const uint32_t* __restrict__ boff, uint32_t* bits, int n,
                                uint64_t m, int W) {
  const int i = blockIdx.y;
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= W) return;
  const int ci = cards[i];
  uint8_t st[32];
  const uint64_t t0 = (uint64_t)w * 32;
  const int nb = (int)(m - t0 < 32 ? m - t0 : 32);
  for (int b = 0; b < 32; ++b) st[b] = b < nb ? cells[(t0 + b) * n + i] : 0xFF;
  for (int x = 0; x < ci; ++x) {
    uint32_t word = 0;
    for (int b = 0; b < nb; ++b) word |= (uint32_t)(st[b] == x) << b;
    bits[boff[i] + (uint32_t)x * W + w] = word;
  }
}

// count_statistics for explicit (node, pset) entries: cell (cfg, x) counted
// as popcount(AND of parent planes & child plane x) over all words.
__global__ void counts_kernel(const uint32_t* __restrict__ bits, const uint32_t* __restrict__ boff,
                              const int* __restrict__ cards, int W, uint32_t last_mask,
                              const int* __restrict__ nodes, const uint64_t* __restrict__ psets,
                              const uint64_t* __restrict__ offsets, uint32_t* out) {
  const int e = blockIdx.x;
  const int v = nodes[e];
  const uint64_t ps = psets[e];
  int par[64], np = 0;
  uint64_t r = 1;
  for (uint64_t m = ps; m; m &= m - 1) {
    par[np] = __ffsll((long long)m) - 1;
    r *= (uint64_t)cards[par[np]];
    ++np;
  }
  const int cv = cards[v];
  for (uint64_t cell = threadIdx.x; cell < r * cv; cell += blockDim.x) {
    const uint64_t cfg = cell / cv;
    const int x = (int)(cell - cfg * cv);
    uint32_t total = 0;
    for (int w = 0; w < W; ++w) {
      uint32_t word = (w == W - 1) ? last_mask : 0xFFFFFFFFu;
      uint64_t rem = cfg;
      for (int j = 0; j < np; ++j) {
        const int cj = cards[par[j]];
        word &= bits[boff[par[j]] + (uint32_t)(rem % cj) * W + w];
        rem /= cj;
      }
      word &= bits[boff[v] + (uint32_t)x * W + w];
      total += __popc(word);
    }
    out[offsets[e] + cell] = total;
  }
}

}  // namespace bnmc_dev

#include "precompute_wide.cuh"

namespace bnmc_host {

struct Bitplanes {
  uint32_t* bits = nullptr;
  uint32_t* boff = nullptr;
  int* cards = nullptr;
  int W = 0;
  uint32_t last_mask = 0;
  ~Bitplanes() {
    if (bits) cudaFree(bits);
    if (boff) cudaFree(boff);
    if (cards) cudaFree(cards);
  }
};

inline void make_bitplanes(Bitplanes& bp, const uint8_t* cells, const int* cards, uint64_t m,
                           int n, cudaStream_t stream) {
  bp.W = static_cast<int>((m + 31) / 32);
  const int rem = static_cast<int>(m % 32);
  bp.last_mask = rem ? ((1u << rem) - 1u) : 0xFFFFFFFFu;
  std::vector<uint32_t> boff(n);
  uint64_t words = 0;
  for (int i = 0; i < n; ++i) {
    boff[i] = static_cast<uint32_t>(words);
    words += static_cast<uint64_t>(cards[i]) * bp.W;
  }
  if (words > 0xFFFFFFFFull) raise(BNMC_CAPACITY, "sample bitplanes exceed 2^32 words");
  CK(cudaMalloc(&bp.bits, std::max<uint64_t>(words, 1) * 4));
  CK(cudaMalloc(&bp.boff, sizeof(uint32_t) * n));
  CK(cudaMalloc(&bp.cards, sizeof(int) * n));
  CK(cudaMemcpyAsync(bp.boff, boff.data(), sizeof(uint32_t) * n, cudaMemcpyHostToDevice, stream));
  CK(cudaMemcpyAsync(bp.cards, cards, sizeof(int) * n, cudaMemcpyHostToDevice, stream));
  if (m > 0) {
    uint8_t* d_cells = nullptr;
    CK(cudaMalloc(&d_cells, m * n));
    CK(cudaMemcpyAsync(d_cells, cells, m * n, cudaMemcpyHostToDevice, stream));
    bnmc_dev::bitplane_kernel<<<dim3((bp.W + 127) / 128, n), 128, 0, stream>>>(
        d_cells, bp.cards, bp.boff, bp.bits, n, m, bp.W);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(stream));
    cudaFree(d_cells);
  }
}

// Distinct parent-configuration counts r = product of <= s cardinalities
// (bounded by the dense limit), by recursion over distinct card values.
inline void products(const std::vector<std::pair<int, int>>& cm, size_t i, int left, uint64_t r,
                     std::set<uint64_t>& out) {
  out.insert(r);
  if (left == 0) return;
  for (size_t j = i; j < cm.size(); ++j) {
    uint64_t rr = r;
    for (int e = 1; e <= std::min(left, cm[j].second); ++e) {
      rr *= static_cast<uint64_t>(cm[j].first);
      if (rr > static_cast<uint64_t>(bnmc_dev::kHMax)) break;
      products(cm, j + 1, left - e, rr, out);
    }
  }
}

// ---------------------------------------------------------------- prefixes
// K1 works per prefix P (|P| <= s) in the global-index order of subsets of
// {0..n-1}: sizes min(s,n)..0, lexicographic within a size (the order
// unrank_global follows). A part of a multi-GPU build owns a contiguous range
// of prefix indices; every entry (v, pi) belongs to exactly one prefix
// (P = pi + {v} minus its largest member), so parts write disjoint entries.

inline uint64_t prefix_total(int n, int s) {
  uint64_t t = 0;
  for (int j = 0; j <= std::min(s, n); ++j) {
    uint64_t c = 1;
    for (int i = 0; i < j; ++i) c = c * (n - i) / (i + 1);
    t += c;
  }
  return t;
}

inline uint64_t host_choose(int n, int k) {
  if (k < 0 || k > n) return 0;
  uint64_t c = 1;
  for (int i = 0; i < k; ++i) c = c * (n - i) / (i + 1);
  return c;
}

// Iterator over prefixes in global-index order from index lo.
struct PrefixWalk {
  int n, s, k;
  int a[bnmc_dev::kMaxPrefix + 1];
  bool done = false;
  PrefixWalk(int n_, int s_, uint64_t lo) : n(n_), s(s_) {
    k = std::min(s, n);
    uint64_t j = lo;
    while (k >= 0 && j >= host_choose(n, k)) {
      j -= host_choose(n, k);
      --k;
    }
    if (k < 0) {
      done = true;
      return;
    }
    int x = 0;
    for (int i = 0; i < k; ++i)
      for (;; ++x) {
        const uint64_t cnt = host_choose(n - x - 1, k - i - 1);
        if (j < cnt) {
          a[i] = x++;
          break;
        }
        j -= cnt;
      }
  }
  void next() {
    for (int i = k - 1; i >= 0; --i)
      if (a[i] < n - k + i) {
        ++a[i];
        for (int j = i + 1; j < k; ++j) a[j] = a[j - 1] + 1;
        return;
      }
    if (--k < 0) {
      done = true;
      return;
    }
    for (int i = 0; i < k; ++i) a[i] = i;
  }
};

// Configurations of a prefix, saturated at 2^62 (only compared with rp_dense).
inline uint64_t prefix_configs(const PrefixWalk& w, const int* cards) {
  const uint64_t cap = uint64_t(1) << 62;
  uint64_t r = 1;
  for (int i = 0; i < w.k; ++i) {
    const uint64_t c = static_cast<uint64_t>(cards[w.a[i]]);
    r = r > cap / c ? cap : r * c;
  }
  return r;
}

// Largest prefix configuration count the dense K1 counter holds: the joint
// histogram of U = P + {u} is r_P * card(u) <= kHMax cells, r_P <= kRPMax.
inline int dense_prefix_limit(const int* cards, int n) {
  const int cmax = *std::max_element(cards, cards + n);
  return std::min(bnmc_dev::kRPMax, bnmc_dev::kHMax / cmax);
}

// Work-balanced split of the prefix range into `parts` contiguous pieces
// (cut[0] = 0, cut[parts] = total). Dense prefix weight ~ word-ANDs of the
// popcount product (r_P x extension states x words) + its scoring cells; wide
// prefix weight ~ keys sorted and walked.
inline std::vector<uint64_t> k1_partition(const int* cards, int n, int s, uint64_t m, int parts) {
  const uint64_t total = prefix_total(n, s);
  std::vector<uint64_t> cut(parts + 1, total);
  cut[0] = 0;
  if (parts <= 1) return cut;
  const int rpd = dense_prefix_limit(cards, n);
  const double W = static_cast<double>((m + 31) / 32);
  std::vector<double> suf_c(n + 1, 0.0), suf_c1(n + 1, 0.0);
  for (int u = n - 1; u >= 0; --u) {
    suf_c[u] = suf_c[u + 1] + cards[u];
    suf_c1[u] = suf_c1[u + 1] + (cards[u] - 1);
  }
  std::vector<double> wt;
  wt.reserve(total);
  double sum = 0.0;
  for (PrefixWalk w(n, s, 0); !w.done; w.next()) {
    const int ext0 = w.k ? w.a[w.k - 1] + 1 : 0;
    double x = 64.0;  // per-CTA overhead
    if (ext0 < n) {
      const uint64_t r = prefix_configs(w, cards);
      if (r <= static_cast<uint64_t>(rpd))
        x += r * ((suf_c1[ext0] + 1.0) * (W + 2.0) + 4.0 * (w.k + 1) * suf_c[ext0]);
      else
        x += 24.0 * (n - ext0) * (w.k + 1) * static_cast<double>(m + 1);
    }
    wt.push_back(x);
    sum += x;
  }
  double acc = 0.0;
  int g = 1;
  for (uint64_t i = 0; i < total && g < parts; ++i) {
    acc += wt[i];
    while (g < parts && acc >= sum * g / parts) cut[g++] = i + 1;
  }
  return cut;
}

struct K1Range {
  uint64_t p_lo = 0, p_hi = ~uint64_t(0);  // prefix indices [p_lo, p_hi)
  int row_begin = 0, row_end = 64;         // only entries of these node rows
};

struct K1Report {
  float ms = 0.f;          // K1 (dense) + K1W (wide) device time
  uint64_t wide_entries = 0;
};

inline void precompute(cudaStream_t stream, double* d_ls, uint64_t S, const uint8_t* cells,
                       const int* cards, uint64_t m, int n, int s, double gamma, double ess,
                       int alpha, const K1Range& range, K1Report* rep) {
  using namespace bnmc_dev;
  const uint64_t total = prefix_total(n, s);
  const uint64_t p_lo = std::min(range.p_lo, total), p_hi = std::min(range.p_hi, total);
  const int row_begin = range.row_begin, row_end = std::min(range.row_end, n);
  // Dense prefixes: r_P <= rpd (joint histograms of <= kHMax cells). Larger
  // prefixes (if any) are counted by K1W.
  std::vector<int> sorted(cards, cards + n);
  std::sort(sorted.rbegin(), sorted.rend());
  const int rpd = dense_prefix_limit(cards, n);
  uint64_t hp = 1;  // largest prefix configuration count (saturated)
  for (int i = 0; i < std::min(n, s); ++i)
    hp = hp > (1ull << 40) / sorted[i] ? (1ull << 40) : hp * sorted[i];
  const bool any_wide = hp > static_cast<uint64_t>(rpd);
  const int cmax = sorted[0];

  Bitplanes bp;
  make_bitplanes(bp, cells, cards, m, n, stream);

  // LUT pairs (r, card) and glibc lgamma values (log10_gamma, scoring.hpp:16-18).
  std::vector<std::pair<int, int>> cm;
  for (int i = 0; i < n;) {
    int j = i;
    while (j < n && sorted[j] == sorted[i]) ++j;
    cm.push_back({sorted[i], j - i});
    i = j;
  }
  std::set<uint64_t> prods;
  products(cm, 0, s, 1, prods);
  std::vector<uint64_t> keys;
  for (uint64_t r : prods)
    for (auto& c : cm)
      if (r * c.first <= static_cast<uint64_t>(kHMax)) keys.push_back(r * 512 + c.first);
  std::sort(keys.begin(), keys.end());
  const uint64_t stride = 2 * (m + 1);
  if (keys.size() * stride * 8 > (uint64_t(2) << 30))
    raise(BNMC_CAPACITY, "lgamma lookup tables would exceed 2 GiB");
  std::vector<double> lut(keys.size() * stride);
  const double K = 0.43429448190325182765;  // 1/ln(10), scoring.hpp:17
  for (size_t p = 0; p < keys.size(); ++p) {
    const uint64_t r = keys[p] / 512;
    const int card = static_cast<int>(keys[p] % 512);
    // Hyperparams::alpha_cell (scoring.hpp:27-31); a_row (scoring.cpp:116)
    const double a_cell = alpha == BNMC_ALPHA_BDEU ? ess / (static_cast<double>(r) * card) : 1.0;
    if (!(a_cell > 0.0)) raise(BNMC_USAGE, "Dirichlet hyperparameter must be positive");
    const double a_row = a_cell * card;
    double* o = lut.data() + p * stride;
    for (uint64_t c = 0; c <= m; ++c) {
      const uint32_t cc = static_cast<uint32_t>(c);
      o[c] = std::lgamma(cc + a_cell) * K;
      o[m + 1 + c] = std::lgamma(a_row + cc) * K;
    }
  }
  uint64_t* d_keys = nullptr;
  double* d_lut = nullptr;
  int* d_err = nullptr;
  CK(cudaMalloc(&d_keys, std::max<size_t>(1, keys.size()) * 8));
  CK(cudaMalloc(&d_lut, std::max<size_t>(1, lut.size()) * 8));
  CK(cudaMalloc(&d_err, sizeof(int)));
  CK(cudaMemcpyAsync(d_keys, keys.data(), keys.size() * 8, cudaMemcpyHostToDevice, stream));
  CK(cudaMemcpyAsync(d_lut, lut.data(), lut.size() * 8, cudaMemcpyHostToDevice, stream));
  CK(cudaMemsetAsync(d_err, 0, sizeof(int), stream));

  K1Args a{};
  a.bits = bp.bits;
  a.boff = bp.boff;
  a.cards = bp.cards;
  a.n = n;
  a.s = s;
  a.W = bp.W;
  a.last_mask = bp.last_mask;
  a.cmax = cmax;
  a.pair_keys = d_keys;
  a.n_pairs = static_cast<int>(keys.size());
  a.lut = d_lut;
  a.lut_stride = stride;
  a.m = m;
  a.log10_gamma = std::log10(gamma);
  a.ls = d_ls;
  a.S = S;
  a.row_begin = row_begin;
  a.row_end = row_end;
  a.rp_dense = rpd;
  // Shared memory, sized for several CTAs per SM so one CTA's scoring phase
  // overlaps other CTAs' counting: prefix counts + CNT for a group of
  // extensions (+ an AND-plane word tile in tiled mode). Tiled mode re-forms
  // the tile once per extension group, so it is used when one group covers
  // a typical prefix's extensions; otherwise AND-planes are formed on the fly.
  const char* kb = std::getenv("BNMC_K1_SMEM_KB");
  const size_t budget = (kb ? std::strtoul(kb, nullptr, 10) : 48) * 1024;
  const int rPmax = static_cast<int>(std::min<uint64_t>(hp, rpd));
  const size_t np_bytes = 4ull * rPmax;
  const int wt_fit = static_cast<int>((budget / 2) / (4ull * rPmax)) - 1;
  int wt = std::max(1, std::min(std::max(bp.W, 1), std::max(32, wt_fit)));
  size_t pb_bytes = 4ull * rPmax * (wt | 1);
  size_t left = budget > pb_bytes + np_bytes ? budget - pb_bytes - np_bytes : 0;
  int eg = static_cast<int>(left / (4ull * rPmax * cmax));
  const char* mode = std::getenv("BNMC_K1_MODE");  // "tiled" / "fly" (development)
  const bool tiled = mode ? std::strcmp(mode, "tiled") == 0 : eg >= std::min(n, 16);
  if (!tiled) {
    wt = 0;
    pb_bytes = 0;
    left = budget > np_bytes ? budget - np_bytes : 0;
    eg = static_cast<int>(left / (4ull * rPmax * cmax));
  }
  a.WT = wt;
  a.EG = std::max(1, std::min(n, eg));
  const size_t cnt_bytes = 4ull * a.EG * rPmax * cmax + np_bytes + pb_bytes +
                           (tiled ? 4ull * rPmax * kMaxPrefix : 0);
  a.error = d_err;
  const size_t shm = cnt_bytes;
  CK(cudaFuncSetAttribute(k1_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          static_cast<int>(shm)));
  CK(cudaFuncSetAttribute(k1_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          static_cast<int>(shm)));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, stream));
  const uint64_t chunk = 1u << 30;
  for (uint64_t base = p_lo; base < p_hi; base += chunk) {
    const unsigned blocks = static_cast<unsigned>(std::min(chunk, p_hi - base));
    if (tiled)
      k1_kernel<true><<<blocks, kK1Threads, shm, stream>>>(a, base);
    else
      k1_kernel<false><<<blocks, kK1Threads, shm, stream>>>(a, base);
    CK(cudaGetLastError());
  }
  CK(cudaEventRecord(e1, stream));
  CK(cudaEventSynchronize(e1));
  float dense_ms = 0.f;
  CK(cudaEventElapsedTime(&dense_ms, e0, e1));
  int err = 0;
  CK(cudaMemcpy(&err, d_err, sizeof(int), cudaMemcpyDeviceToHost));
  cudaFree(d_keys);
  cudaFree(d_lut);
  cudaFree(d_err);
  if (err) raise(BNMC_ERR, "precompute kernel reported internal error " + std::to_string(err));

  // K1W: the entries of wide prefixes (r_P > rpd) in this range.
  float wide_ms = 0.f;
  uint64_t wide_entries = 0;
  if (any_wide && p_lo < p_hi) {
    CK(cudaEventRecord(e0, stream));
    WideScorer ws(stream, cells, cards, bp.cards, m, n, s, gamma, ess, alpha, d_ls, S);
    uint64_t idx = p_lo;
    for (PrefixWalk w(n, s, p_lo); !w.done && idx < p_hi; w.next(), ++idx) {
      const int ext0 = w.k ? w.a[w.k - 1] + 1 : 0;
      if (ext0 >= n || prefix_configs(w, cards) <= static_cast<uint64_t>(rpd)) continue;
      uint64_t pm = 0;
      for (int i = 0; i < w.k; ++i) pm |= 1ull << w.a[i];
      for (int u = ext0; u < n; ++u) {
        const uint64_t U = pm | (1ull << u);
        for (uint64_t vm = U; vm; vm &= vm - 1) {
          const int v = __builtin_ctzll(vm);
          if (v < row_begin || v >= row_end) continue;
          const uint64_t pi = U & ~(1ull << v);
          uint64_t r = 1;
          for (uint64_t q = pi; q; q &= q - 1) {
            const uint64_t c = static_cast<uint64_t>(cards[__builtin_ctzll(q)]);
            if (r > ~0ull / c) raise(BNMC_CAPACITY, "parent configuration space overflows 64 bits");
            r *= c;
          }
          ws.add(WideEntry{v, pi, r});
        }
      }
    }
    ws.flush();
    wide_entries = ws.entries();
    CK(cudaEventRecord(e1, stream));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&wide_ms, e0, e1));
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (rep) {
    rep->ms = dense_ms + wide_ms;
    rep->wide_entries = wide_entries;
  }
}

inline void count_statistics_device(const uint8_t* cells, const int* cards, uint64_t m, int n,
                                    int count, const int* nodes, const uint64_t* psets,
                                    const uint64_t* offsets, uint32_t* out, uint64_t* configs_out) {
  if (n < 1 || n > 64) raise(BNMC_DATA, "dataset must have between 1 and 64 variables");
  uint64_t total = 0;
  for (int e = 0; e < count; ++e) {
    if (nodes[e] < 0 || nodes[e] >= n) raise(BNMC_USAGE, "node out of range");
    if ((psets[e] >> nodes[e]) & 1u) raise(BNMC_DATA, "node cannot appear in its own parent set");
    if (n < 64 && (psets[e] >> n)) raise(BNMC_USAGE, "parent out of range");
    uint64_t r = 1;
    for (uint64_t mm = psets[e]; mm; mm &= mm - 1) {
      const uint64_t c = static_cast<uint64_t>(cards[__builtin_ctzll(mm)]);
      if (r > ~0ull / c) raise(BNMC_CAPACITY, "parent configuration space overflows 64 bits");
      r *= c;
    }
    if (r * cards[nodes[e]] > (1ull << 24)) raise(BNMC_CAPACITY, "count table too large");
    configs_out[e] = r;
    total = std::max<uint64_t>(total, offsets[e] + r * cards[nodes[e]]);
  }
  cudaStream_t stream;
  CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  {
    Bitplanes bp;
    make_bitplanes(bp, cells, cards, m, n, stream);
    int* d_nodes = nullptr;
    uint64_t *d_psets = nullptr, *d_off = nullptr;
    uint32_t* d_out = nullptr;
    CK(cudaMalloc(&d_nodes, sizeof(int) * count));
    CK(cudaMalloc(&d_psets, 8ull * count));
    CK(cudaMalloc(&d_off, 8ull * count));
    CK(cudaMalloc(&d_out, 4ull * std::max<uint64_t>(total, 1)));
    CK(cudaMemcpyAsync(d_nodes, nodes, sizeof(int) * count, cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(d_psets, psets, 8ull * count, cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(d_off, offsets, 8ull * count, cudaMemcpyHostToDevice, stream));
    if (bp.W == 0) {
      CK(cudaMemsetAsync(d_out, 0, 4ull * std::max<uint64_t>(total, 1), stream));
    } else {
      bnmc_dev::counts_kernel<<<count, 256, 0, stream>>>(bp.bits, bp.boff, bp.cards, bp.W,
                                                         bp.last_mask, d_nodes, d_psets, d_off,
                                                         d_out);
      CK(cudaGetLastError());
    }
    CK(cudaMemcpyAsync(out, d_out, 4ull * total, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    cudaFree(d_nodes);
    cudaFree(d_psets);
    cudaFree(d_off);
    cudaFree(d_out);
  }
  cudaStreamDestroy(stream);
}

// count_statistics as the reference's sparse CountTable (ordered map above
// 2^22 cells, scoring.cpp:53-80): the active configurations ascending with
// their card(node) counts, via the K1W key sort on the device. configs_out
// holds up to m entries, counts_out up to m * card(node).
inline void count_statistics_sparse_device(const uint8_t* cells, const int* cards, uint64_t m,
                                           int n, int node, uint64_t pset, uint64_t* configs_out,
                                           uint32_t* counts_out, uint64_t* n_active) {
  if (n < 1 || n > 64) raise(BNMC_DATA, "dataset must have between 1 and 64 variables");
  if (node < 0 || node >= n) raise(BNMC_USAGE, "node out of range");
  if ((pset >> node) & 1u) raise(BNMC_DATA, "node cannot appear in its own parent set");
  if (n < 64 && (pset >> n)) raise(BNMC_USAGE, "parent out of range");
  uint64_t r = 1;
  for (uint64_t mm = pset; mm; mm &= mm - 1) {
    const uint64_t c = static_cast<uint64_t>(cards[__builtin_ctzll(mm)]);
    if (r > ~0ull / c) raise(BNMC_CAPACITY, "parent configuration space overflows 64 bits");
    r *= c;
  }
  const int cv = cards[node];
  cudaStream_t stream;
  CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  int* d_cards = nullptr;
  try {
    CK(cudaMalloc(&d_cards, sizeof(int) * n));
    CK(cudaMemcpyAsync(d_cards, cards, sizeof(int) * n, cudaMemcpyHostToDevice, stream));
    std::vector<uint64_t> keys;
    std::vector<uint8_t> vals;
    bool comp = false;
    {
      WideScorer ws(stream, cells, cards, d_cards, m, n, 0, 0.1, 1.0, BNMC_ALPHA_K2, nullptr, 0);
      ws.sorted_segment(WideEntry{node, pset, r}, keys, vals, comp);
    }
    const uint64_t div = comp ? static_cast<uint64_t>(cv) : 1;
    uint64_t na = 0;
    for (uint64_t i = 0; i < m;) {
      const uint64_t cfg = keys[i] / div;
      configs_out[na] = cfg;
      uint32_t* row = counts_out + na * cv;
      std::fill(row, row + cv, 0u);
      for (; i < m && keys[i] / div == cfg; ++i) ++row[vals[i]];
      ++na;
    }
    *n_active = na;
  } catch (...) {
    cudaFree(d_cards);
    cudaStreamDestroy(stream);
    throw;
  }
  cudaFree(d_cards);
  cudaStreamDestroy(stream);
}

}  // namespace bnmc_host
