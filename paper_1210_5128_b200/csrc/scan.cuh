// K2 — order-scan kernel and K3 — chain step kernel (sm_100a).
//
// K2 replaces OrderScorer::scan_slice + argmax_reduce (engine.cpp:43-58,
// 15-22). One CTA owns a fixed slice of the global-index range; the
// candidate-position masks of that slice (identical for every row, SURVEY
// §8.1.1) are loaded ONCE per launch into registers and reused for every
// (chain, rescanned row) item of the iteration, so DRAM only streams the
// 4-byte fp32 keys (or 8-byte fp64 keys) of the rescanned rows.
//
// Exactness: the fp32 key of an entry is fl32(eff) with eff the reference's
// fp64 effective score lookup + PpfTable::sum (engine.cpp:50-51). Rounding is
// monotone, so the fp64 argmax lies among the entries whose key equals the
// fp32 max; those (rare) key ties are resolved on the exact fp64 value and then
// on the reference's enumeration order over predecessor POSITIONS (first
// maximum wins, engine.cpp:52). The comparator is therefore a
// strict total order and every reduction tree yields the reference's cell.
#pragma once

#include "common.cuh"

namespace bnmc_dev {

constexpr uint32_t kNoIdx = 0xFFFFFFFFu;

struct Item {          // one (chain, rescanned row) pair of an iteration
  uint64_t cpred;      // predecessor set of the row's node, as candidate positions
  uint32_t v;          // node (row)
  uint32_t pad;
};

template <typename K>
struct Partial {
  K k;
  uint32_t g;
};

struct TieCtx {
  const double* __restrict__ ls;     // fp64 local scores, row stride S
  const uint64_t* __restrict__ cmask;
  const double* __restrict__ w;      // PPF weights n x n
  uint64_t S;
  int n;
};

// Exact effective score of entry g of row v: lookup + PpfTable::sum.
__device__ __forceinline__ double exact_eff(const TieCtx& c, int v, uint32_t g) {
  const uint64_t cm = c.cmask[g];
  return c.ls[(uint64_t)v * c.S + g] + ppf_sum(c.w, c.n, v, cand_to_nodes(cm, v));
}

// True iff entry a precedes entry b in the reference enumeration over the
// predecessor positions of the order (sizes descending, then lexicographic on
// sorted positions; combinatorics.hpp:59-64, 83-101). ppos[node] = position.
__device__ __forceinline__ bool tie_prefer(const TieCtx& c, int v, uint32_t ga, uint32_t gb,
                                           const uint8_t* ppos) {
  const uint64_t ma = c.cmask[ga], mb = c.cmask[gb];
  const int sa = __popcll(ma), sb = __popcll(mb);
  if (sa != sb) return sa > sb;
  uint64_t pa = 0, pb = 0;
  for (uint64_t m = ma; m; m &= m - 1) pa |= 1ull << ppos[cand_node(__ffsll((long long)m) - 1, v)];
  for (uint64_t m = mb; m; m &= m - 1) pb |= 1ull << ppos[cand_node(__ffsll((long long)m) - 1, v)];
  const uint64_t d = pa ^ pb;
  return d != 0 && (pa & (d & (0 - d))) != 0;
}

// Strict "a beats b" under (key, exact fp64 eff, reference tie rule).
template <typename K>
__device__ __noinline__ bool better_slow(const TieCtx& c, int v, K ka, uint32_t ga, K kb,
                                         uint32_t gb, const uint8_t* ppos) {
  if (ga == gb) return false;
  if (sizeof(K) == 4) {
    const double ea = exact_eff(c, v, ga), eb = exact_eff(c, v, gb);
    if (ea != eb) return ea > eb;
  }
  return tie_prefer(c, v, ga, gb, ppos);
}

template <typename K>
__device__ __forceinline__ bool better(const TieCtx& c, int v, K ka, uint32_t ga, K kb,
                                       uint32_t gb, const uint8_t* ppos) {
  if (ga == kNoIdx) return false;
  if (gb == kNoIdx) return true;
  if (ka != kb) return ka > kb;
  return better_slow<K>(c, v, ka, ga, kb, gb, ppos);
}

template <typename K>
__device__ __forceinline__ void warp_argmax(const TieCtx& c, int v, K& k, uint32_t& g,
                                            const uint8_t* ppos) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const K ok = __shfl_down_sync(0xffffffffu, k, off);
    const uint32_t og = __shfl_down_sync(0xffffffffu, g, off);
    if (better<K>(c, v, ok, og, k, g, ppos)) {
      k = ok;
      g = og;
    }
  }
}

template <typename K> struct Vec4;
template <> struct Vec4<float> {
  using T = float4;
  static __device__ __forceinline__ void load(const float* p, float (&o)[4]) {
    const float4 x = __ldg(reinterpret_cast<const float4*>(p));
    o[0] = x.x; o[1] = x.y; o[2] = x.z; o[3] = x.w;
  }
};
template <> struct Vec4<double> {
  static __device__ __forceinline__ void load(const double* p, double (&o)[4]) {
    const double2 x = __ldg(reinterpret_cast<const double2*>(p));
    const double2 y = __ldg(reinterpret_cast<const double2*>(p) + 1);
    o[0] = x.x; o[1] = x.y; o[2] = y.x; o[3] = y.y;
  }
};

struct ScanArgs {
  const void* keys;      // n x Sp keys (float or double), padding = -inf
  uint64_t Sp;           // padded row stride (multiple of 32)
  const Item* items;     // [C][n]
  const int* counts;     // [C]
  const uint8_t* ppos;   // [C][64] positions of the proposed order
  void* partials;        // [C][n][G]
  int C, n, G;
  int units;             // Sp / 4
  int L4;                // units per CTA
  TieCtx tie;
};

constexpr int kScanMaxThreads = 512;

// K2: grid = G CTAs, block = T <= 512 threads; each thread owns U float4 units
// of its CTA's slice, masks held in registers across all items of the launch;
// IB items are streamed together so U*IB vector loads are in flight per thread.
template <typename K, int U, int IB>
__global__ void __launch_bounds__(kScanMaxThreads) scan_kernel(ScanArgs a) {
  constexpr int kItemBatch = IB;
  __shared__ K s_k[kItemBatch][32];
  __shared__ uint32_t s_g[kItemBatch][32];
  __shared__ int s_v[kItemBatch];
  const int T = blockDim.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = T >> 5;
  const int u0 = blockIdx.x * a.L4;
  const int u1 = min(u0 + a.L4, a.units);
  const uint64_t* cmask = a.tie.cmask;

  uint64_t mk[U][4];
  int uu[U];
#pragma unroll
  for (int i = 0; i < U; ++i) {
    uu[i] = u0 + threadIdx.x + i * T;
    if (uu[i] < u1) {
      const ulonglong2 x = __ldg(reinterpret_cast<const ulonglong2*>(cmask + 4ull * uu[i]));
      const ulonglong2 y = __ldg(reinterpret_cast<const ulonglong2*>(cmask + 4ull * uu[i]) + 1);
      mk[i][0] = x.x; mk[i][1] = x.y; mk[i][2] = y.x; mk[i][3] = y.y;
    } else {
      mk[i][0] = mk[i][1] = mk[i][2] = mk[i][3] = ~0ull;
      uu[i] = -1;
    }
  }
  const K* keys = static_cast<const K*>(a.keys);
  Partial<K>* parts = static_cast<Partial<K>*>(a.partials);

  for (int c = 0; c < a.C; ++c) {
    const int cnt = a.counts[c];
    const uint8_t* ppos = a.ppos + 64 * c;
    for (int s0 = 0; s0 < cnt; s0 += kItemBatch) {
      const int nb = min(kItemBatch, cnt - s0);
      K bk[kItemBatch];
      uint32_t bg[kItemBatch];
      Item it[kItemBatch];
#pragma unroll
      for (int j = 0; j < kItemBatch; ++j) {
        bk[j] = -INFINITY;
        bg[j] = kNoIdx;
        it[j] = a.items[c * a.n + s0 + min(j, nb - 1)];
      }
      // Stream: issue all loads of the batch, then test.
      K kv[kItemBatch][U][4];
#pragma unroll
      for (int j = 0; j < kItemBatch; ++j)
#pragma unroll
        for (int i = 0; i < U; ++i)
          if (j < nb && uu[i] >= 0)
            Vec4<K>::load(keys + (uint64_t)it[j].v * a.Sp + 4ull * uu[i], kv[j][i]);
#pragma unroll
      for (int j = 0; j < kItemBatch; ++j) {
        if (j >= nb) continue;
        const uint64_t ncp = ~it[j].cpred;
#pragma unroll
        for (int i = 0; i < U; ++i) {
          if (uu[i] < 0) continue;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if ((mk[i][e] & ncp) == 0) {
              const K kk = kv[j][i][e];
              const uint32_t g = 4u * uu[i] + e;
              if (kk > bk[j] || (kk == bk[j] && better<K>(a.tie, it[j].v, kk, g, bk[j], bg[j], ppos))) {
                bk[j] = kk;
                bg[j] = g;
              }
            }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < kItemBatch; ++j) {
        if (j >= nb) continue;
        warp_argmax<K>(a.tie, it[j].v, bk[j], bg[j], ppos);
        if (lane == 0) {
          s_k[j][warp] = bk[j];
          s_g[j][warp] = bg[j];
        }
      }
      if (threadIdx.x < kItemBatch) s_v[threadIdx.x] = it[threadIdx.x].v;
      __syncthreads();
      for (int j = warp; j < nb; j += nwarps) {
        K k = lane < nwarps ? s_k[j][lane] : (K)-INFINITY;
        uint32_t g = lane < nwarps ? s_g[j][lane] : kNoIdx;
        warp_argmax<K>(a.tie, s_v[j], k, g, ppos);
        if (lane == 0) {
          Partial<K> p;
          p.k = k;
          p.g = g;
          parts[((uint64_t)c * a.n + s0 + j) * a.G + blockIdx.x] = p;
        }
      }
      __syncthreads();
    }
  }
}

}  // namespace bnmc_dev
