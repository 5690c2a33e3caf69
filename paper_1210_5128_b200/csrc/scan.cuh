// K2 — full-row order-scan kernel (sm_100a), the scan_mode 1 path.
//
// Replaces OrderScorer::scan_slice + argmax_reduce (engine.cpp:43-58, 15-22)
// for every (chain, rescanned row) pair of one lockstep MCMC iteration by
// streaming the rows' fp32 keys (scan2_kernel below).
//
// Layout and work split
//   * Thread t of CTA (b, y) owns 8 consecutive global indices (one 32-byte key
//     sector) of the step's rows y, y+8, ...; the candidate-position masks of
//     its entries (identical for every row) stay in registers.
//   * The pairs of the iteration arrive bucketed by row (written by the step
//     kernel), so a row needed by several chains is streamed once and tested
//     against each chain's predecessor set.
//   * A sector is loaded only if some pair of the row can admit one of its
//     entries: the intersection of the sector's sets must be a subset of the
//     union of the row's predecessor sets.
//   * Per pair: lane max, warp REDUX, shared 64-bit atomics per CTA, then one
//     pair of global atomics per CTA into two packed 64-bit maxima (key, g) and
//     (key, ~g). The two agree iff the maximal key is held by a single entry;
//     otherwise the step kernel resolves the tie exactly (rare).
//
// Exactness: the fp32 key is fl32(eff), eff = lookup + PpfTable::sum
// (engine.cpp:50-51). Rounding is monotone, so the fp64 argmax is among the
// entries whose key equals the fp32 max; ties on that key are resolved on the
// exact fp64 value, then on the reference's enumeration order over predecessor
// POSITIONS (first maximum wins, engine.cpp:52).
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace bnmc_dev {

constexpr uint32_t kNoIdx = 0xFFFFFFFFu;
constexpr int kMaxChains = 64;

struct PairRec {  // one (chain, rescanned row) pair, bucketed by row
  uint64_t cpred;  // predecessors of the row's node, as candidate positions
  uint16_t chain, slot;
  uint32_t v;
};

struct TieCtx {
  const double* __restrict__ ls;  // fp64 local scores, row stride S
  const uint64_t* __restrict__ cmask;
  const double* __restrict__ w;  // PPF weights n x n
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

// Strict "a beats b" among entries with EQUAL fp32 keys: exact fp64 value,
// then the reference tie rule.
__device__ __noinline__ bool better_slow(const TieCtx& c, int v, uint32_t ga, uint32_t gb,
                                         const uint8_t* ppos) {
  if (ga == gb) return false;
  const double ea = exact_eff(c, v, ga), eb = exact_eff(c, v, gb);
  if (ea != eb) return ea > eb;
  return tie_prefer(c, v, ga, gb, ppos);
}

// Order-preserving image of an fp32 key (0 is reserved for "no entry").
__device__ __forceinline__ uint32_t ordkey(float x) {
  const uint32_t u = __float_as_uint(x);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unordkey(uint32_t o) {
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o);
}
__device__ __forceinline__ uint64_t pack_hi(float k, uint32_t g) {
  return ((uint64_t)ordkey(k) << 32) | g;
}
__device__ __forceinline__ uint64_t pack_lo(float k, uint32_t g) {
  return ((uint64_t)ordkey(k) << 32) | (uint32_t)~g;
}

struct ScanArgs {
  const float* keys;        // n x Sp fp32 keys, padding = -inf
  uint64_t Sp;              // padded row stride (multiple of 32)
  const PairRec* buckets;   // [2][n][kMaxChains] pairs bucketed by row
  const int* rowcnt;        // [2][n] pairs per row
  const int* sel;           // which of the two buckets holds this iteration
  const uint8_t* ppos;      // [C][64] positions of the proposed order
  unsigned long long* cell; // [C][n][2] packed maxima (key,g) / (key,~g)
  int n;
  int sectors;              // Sp / 8
  TieCtx tie;
  unsigned long long* sector_loads;  // optional: sectors streamed (statistics)
};

// ---------------------------------------------------------------------------
// K2 v2 — bandwidth-oriented full-row scan. Thread t of CTA (b, y) owns 8
// consecutive global indices (32 B of keys) of the step's rows y, y+8, ...: its 8 candidate
// masks live in registers for the whole launch (loaded once; identical for all
// rows), so the per-row stream is keys only (4 B/entry, 2 x
// 128-bit loads per thread per row, fully coalesced). Rows of the step are
// processed kScan2Rows at a time with their loads in flight together; a
// sector is not loaded when its masks' intersection holds a node outside the
// union of the row's predecessor sets (no entry can be admissible). Per pair:
// lane max over its 8 admissible keys, warp REDUX, shared 64-bit atomics per
// CTA, one pair of global atomics per CTA and pair — the same (key, g) /
// (key, ~g) cells and exact tie resolution in K3 as the v1 kernel.
constexpr int kScan2Threads = 256;
#ifndef BNMC_SCAN2_PER
#define BNMC_SCAN2_PER 8
#endif
constexpr int kScan2Per = BNMC_SCAN2_PER;  // entries (32-B key sectors x 8) per thread
constexpr int kScan2RowGroups = 8;   // gridDim.y: CTA (x, y) takes rows y, y + 8, ... of the step
constexpr int kScan2MaxRows = (kMaxNodes + kScan2RowGroups - 1) / kScan2RowGroups;

__global__ void __launch_bounds__(kScan2Threads, kScan2Per > 8 ? 2 : 4) scan2_kernel(ScanArgs a) {
  __shared__ int s_cnt[64], s_rows[64], s_nrows, s_sel;
  __shared__ uint64_t s_union[64];
  __shared__ unsigned long long s_cell[kScan2MaxRows][kMaxChains][2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = a.n;
  const uint64_t slot = (uint64_t)blockIdx.x * kScan2Threads + tid;
  const bool mine_ok = slot * kScan2Per < (uint64_t)a.sectors * 8;
  const uint64_t g0 = slot * kScan2Per;
  // ---- prologue (independent of the previous kernel): masks of my sector
  uint64_t m[kScan2Per];
  uint64_t inter = ~0ull;
  {
    const ulonglong2* src = reinterpret_cast<const ulonglong2*>(a.tie.cmask + (mine_ok ? g0 : 0));
#pragma unroll
    for (int h = 0; h < kScan2Per / 2; ++h) {
      const ulonglong2 v2 = mine_ok ? __ldg(src + h) : make_ulonglong2(~0ull, ~0ull);
      m[2 * h] = v2.x;
      m[2 * h + 1] = v2.y;
    }
#pragma unroll
    for (int e = 0; e < kScan2Per; ++e) inter &= m[e];
  }
  // nodes common to every entry of the warp's 256 (lexicographically adjacent)
  // sets: a pair whose predecessors miss one of them has nothing admissible here
  const uint64_t winter = ((uint64_t)__reduce_and_sync(0xffffffffu, (unsigned)(inter >> 32)) << 32) |
                          __reduce_and_sync(0xffffffffu, (unsigned)inter);
  for (int i = tid; i < kScan2MaxRows * kMaxChains * 2; i += kScan2Threads) (&s_cell[0][0][0])[i] = 0ull;
  cudaGridDependencySynchronize();
  if (tid == 0) s_sel = *a.sel;
  __syncthreads();
  const int b = s_sel;
  if (tid < 32) {  // rows with pairs this iteration (warp 0, 2 rows per lane)
    int c[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int v = 2 * lane + h;
      c[h] = v < n ? a.rowcnt[b * n + v] : 0;
      if (v < n) s_cnt[v] = c[h];
    }
    const unsigned b0 = __ballot_sync(0xffffffffu, c[0] > 0), b1 = __ballot_sync(0xffffffffu, c[1] > 0);
    const unsigned below = (1u << lane) - 1u;
    int pos = __popc(b0 & below) + __popc(b1 & below);
    if (c[0] > 0) s_rows[pos++] = 2 * lane;
    if (c[1] > 0) s_rows[pos] = 2 * lane + 1;
    if (lane == 0) s_nrows = __popc(b0) + __popc(b1);
  }
  __syncthreads();
  const int nrows = s_nrows;
  const int ry = blockIdx.y, RG = gridDim.y;
  const int myrows = nrows > ry ? (nrows - ry + RG - 1) / RG : 0;
  for (int i = warp; i < myrows; i += kScan2Threads / 32) {  // union of predecessor sets per row
    const int v = s_rows[ry + i * RG];
    uint64_t u = 0;
    for (int j = lane; j < s_cnt[v]; j += 32) u |= a.buckets[(b * n + v) * kMaxChains + j].cpred;
    for (int o = 16; o > 0; o >>= 1) u |= __shfl_xor_sync(0xffffffffu, u, o);
    if (lane == 0) s_union[v] = u;
  }
  __syncthreads();
  // ---- rows of this CTA, no barriers: the next row's keys are in flight
  // while the current row's pairs are reduced into shared cells
  unsigned long long loads = 0;
  float kn[kScan2Per];
  bool hn = false;
  auto fetch = [&](int i, float* k) -> bool {
    if (i >= myrows || !mine_ok) return false;
    const int v = s_rows[ry + i * RG];
    if ((inter & ~s_union[v]) != 0) return false;  // no entry admissible for any pair
    const float4* src = reinterpret_cast<const float4*>(a.keys + (uint64_t)v * a.Sp + g0);
#pragma unroll
    for (int h = 0; h < kScan2Per / 4; ++h) {
      const float4 x = __ldcs(src + h);  // streamed once per launch
      k[4 * h] = x.x;
      k[4 * h + 1] = x.y;
      k[4 * h + 2] = x.z;
      k[4 * h + 3] = x.w;
    }
    loads += kScan2Per / 4;
    return true;
  };
  hn = fetch(0, kn);
  for (int i = 0; i < myrows; ++i) {
    float k[kScan2Per];
#pragma unroll
    for (int e = 0; e < kScan2Per; ++e) k[e] = hn ? kn[e] : -INFINITY;  // unloaded: nothing admissible
    hn = fetch(i + 1, kn);
    const int v = s_rows[ry + i * RG];
    const int cnt = s_cnt[v];
    for (int q = 0; q < cnt; ++q) {
      const uint64_t ncp = ~a.buckets[(b * n + v) * kMaxChains + q].cpred;
      if ((winter & ncp) != 0) continue;  // warp-uniform: no entry of the warp admissible
      // branch-free lane max: inadmissible entries become -inf (keys are finite)
      float kk[kScan2Per];
#pragma unroll
      for (int e = 0; e < kScan2Per; ++e) kk[e] = (m[e] & ncp) == 0 ? k[e] : -INFINITY;
      float mx = kk[0];
#pragma unroll
      for (int e = 1; e < kScan2Per; ++e) mx = fmaxf(mx, kk[e]);
      const uint32_t ko = mx != -INFINITY ? ordkey(mx) : 0u;
      const uint32_t mxw = __reduce_max_sync(0xffffffffu, ko);
      if (mxw != 0u) {
        // only the lanes holding the warp maximum locate it: first and last
        // entry with that key (they differ iff the lane itself holds a tie)
        const bool win = ko == mxw;
        uint32_t glast = 0u, gfirst = 0xFFFFFFFFu;
        if (win) {
          uint32_t bits = 0;
#pragma unroll
          for (int e = 0; e < kScan2Per; ++e) bits |= (kk[e] == mx ? 1u : 0u) << e;
          gfirst = (uint32_t)g0 + (__ffs(bits) - 1);
          glast = (uint32_t)g0 + (31 - __clz(bits));
        }
        const uint32_t ghi = __reduce_max_sync(0xffffffffu, glast);
        const uint32_t glo = __reduce_min_sync(0xffffffffu, gfirst);
        if (lane == 0) {
          atomicMax(&s_cell[i][q][0], ((unsigned long long)mxw << 32) | ghi);
          atomicMax(&s_cell[i][q][1], ((unsigned long long)mxw << 32) | (uint32_t)~glo);
        }
      }
    }
  }
  __syncthreads();
  // ---- the CTA's maxima of its rows' pairs into the global cells
  for (int i = 0; i < myrows; ++i) {
    const int v = s_rows[ry + i * RG];
    const int cnt = s_cnt[v];
    for (int q = tid; q < cnt; q += kScan2Threads) {
      const unsigned long long c0 = s_cell[i][q][0], c1 = s_cell[i][q][1];
      if (c0 != 0ull) {
        const PairRec pr = a.buckets[(b * n + v) * kMaxChains + q];
        unsigned long long* cell = a.cell + 2ull * (pr.chain * n + pr.slot);
        atomicMax(cell, c0);
        atomicMax(cell + 1, c1);
      }
    }
  }
  if (a.sector_loads) {  // 16-byte key slots loaded
    for (int off = 16; off > 0; off >>= 1) loads += __shfl_down_sync(0xffffffffu, loads, off);
    if (lane == 0 && loads) atomicAdd(a.sector_loads, loads);
  }
}

}  // namespace bnmc_dev
