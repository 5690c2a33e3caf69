// K2 — order-scan kernel (sm_100a).
//
// Replaces OrderScorer::scan_slice + argmax_reduce (engine.cpp:43-58, 15-22)
// for every (chain, rescanned row) pair of one lockstep MCMC iteration.
//
// Layout and work split
//   * Entries are grouped by 8 consecutive global indices ("sectors": 32 B of
//     fp32 keys). CTA b owns a contiguous range of sectors of EVERY row; the
//     candidate-position masks of its sectors (identical for every row, SURVEY
//     §8.1.1) are loaded once per launch into registers, with each sector's
//     intersection mask.
//   * The pairs of the iteration arrive bucketed by row (written by the step
//     kernel), so a row needed by several chains is streamed once and tested
//     against each chain's predecessor set.
//   * A sector is loaded only if some pair of the row can admit one of its
//     entries: the intersection of the sector's sets must be a subset of the
//     predecessors for ANY entry to be admissible, so lexicographic blocks whose
//     common prefix holds a non-predecessor are skipped without touching DRAM.
//   * No reduction trees: every thread folds its local winner of a pair into
//     two packed 64-bit maxima in shared memory — (key, g) and (key, ~g) — and
//     each CTA folds its cell into the same pair of global maxima. The two
//     maxima agree iff the maximal key is held by a single entry; otherwise the
//     step kernel resolves the tie exactly (rare).
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
  int max_pairs;            // C * n (capacity of the shared pair list)
  int sectors;              // Sp / 8
  int Ls;                   // sectors per CTA
  int RB;                   // rows per pipeline stage
  TieCtx tie;
  unsigned long long* sector_loads;  // optional: sectors streamed (statistics)
  int debug_exit;                    // development: stop after phase k (0 = full)
};

constexpr int kScanThreads = 512;
constexpr int kScanWarps = kScanThreads / 32;
constexpr int kMaxLs = 512;

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__host__ __device__ inline int ls_pad(int Ls) { return (Ls + 1) & ~1; }
__host__ __device__ inline int lb_pad(int Ls) { return (((Ls + 31) / 32) + 1) & ~1; }
// Dynamic shared memory of scan_kernel.
__host__ __device__ inline size_t scan_smem_bytes(int Ls, int RB, int max_pairs) {
  return (size_t)Ls * 64            // candidate masks of the slice
         + (size_t)ls_pad(Ls) * 8   // sector intersections
         + (size_t)lb_pad(Ls) * 8   // 32-sector block intersections
         + 2ull * RB * Ls * 32      // two stages of RB rows of keys
         + (size_t)max_pairs * sizeof(PairRec);
}

// K2: grid = G CTAs of 512 threads; CTA b owns sectors [b*Ls, (b+1)*Ls) of
// every row. Masks of the slice and the keys of RB rows per pipeline stage
// live in shared memory (keys staged with cp.async, only sectors whose
// intersection fits the union of the row's predecessor sets, double-buffered).
// Each warp takes whole pairs: 32-sector blocks whose intersection holds a
// non-predecessor are skipped warp-uniformly, surviving sectors are compacted
// so full warps visit them, each lane keeps the max key (and the sector that
// holds it), the lane winners are reduced with REDUX and folded into the
// pair's global maxima with two native 64-bit atomics. A lane that sees its
// max key twice reports a tie so the step kernel resolves it exactly.
__global__ void __launch_bounds__(kScanThreads) scan_kernel(ScanArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __shared__ int s_rowcnt[2][64], s_rowoff[65], s_rows[64], s_slot[64];
  __shared__ uint64_t s_union[64];
  __shared__ int s_nrows, s_sel;
  __shared__ uint16_t s_queue[kScanWarps][64];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int Ls = a.Ls, RB = a.RB, n = a.n;
  uint64_t* s_mask = reinterpret_cast<uint64_t*>(smem_raw);  // [Ls][8]
  uint64_t* s_inter = s_mask + (size_t)Ls * 8;               // [Ls]
  uint64_t* s_binter = s_inter + ls_pad(Ls);                 // [ceil(Ls/32)]
  float* s_keys = reinterpret_cast<float*>(s_binter + lb_pad(Ls));  // [2][RB][Ls][8]
  PairRec* s_pair = reinterpret_cast<PairRec*>(s_keys + 2ull * RB * Ls * 8);

  // ---- prologue (independent of the previous kernel): masks of the slice.
  const int s0 = blockIdx.x * Ls;
  const int ls = min(Ls, a.sectors - s0);
  const int nblk = (ls + 31) / 32;
  {
    const ulonglong2* src = reinterpret_cast<const ulonglong2*>(a.tie.cmask + 8ull * s0);
    ulonglong2* dst = reinterpret_cast<ulonglong2*>(s_mask);
    for (int i = tid; i < ls * 4; i += kScanThreads) dst[i] = __ldg(src + i);
  }
  __syncthreads();
  for (int i = tid; i < nblk * 32; i += kScanThreads) {
    uint64_t x = ~0ull;
    if (i < ls)
#pragma unroll
      for (int e = 0; e < 8; ++e) x &= s_mask[8 * i + e];
    if (i < Ls) s_inter[i] = x;  // sectors past the slice never pass
    // block intersection: AND over the warp's 32 consecutive sectors
    for (int off = 16; off > 0; off >>= 1) x &= __shfl_xor_sync(0xffffffffu, x, off);
    if ((i & 31) == 0) s_binter[i >> 5] = x;
  }
  cudaGridDependencySynchronize();
  if (a.debug_exit == 1) return;
  // ---- the iteration's pairs, bucketed by row (one dependent round trip for
  // the counters, one for the records).
  if (tid < n) {
    s_rowcnt[0][tid] = a.rowcnt[tid];
    s_rowcnt[1][tid] = a.rowcnt[n + tid];
  }
  if (tid == 0) s_sel = *a.sel;
  __syncthreads();
  const int b = s_sel;
  if (tid < 32) {  // prefix sum over rows + list of non-empty rows (warp 0)
    const int c0 = 2 * lane < n ? s_rowcnt[b][2 * lane] : 0;
    const int c1 = 2 * lane + 1 < n ? s_rowcnt[b][2 * lane + 1] : 0;
    int incl = c0 + c1;
    int nz = (c0 > 0) + (c1 > 0);
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int o = __shfl_up_sync(0xffffffffu, incl, off);
      const int z = __shfl_up_sync(0xffffffffu, nz, off);
      if (lane >= off) {
        incl += o;
        nz += z;
      }
    }
    const int excl = incl - c0 - c1;
    int zex = nz - (c0 > 0) - (c1 > 0);
    if (2 * lane < n) {
      s_rowoff[2 * lane] = excl;
      if (c0) s_rows[zex++] = 2 * lane;
    }
    if (2 * lane + 1 < n) {
      s_rowoff[2 * lane + 1] = excl + c0;
      if (c1) s_rows[zex] = 2 * lane + 1;
    }
    if (lane == 31) {
      s_rowoff[n] = incl;
      s_nrows = nz;
    }
  }
  __syncthreads();
  const int nrows = s_nrows;
  // Pair records of each row (warp per row) and the union of its predecessor
  // sets: a sector is staged when its intersection fits in the union.
  for (int r = warp; r < nrows; r += kScanWarps) {
    const int v = s_rows[r];
    const int off = s_rowoff[v], cnt = s_rowoff[v + 1] - off;
    uint64_t u = 0;
    for (int j = lane; j < cnt; j += 32) {
      const PairRec pr = a.buckets[(b * n + v) * kMaxChains + j];
      s_pair[off + j] = pr;
      u |= pr.cpred;
    }
    for (int o = 16; o > 0; o >>= 1) u |= __shfl_xor_sync(0xffffffffu, u, o);
    if (lane == 0) s_union[v] = u;
  }
  __syncthreads();
  if (a.debug_exit == 2) return;
  const int nbatch = (nrows + RB - 1) / RB;
  unsigned long long loads = 0;

  // Stage the keys of batch bi into buffer bi & 1.
  auto issue = [&](int bi) {
    float* stage = s_keys + (size_t)(bi & 1) * RB * Ls * 8;
    const int r0 = bi * RB, r1 = min(nrows, r0 + RB);
    for (int r = r0; r < r1; ++r) {
      const int v = s_rows[r];
      const uint64_t nu = ~s_union[v];
      const float* src = a.keys + (uint64_t)v * a.Sp + 8ull * s0;
      float* dst = stage + (size_t)(r - r0) * Ls * 8;
      for (int i = tid; i < ls; i += kScanThreads) {
        if ((s_binter[i >> 5] & nu) == 0 && (s_inter[i] & nu) == 0) {
          cp_async16(dst + 8 * i, src + 8 * i);
          cp_async16(dst + 8 * i + 4, src + 8 * i + 4);
          ++loads;
        }
      }
    }
    cp_async_commit();
  };

  uint16_t* queue = s_queue[warp];
  if (nbatch > 0) issue(0);
  for (int bi = 0; bi < nbatch; ++bi) {
    if (bi + 1 < nbatch) {
      issue(bi + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    const int r0 = bi * RB, r1 = min(nrows, r0 + RB);
    if (tid < r1 - r0) s_slot[s_rows[r0 + tid]] = tid;
    __syncthreads();
    if (a.debug_exit == 3) {
      __syncthreads();
      continue;
    }
    const float* stage = s_keys + (size_t)(bi & 1) * RB * Ls * 8;
    const int pbeg = s_rowoff[s_rows[r0]], pend = s_rowoff[s_rows[r1 - 1] + 1];
    for (int q = pbeg + warp; q < pend; q += kScanWarps) {
      const PairRec pr = s_pair[q];
      const uint64_t ncp = ~pr.cpred;
      const int v = pr.v;
      const float* rk = stage + (size_t)s_slot[v] * Ls * 8;
      float m = -INFINITY;
      int bs = -1;      // sector holding this lane's max key
      bool tie = false;  // the max key was seen in two sectors
      auto visit = [&](int i) {
        const float4 k0 = *reinterpret_cast<const float4*>(rk + 8 * i);
        const float4 k1 = *reinterpret_cast<const float4*>(rk + 8 * i + 4);
        const float kk[8] = {k0.x, k0.y, k0.z, k0.w, k1.x, k1.y, k1.z, k1.w};
        const ulonglong2* mp = reinterpret_cast<const ulonglong2*>(s_mask + 8 * i);
        float sm = -INFINITY;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const ulonglong2 mm = mp[h];
          if ((mm.x & ncp) == 0) sm = fmaxf(sm, kk[2 * h]);
          if ((mm.y & ncp) == 0) sm = fmaxf(sm, kk[2 * h + 1]);
        }
        if (sm > m) {
          m = sm;
          bs = i;
          tie = false;
        } else if (sm == m && sm != -INFINITY) {
          tie = true;
        }
      };
      // Warp-uniform block skip, then compaction of the surviving sectors.
      int qn = 0;
      for (int j = 0; j < nblk; ++j) {
        if ((s_binter[j] & ncp) != 0) continue;
        const int i = 32 * j + lane;
        const bool pass = i < ls && (s_inter[i] & ncp) == 0;
        const unsigned bal = __ballot_sync(0xffffffffu, pass);
        if (pass) queue[qn + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)i;
        qn += __popc(bal);
        if (qn >= 32) {
          __syncwarp();
          visit(queue[lane]);
          __syncwarp();
          const int rest = qn - 32;
          if (lane < rest) queue[lane] = queue[32 + lane];
          __syncwarp();
          qn = rest;
        }
      }
      __syncwarp();
      if (lane < qn) visit(queue[lane]);
      __syncwarp();
      // Lane winner inside its best sector; a repeated key flags a tie.
      uint32_t g = kNoIdx;
      if (bs >= 0) {
        for (int e = 0; e < 8; ++e) {
          if ((s_mask[8 * bs + e] & ncp) == 0 && rk[8 * bs + e] == m) {
            if (g == kNoIdx) g = 8u * (s0 + bs) + e;
            else tie = true;
          }
        }
      }
      const uint32_t ko = g == kNoIdx ? 0u : ordkey(m);
      const uint32_t mx = __reduce_max_sync(0xffffffffu, ko);
      if (mx != 0u) {
        const bool win = ko == mx;
        const uint32_t ghi = __reduce_max_sync(0xffffffffu, win ? g : 0u);
        // a lane-level tie forces glo != ghi so the step kernel resolves it
        const uint32_t mine = win ? (tie ? (g == 0 ? 1u : g - 1u) : g) : 0xFFFFFFFFu;
        const uint32_t glo = __reduce_min_sync(0xffffffffu, mine);
        if (lane == 0) {
          unsigned long long* cell = a.cell + 2ull * (pr.chain * n + pr.slot);
          atomicMax(cell, ((unsigned long long)mx << 32) | ghi);
          atomicMax(cell + 1, ((unsigned long long)mx << 32) | (uint32_t)~glo);
        }
      }
    }
    __syncthreads();
  }
  if (a.sector_loads) {
    for (int off = 16; off > 0; off >>= 1) loads += __shfl_down_sync(0xffffffffu, loads, off);
    if (lane == 0 && loads) atomicAdd(a.sector_loads, loads);
  }
}

}  // namespace bnmc_dev
