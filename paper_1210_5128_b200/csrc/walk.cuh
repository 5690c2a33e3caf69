// K2W — sorted-row walk + fused device-resident chains (sm_100a).
//
// Exact replacement of OrderScorer::score (engine.cpp:60-98) for every
// (chain, rescanned row) pair, without streaming whole rows:
//
//   * Row v of the table is kept a second time SORTED by the effective score
//     eff = lookup + PpfTable::sum (engine.cpp:50-51, computed in fp64 in the
//     scan's association), descending, with each entry's candidate-position
//     mask. The argmax over the sets admissible for a predecessor set P is the
//     FIRST admissible entry of the sorted row (mask test cm & ~P == 0). All
//     admissible entries with exactly that fp64 value follow contiguously (up
//     to interleaved inadmissible ones); among them the reference keeps the
//     first maximum in predecessor-POSITION order (engine.cpp:52; SURVEY
//     §8.1.2), so ties are resolved on positions.
//   * A node at a small position p has few admissible sets (S(p,s)) while the
//     first admissible sorted entry can lie deep in its row (its strong
//     neighbours come later in the order). For S(p,s) <= kEnumMax the warp
//     instead ENUMERATES the admissible sets in the reference's own PST order
//     (combinatorics.hpp:83-101): position subset -> node mask -> cache index
//     (index_of / global_index) -> exact eff; strict '>' per lane and a
//     (value desc, index asc) reduction reproduce scan_slice + argmax_reduce
//     exactly. Rows with kEnumMax < S(p,s) <= S/512 walk at most 16 S(p,s)
//     entries and then enumerate (capped walks).
//   * Middle rows of a swap whose best avoids the node that moved later
//     (P' = P - X + Y) walk only the per-(row, Y) list of sorted entries
//     containing Y, down to the current best's value (delta walks).
//   * A team of TW warps runs one chain for all its iterations (run_mcmc loop
//     body, sampler.cpp:92-111): propose_swap from the split(2) stream, rescan
//     of the rows whose predecessor sets changed (positions min(a,b)..max(a,b),
//     plus rows whose best is an exact tie), total in ascending node order,
//     mh_accept (device log10 with a host replay when within 2^-48 of the
//     threshold), BestGraphTracker::update, trace row. No per-iteration launch,
//     no host round trip. walk_spec_kernel: one chain per 1024-thread CTA
//     evaluating kSpecD proposals per round.
#pragma once

#include "chain.cuh"

namespace bnmc_dev {

#ifndef BNMC_WALK_ROUND_INLINE
#define BNMC_WALK_ROUND_INLINE __forceinline__
#endif
constexpr int kWalkThreads = 256;
#ifndef BNMC_WALK_CTA1
#define BNMC_WALK_CTA1 256
#endif
constexpr int kWalkThreads1 = BNMC_WALK_CTA1;  // CTA size of one-warp chains (TW = 1)
constexpr int kWalkWarps = kWalkThreads / 32;
#ifndef BNMC_WALK_UNROLL
#define BNMC_WALK_UNROLL 4
#endif
constexpr int kWalkUnroll = BNMC_WALK_UNROLL;  // entries per lane per (deep) walk round
constexpr int kWalkPadRound = kWalkUnroll > 8 ? kWalkUnroll : 8;  // largest round of any variant
#ifndef BNMC_WALK_MINB1
#define BNMC_WALK_MINB1 4
#endif
constexpr int kWalkMinBlocks1 = BNMC_WALK_MINB1;  // CTAs per SM targeted for one-warp chains
#ifndef BNMC_ENUM_UNROLL
#define BNMC_ENUM_UNROLL 1
#endif
#ifndef BNMC_R1
#define BNMC_R1 1
#endif
constexpr int kR1 = BNMC_R1;  // entries per lane of a walk's first round (then 2x, then 4/WU)
constexpr int kEnumUnroll = BNMC_ENUM_UNROLL;  // independent gathers per lane per enumeration step
constexpr uint64_t kEnumMax = 64;          // enumerate when S(p,s) <= this (walk above)
// Rows with kEnumMax < S(p,s) <= walk cap walk at most kWalkBudget * S(p,s)
// sorted entries, then enumerate PST(p): bounds the deep walks of rows with
// few predecessors (their first admissible entry can sit 10^4 deep). The cap
// defaults to S(n-1,s) / kWalkCapDiv (measured: cfg4 1024 -> p <= 12, cfg5
// 16384 -> p <= 18); a gathered enumeration entry costs ~15 walked entries.
#ifndef BNMC_WALK_BUDGET_DEFAULT
#define BNMC_WALK_BUDGET_DEFAULT 16
#endif
constexpr uint64_t kWalkCapDiv = 512;
// Rows longer than this walk 8 entries per lane per deep round (cfg5:
// 13.4M vs 9.0M it/s), shorter rows 4 (cfg4: 100M vs 91M it/s).
constexpr uint64_t kDeepRowEntries = 1ull << 21;
constexpr uint64_t kWalkBudget = BNMC_WALK_BUDGET_DEFAULT;
#ifndef BNMC_XLEVELS
#define BNMC_XLEVELS 6
#endif
constexpr int kXLevels = BNMC_XLEVELS;  // nested exclusion lists per row (strongest parents)
#ifndef BNMC_LOG_SKIP
#define BNMC_LOG_SKIP 1
#endif
constexpr bool kLogSkip = BNMC_LOG_SKIP;  // A/B switch (tools/build_variant.sh)
constexpr int kErrDrift = 7;  // error flag: debug_recheck found a drifted chain total
constexpr uint64_t kRecheckEvery = 100;  // sampler.cpp:105

// i = base, base + stride for n <= 64 nodes and stride >= 32: at most two
// steps, written out so the compiler does not unroll a generic strided loop.
#define BNMC_FOR_NODES(i, base, stride, n) \
  _Pragma("unroll") for (int i##_h = 0; i##_h < 2; ++i##_h) \
    if (const int i = (base) + i##_h * (stride); i < (n))

struct WalkArgs {
  const ulonglong2* __restrict__ srow;  // [n][Sw] (eff bits, candidate mask), eff descending, padded
  const double* __restrict__ eff;     // [n][S] eff in global-index order
  uint64_t Sw;                        // sorted row stride (>= S + one walk round)
  const ulonglong2* __restrict__ yrow;  // [n][n-1][Syw] sorted entries of row v containing
                                       //   candidate q (delta walks), or null
  uint64_t Sy, Syw;                   // entries per list, padded stride
  const ulonglong2* __restrict__ xrow;  // exclusion lists, level j at xoff[j]: [n][Sxw[j]]
                                       //   row v without its j strongest parents, or null
  const uint64_t* __restrict__ xbit;  // [n][kXLevels] candidate bits of those parents
  int xlev;                           // levels built (0..kXLevels)
  uint64_t xoff[kXLevels + 1];
  uint32_t Sx32[kXLevels + 1], Sxw32[kXLevels + 1];  // S(n-1-j, s), padded stride
  const double* __restrict__ ls;      // [n][S] local scores, BNSC order
  const double* __restrict__ w;       // [n][n] PPF weights
  const uint64_t* __restrict__ pst;   // position masks of PST(p) for p <= pc, concatenated
  const uint32_t* __restrict__ pst_off;  // [pc+2]
  const uint64_t* __restrict__ pst2;  // PST(p, s-1) for p < pe: sets of the other positions
  const uint32_t* __restrict__ pst2_off;  // [pe+1]
  int pe;                              // largest enumerated predecessor count
  int pc;                              // largest count with a capped walk (>= pe)
  uint32_t wbud;                       // walk budget, in multiples of S(p,s)
  uint64_t S;
  uint32_t S32, Sw32, Syw32;  // S, Sw, Syw (< 2^32, checked on the host): 32x32->64 index math
  int n, s;
  // chains
  int C;
  uint64_t iters;
  int K, strict;
  const uint64_t* __restrict__ seeds;  // [C]
  const double* __restrict__ thr;      // [C][iters+1] host glibc log10(u_t), or null:
                                       // device log10 + ambiguity flag (exact replay)
  double accept_tol;                   // relative |log10_dev - log10_glibc| bound
  int* ambiguous;                      // [C] set when a decision fell inside the bound
  uint64_t* tmasks;                    // [C][K][n]
  double* ttotals;                     // [C][K]
  uint64_t* thash;                     // [C][K] graph hashes of the tracker entries
  int* tcount;                         // [C]
  uint64_t* smasks;                    // [C][K][n] tracker slots (K <= kTrackSlots), or null:
  double* stotals;                     //   entries unsorted, their order as slot indices in
  uint64_t* shash;                     //   shared memory; sorted into tmasks/ttotals at exit
  double* tr_prop;                     // [C][iters]
  uint8_t* tr_acc;
  double* tr_best;
  int* final_order;                    // [C][n]
  double* final_score;                 // [C]
  unsigned long long* accepted;        // [C]
  unsigned long long* stat;            // [0] pairs [1] walked entries [2] enumerated entries
                                       // [3] first drifted iteration (debug_recheck)
  int* error;
  int recheck;                         // RunConfig::debug_recheck
  int seq_draws;                       // test hook: draw every proposal batch sequentially
  // score-only (OrderScorer::score for C orders)
  const int* perms;                    // [C][n] or null
  uint64_t* out_masks;                 // [C][n]
  double* out_best;                    // [C][n]
  double* out_total;                   // [C]
};

// mh_accept (sampler.cpp:54-56) on the device: log10(u) < delta for the
// iteration's next_unit_open() draw u. u lies in [2^-54, 1 - 2^-54], so
// log10(u) lies in [-16.26, 0): delta >= 0 always accepts and delta < -17
// always rejects without the logarithm (most proposals at equilibrium). In
// between, CUDA's log10 may differ from glibc's in the last bits: a decision
// within tol_rel of the threshold sets *amb and the host replays the chain
// with glibc thresholds (bnmc_gpu_run_chains).
template <class Flag>
__device__ __forceinline__ bool mh_accept_dev(double u, double delta, double tol_rel, Flag* amb) {
  if (kLogSkip) {
    if (delta >= 0.0) return true;
    if (delta < -17.0) return false;
  }
  const double l = log10(u);
  const double tol = fabs(l) * tol_rel;
  if (!(l + tol < delta) && !(l - tol >= delta)) *amb = 1;
  return l < delta;
}

// a precedes b in the reference enumeration over predecessor positions (sizes
// descending, then lexicographic on sorted positions). Masks are candidate
// positions of row v; ppos[node] = position in the current order.
// Out of line: only exact ties reach it (rare), so its code stays out of the
// hot loop's instruction-cache footprint.
__device__ __noinline__ bool prefer_pos(uint64_t ma, uint64_t mb, int v, const uint8_t* ppos) {
  const int sa = __popcll(ma), sb = __popcll(mb);
  if (sa != sb) return sa > sb;
  uint64_t pa = 0, pb = 0;
  for (uint64_t m = ma; m; m &= m - 1) pa |= 1ull << ppos[cand_node(__ffsll((long long)m) - 1, v)];
  for (uint64_t m = mb; m; m &= m - 1) pb |= 1ull << ppos[cand_node(__ffsll((long long)m) - 1, v)];
  const uint64_t d = pa ^ pb;
  return d != 0 && (pa & (d & (0 - d))) != 0;
}

// global_index (combinatorics.cpp:61-76) with a shared-memory binomial table
// bt[c * 9 + j] = C(c, j), j <= 8.
__device__ __forceinline__ uint64_t gidx_smem(uint64_t mask, int c, const uint64_t* off,
                                              const uint64_t* bt) {
  // Lexicographic rank of the sorted members a_1 < ... < a_k of {0..c-1} as
  // C(c,k) - 1 - sum_t C(c-1-a_t, k-t+1) (one table lookup per member; equal to
  // the telescoped sum of combinatorics.cpp:61-76), after the larger size
  // classes off[k] = sum_{j>k} C(c, j).
  const int k = __popcll(mask);
  uint64_t idx = off[k] + bt[c * 9 + k] - 1;
  int j = k;
  for (uint64_t m = mask; m; m &= m - 1, --j) idx -= bt[(c - __ffsll((long long)m)) * 9 + j];
  return idx;
}

// subset_at (combinatorics.cpp:78-90): the position subset at PST index j of
// c positions (sizes s..0, lexicographic within a size), smem binomials.
__device__ __forceinline__ uint64_t unrank_bt(uint32_t j, int c, int s, const uint64_t* bt) {
  int k = s < c ? s : c;
  uint64_t r = j;
  for (; k > 0; --k) {
    const uint64_t block = bt[c * 9 + k];
    if (r < block) break;
    r -= block;
  }
  uint64_t mask = 0;
  int x = 0;
  for (int i = 0; i < k; ++i, ++x) {
    for (uint64_t cnt; r >= (cnt = bt[(c - x - 1) * 9 + (k - i - 1)]); ++x) r -= cnt;
    mask |= 1ull << x;
  }
  return mask;
}

__device__ __forceinline__ double shfl_d(double x, int src) {
  return __hiloint2double(__shfl_sync(0xffffffffu, __double2hiint(x), src),
                          __shfl_sync(0xffffffffu, __double2loint(x), src));
}
__device__ __forceinline__ uint64_t shfl_u64(uint64_t x, int src) {
  return ((uint64_t)__shfl_sync(0xffffffffu, (unsigned)(x >> 32), src) << 32) |
         __shfl_sync(0xffffffffu, (unsigned)x, src);
}

struct WalkHit {
  uint64_t start = ~0ull;  // sorted index of the first admissible entry
  double kstar = 0.0;      // its eff
  uint64_t kcm = 0;        // its candidate mask
  bool next_differs = false;  // the next sorted entry is known to hold another value
};

// One walk round of U entries per lane at sorted indices [base, base + 32U);
// advances base; true once the first admissible entry is found.
template <int U, bool kFloor = false>
__device__ BNMC_WALK_ROUND_INLINE bool walk_round(const ulonglong2* rr, uint64_t ncp,
                                           uint32_t S, uint32_t& base, int lane, WalkHit& h,
                                           double floor = -INFINITY, bool* exhausted = nullptr) {
  if (base >= S) return false;
  double e[U];
  uint64_t c[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t i = base + u * 32 + lane;  // < Sw < 2^32: rows are padded by one round
    const ulonglong2 x = __ldg(rr + i);  // one 16-byte (eff, mask) entry
    e[u] = __longlong_as_double((long long)x.x);
    c[u] = x.y;
  }
  // first group holding an admissible entry (at or above `floor`); its values
  // selected without dynamic register indexing, then one set of shuffles
  int hu = -1;
  unsigned hb = 0;
#pragma unroll
  for (int u = U - 1; u >= 0; --u) {
    const unsigned bal = __ballot_sync(0xffffffffu, (c[u] & ncp) == 0 && (!kFloor || e[u] >= floor));
    if (bal) {
      hu = u;
      hb = bal;
    }
  }
  base += 32 * U;
  if (hu < 0) {
    // sorted descending: once the round's last entry is below the floor, no
    // later entry can qualify
    if (kFloor && __shfl_sync(0xffffffffu, e[U - 1], 31) < floor) *exhausted = true;
    return false;
  }
  double eh = e[0], en = U > 1 ? e[1 < U ? 1 : 0] : e[0];
  uint64_t ch = c[0];
#pragma unroll
  for (int u = 1; u < U; ++u)
    if (u == hu) {
      eh = e[u];
      ch = c[u];
      en = e[u + 1 < U ? u + 1 : u];
    }
  const int f = __ffs(hb) - 1;
  h.start = (uint64_t)(base - 32 * U + hu * 32 + f);
  h.kstar = shfl_d(eh, f);
  h.kcm = shfl_u64(ch, f);
  // value of the next sorted entry, when it is in this round's registers
  const bool known = f < 31 || hu + 1 < U;
  const double nx = shfl_d(f < 31 ? eh : en, (f + 1) & 31);
  h.next_differs = known && nx != h.kstar;
  return true;
}

// Admissible entries after sorted index `start` holding exactly kstar: the
// reference keeps the first of them in predecessor-position order. Returns the
// chosen candidate mask; *ties = number of further admissible equal entries.
__device__ __noinline__ uint64_t collect_ties(const ulonglong2* rr, uint64_t ncp,
                                              uint64_t S, uint64_t start, double kstar,
                                              uint64_t kcm, int v, const uint8_t* ppos, int* ties_out) {
  const int lane = threadIdx.x & 31;
  uint64_t best_cm = kcm;
  int ties = 0;
  for (uint64_t i0 = start + 1;; i0 += 32) {
    const uint64_t i = i0 + lane;
    const ulonglong2 x = i < S ? __ldg(rr + i) : make_ulonglong2(0ull, ~0ull);
    const bool eq = i < S && __longlong_as_double((long long)x.x) == kstar;
    const uint64_t cm = eq ? x.y : ~0ull;
    const bool adm = eq && (cm & ncp) == 0;
    const unsigned bal = __ballot_sync(0xffffffffu, adm);
    if (bal) {
      ties += __popc(bal);
      uint64_t mine = adm ? cm : ~0ull;
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t other = shfl_u64(mine, lane ^ o);
        if (other != ~0ull && (mine == ~0ull || prefer_pos(other, mine, v, ppos))) mine = other;
      }
      if (prefer_pos(mine, best_cm, v, ppos)) best_cm = mine;
    }
    if (__ballot_sync(0xffffffffu, eq) != 0xffffffffu) break;
  }
  *ties_out = ties;
  return best_cm;
}

struct PairOut {
  double eff;
  uint64_t cm;  // candidate mask of the chosen set
  int tied;     // another admissible set has exactly the same eff
  uint32_t nw = 0, ne = 0;  // statistics: sorted entries walked, PST entries enumerated
};

// Warp-cooperative exact argmax of row v for the node at position p whose
// predecessors are `cpred` (candidate positions). order[pos] = node, ppos[node]
// = pos of the order being scored; bt = binomial table in shared memory.
// Exact argmax over the position subsets listed in pst[0..cnt) (PST order:
// first maximum wins, as scan_slice + argmax_reduce). ins >= 0 inserts that
// position into every listed subset (the listed subsets then range over the
// other positions): used to enumerate only the sets containing one node.
template <int EU>
__device__ __forceinline__ PairOut enum_pst(const WalkArgs& A, int v, const uint64_t* __restrict__ pst, uint32_t cnt,
                            int ins, const uint8_t* order, const uint64_t* bt, const uint64_t* boff) {
  const int lane = threadIdx.x & 31;
  const uint64_t lowm = ins >= 0 ? (1ull << ins) - 1 : ~0ull;
  const uint64_t insb = ins >= 0 ? 1ull << ins : 0ull;
  double best = -INFINITY;
  uint32_t bj = 0xFFFFFFFFu;
  bool dup = false;
  for (uint32_t j0 = 0; j0 < cnt; j0 += 32 * EU) {
    uint64_t nm[EU];
    double lv[EU];
#pragma unroll
    for (int u = 0; u < EU; ++u) {
      const uint32_t j = j0 + u * 32 + lane;
      nm[u] = 0;
      lv[u] = -INFINITY;
      if (j < cnt) {
        const uint64_t pm0 = __ldg(pst + j);
        const uint64_t pm = (pm0 & lowm) | ((pm0 & ~lowm) << 1) | insb;
        for (uint64_t m = pm; m; m &= m - 1) nm[u] |= 1ull << order[__ffsll((long long)m) - 1];
        const uint64_t g = gidx_smem(nodes_to_cand(nm[u], v), A.n - 1, boff, bt);
        lv[u] = __ldg(A.eff + (uint64_t)(uint32_t)v * A.S32 + g);
      }
    }
#pragma unroll
    for (int u = 0; u < EU; ++u) {
      const uint32_t j = j0 + u * 32 + lane;
      if (j >= cnt) continue;
      const double e = lv[u];  // ls + PpfTable::sum, precomputed (eff64_kernel)
      if (e > best) {
        best = e;
        bj = j;
        dup = false;
      } else if (e == best) {
        dup = true;
      }
    }
  }
  double m = best;
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  const bool at_max = best == m && bj != 0xFFFFFFFFu;
  const unsigned win = __ballot_sync(0xffffffffu, at_max);
  const uint32_t jmin = __reduce_min_sync(0xffffffffu, at_max ? bj : 0xFFFFFFFFu);
  PairOut r;
  r.tied = __popc(win) > 1 || __any_sync(0xffffffffu, at_max && dup);
  r.eff = m;
  r.cm = 0;
  if (jmin != 0xFFFFFFFFu) {
    const uint64_t pm0 = __ldg(pst + jmin);
    const uint64_t pm = (pm0 & lowm) | ((pm0 & ~lowm) << 1) | insb;
    uint64_t nm = 0;
    for (uint64_t q = pm; q; q &= q - 1) nm |= 1ull << order[__ffsll((long long)q) - 1];
    r.cm = nodes_to_cand(nm, v);
  }
  return r;
}

// Per-CTA shared-memory copies of the small read-only tables a pair consults:
// binomials and global_index size-class offsets, PST offsets (the walk cap and
// the enumeration ranges) and the rows' strongest-parent bits (exclusion
// levels) — shared loads instead of dependent global ones on every pair.
struct WalkSm {
  const uint64_t* bt;     // [65 * 9] binomials
  const uint64_t* boff;   // [9] global_index size-class offsets (c = n - 1)
  const uint32_t* poff;   // pst_off [pc + 2]
  const uint32_t* poff2;  // pst2_off [pe + 1]
  const uint64_t* xbit;   // [n][kXLevels]
  const uint32_t* cap;    // [kMaxNodes] walk cap by predecessor count (capped walks)
  const uint64_t* lm;     // [kMaxNodes] (1 << v) - 1: candidate <-> node mask remaps
};

// nodes_to_cand / cand_to_nodes (common.cuh) with row v's low mask from a table.
__device__ __forceinline__ uint64_t n2c(uint64_t pm, uint64_t lm) { return (pm & lm) | ((pm >> 1) & ~lm); }
__device__ __forceinline__ uint64_t c2n(uint64_t cm, uint64_t lm) {
  return (cm & lm) | ((cm << 1) & ~((lm << 1) | 1ull));
}
constexpr int kPoffMax = kMaxNodes + 2;

// Fill the WalkSm tables (every thread of the CTA; a barrier must follow).
__device__ __forceinline__ void walk_sm_fill(const WalkArgs& A, uint64_t* bt, uint64_t* boff, uint32_t* poff,
                                             uint32_t* poff2, uint64_t* xbit, uint32_t* cap, uint64_t* lm,
                                             int tid, int nthreads) {
  for (int p = tid; p < kMaxNodes; p += nthreads) {
    cap[p] = p <= A.pc ? (uint32_t)min((uint64_t)0xFFFFFFFFu,
                                       (uint64_t)A.wbud * (A.pst_off[p + 1] - A.pst_off[p]))
                       : 0xFFFFFFFFu;
    lm[p] = (1ull << p) - 1ull;
  }
  for (int i = tid; i < 65 * 9; i += nthreads) bt[i] = binom(i / 9, i % 9);
  if (tid < 9) {
    uint64_t o = 0;
    for (int j = tid + 1; j <= A.s; ++j) o += binom(A.n - 1, j);
    boff[tid] = o;
  }
  for (int i = tid; i < A.pc + 2; i += nthreads) poff[i] = A.pst_off[i];
  for (int i = tid; i < A.pe + 1; i += nthreads) poff2[i] = A.pst2_off[i];
  if (A.xrow)
    for (int i = tid; i < A.n * kXLevels; i += nthreads) xbit[i] = A.xbit[i];
}

// Row of a node whose predecessor set changed from P to P - {X} + {Y}, whose
// current best (old_eff, old_cm) does not contain X and is not an exact tie:
// the best over P' is the better of the old best and the best set containing
// Y (any other admissible set was admissible before and scored <= old_eff).
struct DeltaIn {
  bool on;
  int ypos;        // position of Y in the proposed order
  int ynode;       // Y
  double old_eff;
  uint64_t old_cm;  // candidate mask of the current best
};

// Warp-cooperative exact argmax of row v for the node at position p whose
// predecessors are `cpred` (candidate positions). order[pos] = node, ppos[node]
// = pos of the order being scored; bt = binomial table in shared memory.
template <int EU, int WU>
__device__ PairOut pair_argmax(const WalkArgs& A, int v, int p, uint64_t cpred, const uint8_t* order,
                               const uint8_t* ppos, const WalkSm& sm, const DeltaIn& d) {
  const int lane = threadIdx.x & 31;
  PairOut r;
  uint32_t walked_n = 0;
  if (p > A.pe) {
    const uint64_t ncp = ~cpred;
    if (d.on && A.yrow) {
      // ---- delta walk: only sets containing Y can beat the current best, so
      // walk row v's list of entries containing Y down to the current best's
      // value (SURVEY §7 "incremental middle rows")
      const int qy = d.ynode - (d.ynode > v);
      const uint64_t lo = (uint64_t)(uint32_t)(v * (A.n - 1) + qy) * A.Syw32;
      const ulonglong2* yr = A.yrow + lo;
      r.eff = d.old_eff;
      r.cm = d.old_cm;
      r.tied = 0;
      // the list's head is the best set containing Y (admissible or not):
      // below the current best, nothing containing Y can change the row
      // (the pair list already dropped rows whose list head is below their best)
      WalkHit h;
      bool done = false;
      uint32_t base = 0;
      const uint32_t Sy = (uint32_t)A.Sy;
      if (!walk_round<kR1, true>(yr, ncp, Sy, base, lane, h, d.old_eff, &done) && !done &&
          !walk_round<2 * kR1, true>(yr, ncp, Sy, base, lane, h, d.old_eff, &done) && !done)
        while (base < Sy && !done && !walk_round<WU, true>(yr, ncp, Sy, base, lane, h, d.old_eff, &done)) {
        }
      r.nw = base;
      if (h.start == ~0ull) return r;  // no set containing Y reaches the current best
      int ties = 0;
      uint64_t cm = h.kcm;
      if (!h.next_differs) cm = collect_ties(yr, ncp, A.Sy, h.start, h.kstar, h.kcm, v, ppos, &ties);
      if (h.kstar > d.old_eff) {
        r.eff = h.kstar;
        r.cm = cm;
        r.tied = ties > 0;
      } else {  // equal to the current best: an exact tie, position rule decides
        r.tied = 1;
        if (!prefer_pos(d.old_cm, cm, v, ppos)) r.cm = cm;
      }
      return r;
    }
    // ---- walk of the sorted row; rows with a PST(p) stop after the budget
    // and enumerate instead. When the row's strongest parent is not a
    // predecessor, no admissible set contains it: walk the row's exclusion
    // list (same admissible entries in the same order, the others skipped).
    int xj = 0;  // leading strongest parents missing from the predecessors
    if (A.xrow)
      while (xj < A.xlev && (ncp & sm.xbit[v * kXLevels + xj])) ++xj;
    const ulonglong2* rr;
    uint32_t S;
    if (xj) {
      const uint64_t ro = A.xoff[xj] + (uint64_t)(uint32_t)v * A.Sxw32[xj];
      rr = A.xrow + ro;
      S = A.Sx32[xj];
    } else {
      const uint64_t ro = (uint64_t)(uint32_t)v * A.Sw32;
      rr = A.srow + ro;
      S = A.S32;
    }
    const uint32_t lim = min(S, sm.cap[p]);
    WalkHit h;
    // Rounds grow 32, 64, 128, then 32 * WU entries: most first admissible
    // entries sit in the first 32, deep walks still get WU loads per lane in flight.
    uint32_t base = 0;
    if (walk_round<kR1>(rr, ncp, S, base, lane, h) || walk_round<2 * kR1>(rr, ncp, S, base, lane, h) ||
        walk_round<4>(rr, ncp, S, base, lane, h)) {
    } else {
      while (base < lim && base < S && !walk_round<WU>(rr, ncp, S, base, lane, h)) {
      }
    }
    walked_n = base;
    if (h.start != ~0ull) {
      r.nw = base;
      r.eff = h.kstar;
      r.cm = h.kcm;
      r.tied = 0;
      // Fast exit: the entry after `start` is still in registers of this round and
      // has a different value (exact ties are rare), so no tie is possible.
      if (h.next_differs) return r;
      // Tie collection (rare): admissible entries after `start` with eff == kstar.
      int ties = 0;
      r.cm = collect_ties(rr, ncp, S, h.start, h.kstar, h.kcm, v, ppos, &ties);
      r.tied = ties > 0;
      return r;
    }
    if (p > A.pc) {  // cannot happen: the empty set is admissible in every row
      if (lane == 0) atomicExch(A.error, 4);
      r.eff = -INFINITY;
      r.cm = 0;
      r.tied = 0;
      return r;
    }
  }
  // ---- PST enumeration. Delta rows (p <= pe): the sets containing Y only
  // (PST(p-1, s-1) with Y's position inserted); otherwise every admissible set
  // (PST(p, s)), also after a walk that ran out of budget.
  const bool de = d.on && p <= A.pe;
  const uint64_t* pst = de ? A.pst2 + sm.poff2[p - 1] : A.pst + sm.poff[p];
  const uint32_t cnt = de ? sm.poff2[p] - sm.poff2[p - 1] : sm.poff[p + 1] - sm.poff[p];
  r = enum_pst<EU>(A, v, pst, cnt, de ? d.ypos : -1, order, sm.bt, sm.boff);
  r.nw = walked_n;
  r.ne = cnt;
  if (de) {
    if (!(r.eff >= d.old_eff)) {  // also covers cnt == 0 (s == 0)
      r.eff = d.old_eff;
      r.cm = d.old_cm;
      r.tied = 0;
    } else if (r.eff == d.old_eff) {
      r.tied = 1;
      if (prefer_pos(d.old_cm, r.cm, v, ppos)) r.cm = d.old_cm;
    }
  }
  return r;
}

// BestGraphTracker::update (sampler.cpp:32-41) by one warp: dedupe by full
// graph equality, reject when full and total <= the minimum, insert at the
// lower bound of (total desc, Dag operator< over the parent masks).
template <bool kCache>
__device__ __noinline__ void tracker_insert_warp(uint64_t* tm, double* tt, uint64_t* th, int K, int n,
                                                 const uint64_t* pm, double proposed, int* tcount,
                                                 double* tcache) {
  const int lane = threadIdx.x & 31;
  const int count = *tcount;
  const bool full = count == K;
  // graph hash: dedupe compares hashes first, masks only on a hash match
  uint64_t hv = 0;
  BNMC_FOR_NODES(i, lane, 32, n) hv ^= Rng::mix(pm[i] + 0x9E3779B97F4A7C15ull * (uint64_t)(i + 1));
  const uint64_t h = ((uint64_t)__reduce_xor_sync(0xffffffffu, (unsigned)(hv >> 32)) << 32) |
                     __reduce_xor_sync(0xffffffffu, (unsigned)hv);
  for (int e0 = 0; e0 < count; e0 += 32) {
    const int e1 = e0 + lane;
    unsigned cand = __ballot_sync(0xffffffffu, e1 < count && th[e1] == h);
    while (cand) {
      const int e = e0 + __ffs(cand) - 1;
      cand &= cand - 1;
      bool eq = true;
      BNMC_FOR_NODES(i, lane, 32, n) eq &= tm[(uint64_t)e * n + i] == pm[i];
      if (__all_sync(0xffffffffu, eq)) return;  // already tracked
    }
  }
  int ins = 0;
  for (int e0 = 0; e0 < count; e0 += 32) {
    const int e = e0 + lane;
    bool prec = false;
    if (e < count) {
      const double et = tt[e];
      if (et != proposed) {
        prec = et > proposed;
      } else {
        for (int i = 0; i < n; ++i) {
          const uint64_t x = tm[(uint64_t)e * n + i], y = pm[i];
          if (x != y) {
            prec = x < y;
            break;
          }
        }
      }
    }
    ins += __popc(__ballot_sync(0xffffffffu, prec));
  }
  const int last = full ? count - 1 : count;
  __syncwarp();  // every lane's reads of the tracker above precede the writes below
  for (int e = last; e > ins; --e) {  // move entries [ins, last) down one slot
    BNMC_FOR_NODES(i, lane, 32, n) tm[(uint64_t)e * n + i] = tm[(uint64_t)(e - 1) * n + i];
    if (lane == 0) {
      tt[e] = tt[e - 1];
      th[e] = th[e - 1];
    }
    __syncwarp();
  }
  BNMC_FOR_NODES(i, lane, 32, n) tm[(uint64_t)ins * n + i] = pm[i];
  if (lane == 0) {
    tt[ins] = proposed;
    th[ins] = h;
    const int cnt = full ? count : count + 1;
    *tcount = cnt;
    if constexpr (kCache) {
      tcache[0] = tt[0];                                // best (trace rows)
      tcache[1] = cnt == K ? tt[K - 1] : -INFINITY;     // admission threshold when full
    }
  }
  __syncwarp();
}

constexpr int kTrackSlots = 32;  // largest track_top served by the slot tracker

// BestGraphTracker::update (sampler.cpp:32-41) with the entries in unsorted
// slots (tm/tt/th) and their order as slot indices in shared memory (ord): an
// insertion writes one slot and shifts at most K one-byte indices, instead of
// moving every lower entry's n masks one place down in global memory. Same
// dedupe (graph equality, hash first), same lower bound on (total desc, Dag
// operator<); K <= kTrackSlots, so one ballot covers every entry.
__device__ __noinline__ void tracker_insert_slots(uint64_t* tm, double* tt, uint64_t* th, int K, int n,
                                                  const uint64_t* pm, double proposed, int* tcount,
                                                  uint8_t* ord, double* tmin, double* tbest) {
  const int lane = threadIdx.x & 31;
  const int count = *tcount;
  const bool full = count == K;
  uint64_t hv = 0;
  BNMC_FOR_NODES(i, lane, 32, n) hv ^= Rng::mix(pm[i] + 0x9E3779B97F4A7C15ull * (uint64_t)(i + 1));
  const uint64_t h = ((uint64_t)__reduce_xor_sync(0xffffffffu, (unsigned)(hv >> 32)) << 32) |
                     __reduce_xor_sync(0xffffffffu, (unsigned)hv);
  unsigned cand = __ballot_sync(0xffffffffu, lane < count && th[lane] == h);  // slots, any order
  while (cand) {
    const int e = __ffs(cand) - 1;
    cand &= cand - 1;
    bool eq = true;
    BNMC_FOR_NODES(i, lane, 32, n) eq &= tm[(uint64_t)e * n + i] == pm[i];
    if (__all_sync(0xffffffffu, eq)) return;  // already tracked
  }
  bool prec = false;  // the lane-th best entry precedes the proposal
  uint8_t sl = 0;
  if (lane < count) {
    sl = ord[lane];
    const double et = tt[sl];
    if (et != proposed) {
      prec = et > proposed;
    } else {
      for (int i = 0; i < n; ++i) {
        const uint64_t x = tm[(uint64_t)sl * n + i], y = pm[i];
        if (x != y) {
          prec = x < y;
          break;
        }
      }
    }
  }
  const int ins = __popc(__ballot_sync(0xffffffffu, prec));
  const int last = full ? count - 1 : count;
  const int evict = __shfl_sync(0xffffffffu, (int)sl, K - 1);
  const int slot = full ? evict : count;  // the minimum's slot is reused when full
  const int prev = __shfl_up_sync(0xffffffffu, (int)sl, 1);
  __syncwarp();
  if (lane > ins && lane <= last) ord[lane] = (uint8_t)prev;  // entries [ins, last) move down
  if (lane == ins) ord[ins] = (uint8_t)slot;
  BNMC_FOR_NODES(i, lane, 32, n) tm[(uint64_t)slot * n + i] = pm[i];
  if (lane == 0) {
    tt[slot] = proposed;
    th[slot] = h;
    const int cnt = full ? count : count + 1;
    *tcount = cnt;
  }
  __syncwarp();
  if (lane == 0) {
    const int cnt = *tcount;
    *tbest = tt[ord[0]];
    *tmin = cnt == K ? tt[ord[K - 1]] : -INFINITY;
  }
  __syncwarp();
}

// kCache: tcache (shared) holds [0] the tracker best and [1] its minimum when
// full (else -inf), kept current by the insert so the common rejection needs
// no global load (single-chain kernel); otherwise the tracker is read directly.
template <bool kCache>
__device__ __forceinline__ void tracker_offer_warp(uint64_t* tm, double* tt, uint64_t* th, int K, int n,
                                                   const uint64_t* pm, double proposed, int* tcount,
                                                   double* tcache) {
  if constexpr (kCache) {
    if (proposed <= tcache[1]) return;  // full: not above the minimum
  } else {
    const int count = *tcount;
    if (count == K && proposed <= tt[count - 1]) return;
  }
  tracker_insert_warp<kCache>(tm, tt, th, K, n, pm, proposed, tcount, tcache);
}

// Barrier over the TW warps of one team (a team runs one chain).
template <int TW>
__device__ __forceinline__ void team_sync(int team) {
  constexpr int kCta = TW == 1 ? kWalkThreads1 : (TW * 32 > kWalkThreads ? TW * 32 : kWalkThreads);
  if constexpr (TW == 1) {
    __syncwarp();
  } else if constexpr (TW * 32 == kCta) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(team + 1), "r"(TW * 32) : "memory");
  }
}

struct TeamState;
__device__ __noinline__ void init_team_state(TeamState& S, const WalkArgs& A, int c, int n,
                                             bool score_only);

// Per-team chain state in shared memory.
struct TeamState {
  uint8_t order[64], prop[64], ppos[64];
  uint8_t pv[64], pp[64], pt[64];  // pair -> node, position, exact-tie flag
  uint8_t pd[64];                  // pair -> delta rescan eligible (P' = P - X + Y)
  uint64_t pc[64];                 // pair -> candidate predecessor mask
  uint64_t pm[64];                 // proposed graph (parent node masks by node)
  alignas(16) double pb[64];       // proposed per-node bests
  uint64_t cm[64];                 // current graph
  double cb[64];                   // current per-node bests
  uint64_t tied, tied_new, rng, arng;
  double total, cur_total;
  double tmin;  // tracker minimum when full (-inf before), kept by the insert path
  double tbest;                    // tracker maximum (slot tracker: trace rows)
  uint8_t tord[32];                // slot tracker: slot of the e-th best entry
  uint8_t qa[32], qb[32];          // proposals of the current batch of 32 iterations
  double qu[32];                   // their accept draws next_unit_open()
  unsigned long long acc;
  int np, a, b, accept, tcount, amb;
};

// Chain start (one thread, out of line: once per chain): the order to score,
// or the initial shuffle of the split(1) stream and the split(2)/(3) streams
// (sampler.cpp:77-86).
__device__ __noinline__ void init_team_state(TeamState& S, const WalkArgs& A, int c, int n,
                                             bool score_only) {
  if (score_only) {
    for (int i = 0; i < n; ++i) S.order[i] = (uint8_t)A.perms[(uint64_t)c * n + i];
  } else {
    const Rng master{A.seeds[c]};
    Rng init = master.split(1);
    for (int i = 0; i < n; ++i) S.order[i] = (uint8_t)i;
    for (int i = n; i > 1; --i) {
      const int j = (int)init.next_below((uint64_t)i);
      const uint8_t t = S.order[i - 1];
      S.order[i - 1] = S.order[j];
      S.order[j] = t;
    }
    S.rng = master.split(2).s;
    S.arng = master.split(3).s;
  }
  S.tied = 0;
  S.amb = 0;
  S.tcount = 0;
  S.tmin = -INFINITY;
  S.tbest = -INFINITY;
  S.acc = 0;
  S.cur_total = 0.0;
}

constexpr int kPropBatch = 32;  // iterations whose proposals are drawn together

// The next kPropBatch iterations' propose_swap draws (split(2) stream: a =
// next_below(n), b = next_below(n - 1), b += b >= a) and mh_accept draws
// (split(3) stream: next_unit_open), lane i for iteration i of the batch, by
// direct indexing of the splitmix64 sequence (rng.hpp:14-45). Exact: when any
// draw of the batch falls below next_below's rejection threshold, lane 0
// redraws the batch sequentially with rejection.
__device__ __noinline__ void draw_proposal_batch(TeamState& S, const FastDiv* div, int lane, bool seq) {
  constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
  const uint64_t s0 = S.rng, sa = S.arng;
  const uint64_t x0 = Rng::mix(s0 + kGamma * (uint64_t)(2 * lane + 1));
  const uint64_t x1 = Rng::mix(s0 + kGamma * (uint64_t)(2 * lane + 2));
  const uint64_t xu = Rng::mix(sa + kGamma * (uint64_t)(lane + 1));
  S.qu[lane] = ((double)(xu >> 11) + 0.5) * 0x1.0p-53;
  if (!seq && __all_sync(0xffffffffu, x0 >= div[0].thr && x1 >= div[1].thr)) {
    const int a = (int)div[0].mod(x0);
    int b = (int)div[1].mod(x1);
    if (b >= a) ++b;
    S.qa[lane] = (uint8_t)a;
    S.qb[lane] = (uint8_t)b;
    __syncwarp();
    if (lane == 0) S.rng = s0 + kGamma * (uint64_t)(2 * kPropBatch);
  } else {
    __syncwarp();
    if (lane == 0) {
      Rng pr{s0};
      for (int i = 0; i < kPropBatch; ++i) {
        const int a = (int)pr.next_below(div[0]);
        int b = (int)pr.next_below(div[1]);
        if (b >= a) ++b;
        S.qa[i] = (uint8_t)a;
        S.qb[i] = (uint8_t)b;
      }
      S.rng = pr.s;
    }
  }
  if (lane == 0) S.arng = sa + kGamma * (uint64_t)kPropBatch;
  __syncwarp();
}

template <int TW>
__host__ __device__ constexpr int walk_cta_threads() {
  return TW == 1 ? kWalkThreads1 : (TW * 32 > kWalkThreads ? TW * 32 : kWalkThreads);
}

// TW warps per chain, max(256, 32 TW) / (32 TW) chains per CTA. TW >= 8 gives
// one chain the whole CTA (lower latency per iteration); TW = 1 runs a chain
// per warp, barrier-free, for throughput over many chains.

// WU: entries per lane per deep walk round (4 for rows of ~10^5-10^6 entries
// whose walks end early; 8 for deeper rows, e.g. cfg5, where more loads in
// flight pay).
// RC: debug_recheck instantiation (a separate variant keeps the recheck state
// out of the registers of the production kernel).
template <int TW, int WU = (TW >= 8 ? 8 : kWalkUnroll), bool RC = false>
__global__ void __launch_bounds__(walk_cta_threads<TW>(), TW == 1 ? kWalkMinBlocks1 : (TW > 8 ? 1024 / (TW * 32) : 4))
    walk_chain_kernel(WalkArgs A) {
  constexpr int kCta = walk_cta_threads<TW>();
  constexpr int kTeams = kCta / (32 * TW);
  __shared__ uint64_t s_bt[65 * 9];
  __shared__ uint64_t s_boff[9];  // size-class offsets of global_index for c = n - 1
  __shared__ TeamState s_team[kTeams];
  __shared__ FastDiv s_div[2];  // propose_swap's bounds n and n - 1
  __shared__ uint32_t s_poff[kPoffMax], s_poff2[kPoffMax];
  __shared__ uint64_t s_xbit[kMaxNodes * kXLevels];
  __shared__ uint32_t s_cap[kMaxNodes];
  __shared__ uint64_t s_lm[kMaxNodes];
  const int tid = threadIdx.x, lane = tid & 31;
  const int team = (tid >> 5) / TW, twarp = (tid >> 5) % TW, ttid = tid - team * TW * 32;
  const int c = blockIdx.x * kTeams + team;
  const int n = A.n;
  if (tid < 2) s_div[tid] = FastDiv::make((uint64_t)(n - tid));
  walk_sm_fill(A, s_bt, s_boff, s_poff, s_poff2, s_xbit, s_cap, s_lm, tid, kCta);
  const WalkSm sm{s_bt, s_boff, s_poff, s_poff2, s_xbit, s_cap, s_lm};
  __syncthreads();
  if (c >= A.C) return;  // whole teams only: no later CTA-wide barrier when TW < 8
  TeamState& S = s_team[team];
  const bool score_only = A.perms != nullptr;
  if (ttid == 0) init_team_state(S, A, c, n, score_only);
  team_sync<TW>(team);
  uint32_t walked = 0, enumerated = 0;  // statistics per warp (u32: statistics only)
  uint32_t pairs = 0;
  const uint64_t T = score_only ? 0 : A.iters;
  // rc: a debug_recheck pass (sampler.cpp:105-110) after iteration t-1: the
  // current order is re-scored from scratch (every row, full walks, no delta
  // or tie state) and its total compared with the chain's running total
  uint64_t t = 0;
  bool rc = false;
  while (t <= T || (RC && rc)) {
    // fresh: score every row of S.order, no proposal (recomputed at each use:
    // a live predicate costs the production kernel a register)
#define BNMC_FRESH (t == 0 || (RC && rc))
    // ---- proposal: propose_swap (sampler.cpp:43-52) from the split(2) stream.
    // The proposal and accept streams do not depend on the chain's state, and
    // splitmix64's k-th draw is mix(state + k*gamma): every 32 iterations the
    // team's first warp draws the next 32 proposals and accept draws at once,
    // one iteration per lane. next_below's rejection (probability ~n/2^64) is
    // detected exactly; such a batch is redrawn in sequence by lane 0.
    if (!BNMC_FRESH && twarp == 0 && ((t - 1) & (kPropBatch - 1)) == 0)
      draw_proposal_batch(S, s_div, lane, A.seq_draws != 0);
    if (ttid == 0) {
      int a = 0, b = n - 1;
      if (!BNMC_FRESH) {
        const int k = (int)((t - 1) & (kPropBatch - 1));
        a = S.qa[k];
        b = S.qb[k];
      }
      S.a = a;
      S.b = b;
    }
    team_sync<TW>(team);
    const int pa = S.a, pb = S.b;
    const int lo = !BNMC_FRESH ? min(pa, pb) : 0, hi = !BNMC_FRESH ? max(pa, pb) : n - 1;
    BNMC_FOR_NODES(i, ttid, TW * 32, n) {
      const int src = BNMC_FRESH ? i : (i == pa ? pb : (i == pb ? pa : i));
      S.prop[i] = S.order[src];
      S.pm[i] = S.cm[i];
      S.pb[i] = S.cb[i];
    }
    team_sync<TW>(team);
    // pair list (first warp of the team): positions lo..hi plus positions > hi
    // whose best is an exact tie (their position-order tie-break may change)
    if (twarp == 0) {
      uint64_t bit[2];
      bool take[2], dl[2];
      const int xnode = S.prop[hi], ynode = S.prop[lo];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int p = 2 * lane + h;
        const int v = p < n ? S.prop[p] : 0;
        bit[h] = p < n ? 1ull << v : 0ull;
        take[h] = p < n && ((p >= lo && p <= hi) || (p > hi && (S.tied & bit[h])));
        // middle rows of a swap: the node at hi (X) left the predecessors, the
        // node at lo (Y) joined; delta-eligible when the current best avoids X
        // and is not an exact tie. A walked delta row whose Y-list head (the
        // best set containing Y) is below its current best keeps its best: it
        // is dropped here, one load per row in parallel, instead of costing a
        // pair (pair_argmax's delta early exit, same test)
        dl[h] = take[h] && !BNMC_FRESH && p > lo && p < hi && (p <= A.pe || A.yrow) &&
                !(S.tied & bit[h]) && !((S.cm[v] >> xnode) & 1ull);
        if (dl[h] && p > A.pe &&
            __longlong_as_double((long long)__ldg(&A.yrow[(uint64_t)(uint32_t)(v * (n - 1) + ynode - (ynode > v)) * A.Syw32].x)) <
                S.cb[v])
          take[h] = false;
      }
      uint64_t incl = bit[0] | bit[1];
      int cnt = (int)take[0] + (int)take[1];
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint64_t o = __shfl_up_sync(0xffffffffu, incl, off);
        const int k = __shfl_up_sync(0xffffffffu, cnt, off);
        if (lane >= off) {
          incl |= o;
          cnt += k;
        }
      }
      int slot = cnt - (int)take[0] - (int)take[1];
      const uint64_t pre0 = incl & ~(bit[0] | bit[1]);
      const uint64_t pre[2] = {pre0, pre0 | bit[0]};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int p = 2 * lane + h;
        if (p >= n) continue;
        const int v = S.prop[p];
        S.ppos[v] = (uint8_t)p;
        if (!take[h]) continue;
        S.pv[slot] = (uint8_t)v;
        S.pp[slot] = (uint8_t)p;
        S.pc[slot] = nodes_to_cand(pre[h], v);
        S.pd[slot] = (uint8_t)dl[h];
        ++slot;
      }
      if (lane == 31) S.np = cnt;
    }
    team_sync<TW>(team);
    // ---- exact argmax of every rescanned row, one warp per pair (the bound is
    // re-read from shared memory: a register for it was spilled around pairs)
    for (int q = twarp; q < *reinterpret_cast<volatile int*>(&S.np); q += TW) {
      const int v = S.pv[q];
      DeltaIn d;
      d.on = S.pd[q] != 0;
      d.ypos = lo;
      d.ynode = S.prop[lo];
      d.old_eff = S.cb[v];
      d.old_cm = n2c(S.cm[v], sm.lm[v]);
      // few chains in flight (TW >= 8): more independent gathers per lane
      const PairOut o = pair_argmax<TW >= 8 ? 4 : kEnumUnroll, WU>(A, v, S.pp[q], S.pc[q], S.prop, S.ppos, sm, d);
      walked += o.nw;
      enumerated += o.ne;
      if (lane == 0) {
        S.pm[v] = c2n(o.cm, sm.lm[v]);
        S.pb[v] = o.eff;
        S.pt[q] = (uint8_t)o.tied;
      }
    }
    pairs += S.np;
    team_sync<TW>(team);
    // ---- total in ascending node order (engine.cpp:95-96), tie bits, mh_accept
    if (twarp == 0) {
      // tie bits of the rescanned rows (distinct nodes: order-free), by the warp
      uint64_t clr = 0, set = 0;
      const int np = S.np;
      BNMC_FOR_NODES(q, lane, 32, np) {
        const uint64_t b = 1ull << S.pv[q];
        clr |= b;
        set |= S.pt[q] ? b : 0ull;
      }
      clr = ((uint64_t)__reduce_or_sync(0xffffffffu, (unsigned)(clr >> 32)) << 32) |
            __reduce_or_sync(0xffffffffu, (unsigned)clr);
      set = ((uint64_t)__reduce_or_sync(0xffffffffu, (unsigned)(set >> 32)) << 32) |
            __reduce_or_sync(0xffffffffu, (unsigned)set);
      if (lane == 0) S.tied_new = (S.tied & ~clr) | set;
    }
    if (ttid == 0) {
      // serial sum in ascending node order (bit-exact), two values per load
      double tot = 0.0;
      const double2* pb2 = reinterpret_cast<const double2*>(S.pb);
      for (int i = 0; i < (n >> 1); ++i) {
        const double2 x = pb2[i];
        tot += x.x;
        tot += x.y;
      }
      if (n & 1) tot += S.pb[n - 1];
      S.total = tot;
      if (RC && rc && tot != S.cur_total) {  // debug_recheck drift: first report wins
        atomicCAS(A.stat + 3, 0ull, (unsigned long long)(t - 1));
        atomicExch(A.error, kErrDrift);
      }
      // mh_accept, sampler.cpp:54-56: log10(u) < new - old, with the host's glibc
      // log10(u) when A.thr, else the batch's draw u (logarithm only when needed)
      const double delta = tot - S.cur_total;
      bool acc = true;
      if (!BNMC_FRESH)
        acc = A.thr ? A.thr[(uint64_t)c * (A.iters + 1) + t] < delta
                    : mh_accept_dev(S.qu[(t - 1) & (kPropBatch - 1)], delta, A.accept_tol, &S.amb);
      S.accept = acc;
    }
    team_sync<TW>(team);
    if (RC && rc) {  // nothing of the recheck pass is committed
      rc = false;
      continue;
    }
    if (score_only) {
      BNMC_FOR_NODES(i, ttid, TW * 32, n) {
        A.out_masks[(uint64_t)c * n + i] = S.pm[i];
        A.out_best[(uint64_t)c * n + i] = S.pb[i];
      }
      if (ttid == 0) A.out_total[c] = S.total;
      break;
    }
    const double proposed = S.total;
    const bool accepted = S.accept;
    // ---- BestGraphTracker::update; every proposal is offered unless strict
    // (the full tracker's minimum is mirrored in shared memory: the common
    // rejection needs no global load)
    if (twarp == 0 && (t == 0 || accepted || !A.strict) && !(S.tcount == A.K && proposed <= S.tmin)) {
      double* tt = A.ttotals + (uint64_t)c * A.K;
      if (A.smasks) {
        const uint64_t so = (uint64_t)c * A.K;
        tracker_insert_slots(A.smasks + so * n, A.stotals + so, A.shash + so, A.K, n, S.pm, proposed,
                             &S.tcount, S.tord, &S.tmin, &S.tbest);
      } else {
        tracker_insert_warp<false>(A.tmasks + (uint64_t)c * A.K * n, tt, A.thash + (uint64_t)c * A.K,
                                   A.K, n, S.pm, proposed, &S.tcount, nullptr);
        __syncwarp();
        if (lane == 0 && S.tcount == A.K) S.tmin = tt[A.K - 1];
      }
    }
    // ---- commit + trace row
    if (accepted)
      BNMC_FOR_NODES(i, ttid, TW * 32, n) {
        S.cm[i] = S.pm[i];
        S.cb[i] = S.pb[i];
        S.order[i] = S.prop[i];
      }
    if (ttid == 0) {
      if (accepted) {
        S.cur_total = proposed;
        S.tied = S.tied_new;
        if (t > 0) ++S.acc;
      }
      if (t > 0) {
        const uint64_t o = (uint64_t)c * A.iters + (t - 1);
        A.tr_prop[o] = proposed;
        A.tr_acc[o] = accepted ? 1 : 0;
        A.tr_best[o] = A.smasks ? S.tbest : A.ttotals[(uint64_t)c * A.K];
      }
    }
    team_sync<TW>(team);
    if constexpr (RC) rc = t > 0 && t % kRecheckEvery == 0;
    ++t;
  }
#undef BNMC_FRESH
  if (!score_only) {
    BNMC_FOR_NODES(i, ttid, TW * 32, n) A.final_order[(uint64_t)c * n + i] = S.order[i];
    if (A.smasks && twarp == 0) {  // slot tracker -> tmasks/ttotals in (total desc, Dag <) order
      const uint64_t so = (uint64_t)c * A.K;
      for (int e = 0; e < S.tcount; ++e) {
        const uint64_t sl = S.tord[e];
        BNMC_FOR_NODES(i, lane, 32, n) A.tmasks[(so + e) * n + i] = A.smasks[(so + sl) * n + i];
        if (lane == 0) A.ttotals[so + e] = A.stotals[so + sl];
      }
    }
    if (ttid == 0) {
      A.final_score[c] = S.cur_total;
      A.accepted[c] = S.acc;
      A.tcount[c] = S.tcount;
      if (A.ambiguous) A.ambiguous[c] = S.amb;
    }
  }
  if (lane == 0 && A.stat) {
    atomicAdd(A.stat + 1, (unsigned long long)walked);
    atomicAdd(A.stat + 2, (unsigned long long)enumerated);
    if (twarp == 0) atomicAdd(A.stat, (unsigned long long)pairs);
  }
}

// ---------------------------------------------------------------------------
// Speculative single-chain kernel (one chain per 1024-thread CTA).
//
// The proposal positions and the acceptance draws are state-independent
// streams (split(2), split(3)); only the base order depends on earlier
// acceptances, and most proposals are rejected. Each round therefore
// evaluates the next D proposals all against the CURRENT order (their rows
// in parallel, one warp per rescanned row), then commits them in sequence
// exactly as run_mcmc would (sampler.cpp:92-111): total, mh_accept, tracker
// offer, trace row — up to and including the first accepted proposal, whose
// graph becomes the state. Later proposals of the round were evaluated on a
// stale order and are discarded; both streams are rewound to just after the
// last committed iteration. Results are the reference's bit for bit.
#ifndef BNMC_SPEC_D
#define BNMC_SPEC_D 4
#endif
constexpr int kSpecD = BNMC_SPEC_D;  // proposals evaluated per round

struct SpecSlot {
  uint8_t prop[64], ppos[64];
  uint8_t pv[64], pp[64], pt[64], pd[64];
  uint64_t pc[64];
  uint64_t pm[64];
  alignas(16) double pb[64];
  uint64_t rng_after, arng_after;
  double thr, total;
  int a, b, np, first;  // first: index of this slot's first pair in the flat list
  uint8_t acc, amb;
};

__global__ void __launch_bounds__(1024, 1) walk_spec_kernel(WalkArgs A) {
  constexpr int kThreads = 1024, kWarps = kThreads / 32;
  __shared__ uint64_t s_bt[65 * 9];
  __shared__ uint64_t s_boff[9];
  __shared__ SpecSlot s_sl[kSpecD];
  __shared__ uint8_t s_order[64];
  __shared__ uint64_t s_cm[64];
  __shared__ double s_cb[64];
  __shared__ uint64_t s_tied, s_rng, s_arng;
  __shared__ double s_cur_total;
  __shared__ unsigned long long s_acc;
  __shared__ int s_tcount, s_amb, s_d, s_npairs, s_done_to;
  __shared__ double s_tcache[2];
  __shared__ uint8_t s_tord[kTrackSlots];  // slot tracker order (A.smasks)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = blockIdx.x;
  const int n = A.n;
  __shared__ FastDiv s_div[2];  // propose_swap's bounds n and n - 1
  __shared__ uint32_t s_poff[kPoffMax], s_poff2[kPoffMax];
  __shared__ uint64_t s_xbit[kMaxNodes * kXLevels];
  __shared__ uint32_t s_cap[kMaxNodes];
  __shared__ uint64_t s_lm[kMaxNodes];
  if (threadIdx.x < 2) s_div[threadIdx.x] = FastDiv::make((uint64_t)(n - threadIdx.x));
  walk_sm_fill(A, s_bt, s_boff, s_poff, s_poff2, s_xbit, s_cap, s_lm, tid, kThreads);
  const WalkSm sm{s_bt, s_boff, s_poff, s_poff2, s_xbit, s_cap, s_lm};
  if (tid == 0) {
    const Rng master{A.seeds[c]};
    Rng init = master.split(1);  // initial order: shuffle (sampler.cpp:83-86)
    for (int i = 0; i < n; ++i) s_order[i] = (uint8_t)i;
    for (int i = n; i > 1; --i) {
      const int j = (int)init.next_below((uint64_t)i);
      const uint8_t t = s_order[i - 1];
      s_order[i - 1] = s_order[j];
      s_order[j] = t;
    }
    s_rng = master.split(2).s;
    s_arng = master.split(3).s;
    for (int i = 0; i < 64; ++i) {
      s_cm[i] = 0;
      s_cb[i] = 0.0;
    }
    s_tied = 0;
    s_tcount = 0;
    s_tcache[0] = -INFINITY;
    s_tcache[1] = -INFINITY;
    s_acc = 0;
    s_amb = 0;
    s_cur_total = 0.0;
  }
  __syncthreads();
  unsigned long long walked = 0, enumerated = 0;  // statistics (lane 0 of each warp)
  unsigned long long pairs = 0;
  uint64_t t = 0;  // iterations committed so far (0 = initial order not yet scored)
  while (t <= A.iters) {
    // ---- proposals of this round (warp 0, lane i for slot i): positions and
    // accept draws by direct indexing of the splitmix64 streams (k-th draw =
    // mix(state + k*gamma)); a next_below rejection anywhere in the round
    // (probability ~n/2^64) sends the round to lane 0's sequential draws
    if (warp == 0) {
      constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
      const int d = t == 0 ? 1 : (int)min((uint64_t)kSpecD, A.iters - t + 1);
      const uint64_t s0 = s_rng, sa = s_arng;
      const bool mine = lane < d;
      uint64_t x0 = 0, x1 = 0;
      if (mine && t > 0) {
        x0 = Rng::mix(s0 + kGamma * (uint64_t)(2 * lane + 1));
        x1 = Rng::mix(s0 + kGamma * (uint64_t)(2 * lane + 2));
      }
      const bool ok = __all_sync(0xffffffffu, !mine || t == 0 || (x0 >= s_div[0].thr && x1 >= s_div[1].thr));
      if (ok && mine) {
        SpecSlot& S = s_sl[lane];
        if (t == 0) {
          S.a = 0;
          S.b = n - 1;
          S.thr = 0.0;
          S.rng_after = s0;
          S.arng_after = sa;
        } else {
          const int a = (int)s_div[0].mod(x0);  // propose_swap, sampler.cpp:43-52
          int b = (int)s_div[1].mod(x1);
          if (b >= a) ++b;
          S.a = a;
          S.b = b;
          const uint64_t xu = Rng::mix(sa + kGamma * (uint64_t)(lane + 1));
          // host glibc log10(u) with host thresholds (the device stream still advances)
          S.thr = A.thr ? A.thr[(uint64_t)c * (A.iters + 1) + t + lane] : ((double)(xu >> 11) + 0.5) * 0x1.0p-53;
          S.rng_after = s0 + kGamma * (uint64_t)(2 * lane + 2);
          S.arng_after = sa + kGamma * (uint64_t)(lane + 1);
        }
        S.amb = 0;
      } else if (!ok && lane == 0) {
        Rng pr{s0}, ar{sa};
        for (int i = 0; i < d; ++i) {
          SpecSlot& S = s_sl[i];
          int a = (int)pr.next_below(s_div[0]);
          int b = (int)pr.next_below(s_div[1]);
          if (b >= a) ++b;
          S.a = a;
          S.b = b;
          const uint64_t it = t + i;
          if (A.thr) {
            S.thr = A.thr[(uint64_t)c * (A.iters + 1) + it];
            ar.next_u64();
          } else {
            S.thr = ar.next_unit_open();
          }
          S.rng_after = pr.s;
          S.arng_after = ar.s;
          S.amb = 0;
        }
      }
      if (lane == 0) s_d = d;
    }
    __syncthreads();
    const int d = s_d;
    // ---- proposed orders (every slot swaps two positions of the CURRENT order)
    for (int idx = tid; idx < d * 64; idx += kThreads) {
      const int i = idx >> 6, p = idx & 63;
      if (p >= n) continue;
      SpecSlot& S = s_sl[i];
      const int src = t == 0 ? p : (p == S.a ? S.b : (p == S.b ? S.a : p));
      S.prop[p] = s_order[src];
      S.pm[p] = s_cm[p];
      S.pb[p] = s_cb[p];
    }
    __syncthreads();
    // ---- pair lists, one warp per slot (positions lo..hi + exact-tie rows)
    if (warp < d) {
      SpecSlot& S = s_sl[warp];
      const int lo = t > 0 ? min(S.a, S.b) : 0, hi = t > 0 ? max(S.a, S.b) : n - 1;
      uint64_t bit[2];
      bool take[2], dl[2];
      const int xnode = S.prop[hi], ynode = S.prop[lo];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int p = 2 * lane + h;
        const int v = p < n ? S.prop[p] : 0;
        bit[h] = p < n ? 1ull << v : 0ull;
        take[h] = p < n && ((p >= lo && p <= hi) || (p > hi && (s_tied & bit[h])));
        // delta rows whose Y-list head is below the current best keep it
        // (as in walk_chain_kernel's pair list)
        dl[h] = take[h] && t > 0 && p > lo && p < hi && (p <= A.pe || A.yrow) &&
                !(s_tied & bit[h]) && !((s_cm[v] >> xnode) & 1ull);
        if (dl[h] && p > A.pe &&
            __longlong_as_double((long long)__ldg(&A.yrow[(uint64_t)(uint32_t)(v * (n - 1) + ynode - (ynode > v)) * A.Syw32].x)) <
                s_cb[v])
          take[h] = false;
      }
      uint64_t incl = bit[0] | bit[1];
      int cnt = (int)take[0] + (int)take[1];
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint64_t o = __shfl_up_sync(0xffffffffu, incl, off);
        const int kk = __shfl_up_sync(0xffffffffu, cnt, off);
        if (lane >= off) {
          incl |= o;
          cnt += kk;
        }
      }
      int slot = cnt - (int)take[0] - (int)take[1];
      const uint64_t pre0 = incl & ~(bit[0] | bit[1]);
      const uint64_t pre[2] = {pre0, pre0 | bit[0]};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int p = 2 * lane + h;
        if (p >= n) continue;
        const int v = S.prop[p];
        S.ppos[v] = (uint8_t)p;
        if (!take[h]) continue;
        S.pv[slot] = (uint8_t)v;
        S.pp[slot] = (uint8_t)p;
        S.pc[slot] = nodes_to_cand(pre[h], v);
        S.pd[slot] = (uint8_t)dl[h];
        ++slot;
      }
      if (lane == 31) S.np = cnt;
    }
    __syncthreads();
    if (tid == 0) {
      int f = 0;
      for (int i = 0; i < d; ++i) {
        s_sl[i].first = f;
        f += s_sl[i].np;
      }
      s_npairs = f;
    }
    __syncthreads();
    // ---- every rescanned row of every slot, one warp per pair
    const int total_pairs = s_npairs;
    for (int q = warp; q < total_pairs; q += kWarps) {
      int i = 0;
      while (i + 1 < d && q >= s_sl[i + 1].first) ++i;
      SpecSlot& S = s_sl[i];
      const int qi = q - S.first;
      const int v = S.pv[qi];
      const int lo = t > 0 ? min(S.a, S.b) : 0;
      DeltaIn dl;
      dl.on = S.pd[qi] != 0;
      dl.ypos = lo;
      dl.ynode = S.prop[lo];
      dl.old_eff = s_cb[v];
      dl.old_cm = n2c(s_cm[v], sm.lm[v]);
      const PairOut o = pair_argmax<4, 8>(A, v, S.pp[qi], S.pc[qi], S.prop, S.ppos, sm, dl);
      walked += o.nw;
      enumerated += o.ne;
      if (lane == 0) {
        S.pm[v] = c2n(o.cm, sm.lm[v]);
        S.pb[v] = o.eff;
        S.pt[qi] = (uint8_t)o.tied;
      }
    }
    __syncthreads();
    // ---- totals and mh_accept of every slot in parallel (warp i, slot i): until
    // the first acceptance every slot compares against the same current total
    if (warp < d && lane == 0) {
      SpecSlot& S = s_sl[warp];
      const uint64_t it = t + warp;
      double tot = 0.0;  // ascending node order, engine.cpp:95-96 (two values per load)
      const double2* pb2 = reinterpret_cast<const double2*>(S.pb);
      for (int j = 0; j < (n >> 1); ++j) {
        const double2 x = pb2[j];
        tot += x.x;
        tot += x.y;
      }
      if (n & 1) tot += S.pb[n - 1];
      S.total = tot;
      const double delta = tot - s_cur_total;
      // mh_accept, sampler.cpp:54-56 (S.thr: host glibc log10(u) when A.thr, else u)
      S.acc = (uint8_t)(it == 0 || (A.thr ? S.thr < delta : mh_accept_dev(S.thr, delta, A.accept_tol, &S.amb)));
    }
    __syncthreads();
    // ---- commit in sequence (warp 0) up to and including the first acceptance
    if (warp == 0) {
      int committed = d;
      for (int i = 0; i < d; ++i)
        if (s_sl[i].acc) {
          committed = i + 1;
          break;
        }
      for (int i = 0; i < committed; ++i) {
        SpecSlot& S = s_sl[i];
        const uint64_t it = t + i;
        const bool acc = S.acc != 0;
        if (lane == 0 && S.amb) s_amb = 1;
        if (it == 0 || acc || !A.strict) {
          const uint64_t so = (uint64_t)c * A.K;
          if (!A.smasks)
            tracker_offer_warp<true>(A.tmasks + so * n, A.ttotals + so, A.thash + so, A.K, n, S.pm, S.total,
                                     &s_tcount, s_tcache);
          else if (!(s_tcount == A.K && S.total <= s_tcache[1]))
            tracker_insert_slots(A.smasks + so * n, A.stotals + so, A.shash + so, A.K, n, S.pm, S.total,
                                 &s_tcount, s_tord, &s_tcache[1], &s_tcache[0]);
        }
        if (lane == 0 && it > 0) {
          const uint64_t o = (uint64_t)c * A.iters + (it - 1);
          A.tr_prop[o] = S.total;
          A.tr_acc[o] = acc ? 1 : 0;
          A.tr_best[o] = s_tcache[0];
        }
        pairs += (unsigned long long)S.np;
      }
      SpecSlot& L = s_sl[committed - 1];
      if (L.acc) {
        for (int j = lane; j < n; j += 32) {
          s_cm[j] = L.pm[j];
          s_cb[j] = L.pb[j];
          s_order[j] = L.prop[j];
        }
        if (lane == 0) {
          uint64_t tn = s_tied;
          for (int q = 0; q < L.np; ++q) {
            const uint64_t bb = 1ull << L.pv[q];
            tn = L.pt[q] ? (tn | bb) : (tn & ~bb);
          }
          s_tied = tn;
          s_cur_total = L.total;
          if (t + committed - 1 > 0) ++s_acc;
        }
      }
      if (lane == 0) {
        s_rng = L.rng_after;
        s_arng = L.arng_after;
        s_done_to = committed;
      }
    }
    __syncthreads();
    t += s_done_to;
  }
  if (tid < n) A.final_order[(uint64_t)c * n + tid] = s_order[tid];
  if (A.smasks && warp == 0) {  // slot tracker -> tmasks/ttotals in order
    const uint64_t so = (uint64_t)c * A.K;
    for (int e = 0; e < s_tcount; ++e) {
      const uint64_t sl = s_tord[e];
      BNMC_FOR_NODES(i, lane, 32, n) A.tmasks[(so + e) * n + i] = A.smasks[(so + sl) * n + i];
      if (lane == 0) A.ttotals[so + e] = A.stotals[so + sl];
    }
  }
  if (tid == 0) {
    A.final_score[c] = s_cur_total;
    A.accepted[c] = s_acc;
    A.tcount[c] = s_tcount;
    if (A.ambiguous) A.ambiguous[c] = s_amb;
    if (A.stat) atomicAdd(A.stat, pairs);
  }
  if (lane == 0 && A.stat) {
    atomicAdd(A.stat + 1, walked);
    atomicAdd(A.stat + 2, enumerated);
  }
}

}  // namespace bnmc_dev
