// K3 — device-resident MCMC step (sm_100a): one CTA per chain.
//
// Restates run_mcmc's loop body (sampler.cpp:92-111) on the device:
//   read the argmax cell of every rescanned row (the K2 maxima; argmax_reduce,
//   engine.cpp:15-22, 85-93) -> proposed per-node bests and parent sets;
//   total in ascending node order (engine.cpp:95-96); mh_accept
//   (sampler.cpp:54-56) against the host-precomputed glibc log10(u_t) of the
//   acceptance stream; BestGraphTracker::update (sampler.cpp:32-41); commit;
//   trace row; then the next proposal's rescan pairs, bucketed by row for K2.
// Only rows at positions min(a,b)..max(a,b) of the proposed order change their
// predecessor sets, so only those are rescanned (the reference rescans all n,
// engine.cpp:71-76; the results are identical).
// The chain state is staged in shared memory; loops over nodes, tracker
// entries and positions are spread over the CTA's threads.
#pragma once

#include "scan.cuh"

namespace bnmc_dev {

struct ChainState {
  uint64_t iter;       // next iteration to finalize (0 = initial order scoring)
  uint64_t accepted;
  double total;        // current chain score
  int done;
  int tcount;          // tracker entries
  int a, b;            // pending proposal positions (-1 for the initial scoring)
  uint64_t tied;       // nodes whose current best is an exact fp64 tie
  uint8_t order[64];   // current order: order[pos] = node
  uint8_t prop[64];    // proposed order
  uint64_t masks[64];  // current graph (parent masks by node)
  double best[64];     // current per-node effective bests
};

struct Item {  // per-chain copy of its rescan pairs (slot -> row, predecessors)
  uint64_t cpred;
  uint32_t v, pad;
};

struct StepArgs {
  ChainState* st;           // [C]
  Item* items;              // [C][64]
  int* counts;              // [C]
  uint8_t* ppos;            // [C][64]
  PairRec* buckets;         // [2][n][kMaxChains]
  int* rowcnt;              // [2][n]
  int* sel;                 // bucket holding the next iteration's pairs
  unsigned long long* cell; // [C][n][2] argmax maxima from K2 (reset here)
  const float* keys;        // fp32 scan keys (exact tie resolution)
  uint64_t Sp;
  const uint8_t* props;     // [C][iters+1][2] proposal positions (a,b)
  const double* thr;        // [C][iters+1] log10(u_t) of the acceptance stream
  uint64_t* tmasks;         // [C][K][n] tracker graphs
  double* ttotals;          // [C][K]
  double* tr_prop;          // [C][iters]
  uint8_t* tr_acc;          // [C][iters]
  double* tr_best;          // [C][iters]
  unsigned long long* stat_rows;  // rows rescanned (sum over chains and iterations)
  int* error;               // internal-consistency flag
  uint64_t iters;
  int n, K, strict;
  int score_only;           // bnmc_gpu_score_orders: write graphs, no chain logic
  uint64_t* out_masks;      // score_only outputs [C][n]
  double* out_best;         // [C][n]
  double* out_total;        // [C]
  TieCtx tie;
};

constexpr int kStepThreads = 256;
constexpr int kTrackerSmem = 2048;  // u64 slots for staging tracker shifts

// Rescan pairs of the proposed order `prop`: positions lo..hi (their
// predecessor sets changed) plus positions after hi whose node's best is an
// exact tie (`tied`): their predecessor SET is unchanged, but the swapped
// nodes changed positions, and the reference breaks exact ties by the first
// maximum in predecessor-POSITION order (engine.cpp:52), so the chosen set can
// change. Written into bucket `nb` and the chain's own item list, plus the
// position table. Warp 0: prefix-OR of predecessor bits and slot prefix sums
// by shuffle.
__device__ void prepare_items_warp(const StepArgs& A, int c, const uint8_t* prop, int lo, int hi,
                                   uint64_t tied, int nb) {
  const int lane = threadIdx.x & 31;
  const int n = A.n;
  uint64_t bit[2], pre[2];
  bool take[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int p = 2 * lane + h;
    bit[h] = p < n ? 1ull << prop[p] : 0ull;
    take[h] = p < n && ((p >= lo && p <= hi) || (p > hi && (tied & bit[h])));
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
  const int total = __shfl_sync(0xffffffffu, cnt, 31);
  int slot = cnt - (int)take[0] - (int)take[1];
  pre[0] = incl & ~(bit[0] | bit[1]);
  pre[1] = pre[0] | bit[0];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int p = 2 * lane + h;
    if (p >= n) continue;
    const int v = prop[p];
    A.ppos[64 * c + v] = (uint8_t)p;
    if (!take[h]) continue;
    const uint64_t cpred = nodes_to_cand(pre[h], v);
    Item it;
    it.cpred = cpred;
    it.v = (uint32_t)v;
    it.pad = 0;
    A.items[64 * c + slot] = it;
    const int pos = atomicAdd(&A.rowcnt[nb * n + v], 1);
    PairRec pr;
    pr.cpred = cpred;
    pr.chain = (uint16_t)c;
    pr.slot = (uint16_t)slot;
    pr.v = (uint32_t)v;
    A.buckets[(nb * n + v) * kMaxChains + pos] = pr;
    ++slot;
  }
  if (lane == 0) A.counts[c] = total;
}

// Exact argmax of row v among admissible entries whose fp32 key has order
// image `okey` (the cells reported a key tie); *tied is set when another
// admissible entry has exactly the winner's fp64 value. Whole CTA; rare path.
__device__ uint32_t resolve_tie(const StepArgs& A, int v, uint64_t cpred, uint32_t okey,
                                const uint8_t* ppos, uint32_t* s_cand, int* tied) {
  uint32_t best = kNoIdx;
  const float* row = A.keys + (uint64_t)v * A.Sp;
  for (uint64_t g = threadIdx.x; g < A.tie.S; g += blockDim.x) {
    if (ordkey(row[g]) != okey) continue;
    if ((A.tie.cmask[g] & ~cpred) != 0) continue;
    if (best == kNoIdx || better_slow(A.tie, v, (uint32_t)g, best, ppos)) best = (uint32_t)g;
  }
  s_cand[threadIdx.x] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t w = kNoIdx;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      const uint32_t g = s_cand[i];
      if (g != kNoIdx && (w == kNoIdx || better_slow(A.tie, v, g, w, ppos))) w = g;
    }
    s_cand[0] = w;
  }
  __syncthreads();
  const uint32_t w = s_cand[0];
  const double ew = exact_eff(A.tie, v, w);
  int mine = 0;
  for (uint64_t g = threadIdx.x; g < A.tie.S; g += blockDim.x) {
    if (g == w || ordkey(row[g]) != okey) continue;
    if ((A.tie.cmask[g] & ~cpred) != 0) continue;
    mine |= exact_eff(A.tie, v, (uint32_t)g) == ew;
  }
  const int any = __syncthreads_or(mine);
  if (threadIdx.x == 0) *tied = any;
  __syncthreads();
  return w;
}

// BestGraphTracker::update (sampler.cpp:32-41) for one chain, whole CTA:
// dedupe by full graph equality, reject when full and total <= minimum,
// insert at lower_bound of (total desc, Dag operator< on the masks). tm/tt
// are the chain's K x n masks and K totals; pm is the offered graph (shared
// memory); *s_tcount the entry count (shared).
__device__ void tracker_offer(uint64_t* tm, double* tt, int K_, int n, const uint64_t* pm,
                              double proposed, int* s_tcount, int* s_go, uint64_t* s_stage,
                              int stage_cap = kTrackerSmem) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nthr = blockDim.x, nwarps = nthr >> 5;
  const int count = *s_tcount;
  const bool full = count == K_;
  // A full tracker rejects totals <= its minimum whether or not the graph is
  // a duplicate, so that test runs first.
  if (tid == 0) *s_go = !(full && proposed <= tt[count - 1]);
  __syncthreads();
  if (*s_go) {
    int dup_local = 0;
    for (int e = warp; e < count; e += nwarps) {
      bool eq = true;
      for (int i = lane; i < n; i += 32) eq &= tm[(uint64_t)e * n + i] == pm[i];
      dup_local |= __all_sync(0xffffffffu, eq);
    }
    if (!__syncthreads_or(dup_local)) {
      int ins = 0;
      for (int e0 = 0; e0 < count; e0 += nthr) {
        const int e = e0 + tid;
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
        ins += __syncthreads_count(prec);
      }
      const int last = full ? count - 1 : count;
      const int moving = last - ins;  // entries [ins, last) move down one slot
      if ((long long)moving * n <= stage_cap) {
        for (int idx = tid; idx < moving * n; idx += nthr) s_stage[idx] = tm[(uint64_t)ins * n + idx];
        __syncthreads();
        for (int idx = tid; idx < moving * n; idx += nthr) tm[(uint64_t)(ins + 1) * n + idx] = s_stage[idx];
      } else {
        for (int e = last; e > ins; --e) {
          for (int i = tid; i < n; i += nthr) tm[(uint64_t)e * n + i] = tm[(uint64_t)(e - 1) * n + i];
          __syncthreads();
        }
      }
      if (tid == 0)
        for (int e = last; e > ins; --e) tt[e] = tt[e - 1];
      __syncthreads();
      for (int i = tid; i < n; i += nthr) tm[(uint64_t)ins * n + i] = pm[i];
      if (tid == 0) {
        tt[ins] = proposed;
        if (!full) *s_tcount = count + 1;
      }
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kStepThreads) step_kernel(StepArgs A) {
  const int c = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5;
  __shared__ uint64_t s_pm[64];
  __shared__ double s_pb[64];
  __shared__ uint8_t s_order[64], s_prop[64], s_ppos[64];
  __shared__ Item s_item[64];
  __shared__ uint32_t s_g[64];
  __shared__ uint32_t s_key[64];
  __shared__ int s_tie[64];
  __shared__ double s_total, s_cur_total;
  __shared__ int s_cnt, s_done, s_tcount, s_go, s_anytie, s_tflag;
  __shared__ uint64_t s_iter, s_tied, s_tied_new;
  __shared__ uint64_t s_stage[kTrackerSmem];
  __shared__ uint32_t s_cand[kStepThreads];
  cudaGridDependencySynchronize();
  ChainState* st = A.st + c;
  const int n = A.n;
  if (tid == 0) {
    s_cnt = A.counts[c];
    s_anytie = 0;
    if (A.score_only) {
      s_done = 0;
    } else {
      s_done = st->done;
      s_iter = st->iter;
      s_cur_total = st->total;
      s_tcount = st->tcount;
      s_tied = st->tied;
    }
  }
  if (tid < 64) {
    s_ppos[tid] = A.ppos[64 * c + tid];
    s_item[tid] = A.items[64 * c + tid];
    if (!A.score_only && tid < n) {
      s_prop[tid] = st->prop[tid];
      s_pm[tid] = st->masks[tid];
      s_pb[tid] = st->best[tid];
      s_order[tid] = st->order[tid];
    }
  }
  __syncthreads();
  // Bucket housekeeping for the next scan (CTA 0): the bucket that this
  // iteration's scan read is cleared; `sel` points at the one filled below.
  if (!A.score_only && c == 0 && tid < n) {
    const int nb = s_done ? *A.sel : (int)(s_iter & 1);
    A.rowcnt[(1 - nb) * n + tid] = 0;
    if (s_done) A.rowcnt[nb * n + tid] = 0;
    if (tid == 0) *A.sel = nb;
  }
  if (s_done) return;
  const int cnt = s_cnt;
  // 1. the argmax cell of every rescanned row; reset the cells.
  if (tid < cnt) {
    unsigned long long* cell = A.cell + 2ull * (c * n + tid);
    const unsigned long long hi = cell[0], lo = cell[1];
    cell[0] = 0ull;
    cell[1] = 0ull;
    const uint32_t g1 = (uint32_t)hi, g2 = ~(uint32_t)lo;
    s_key[tid] = (uint32_t)(hi >> 32);
    s_g[tid] = g1;
    s_tie[tid] = g1 != g2;
    if (hi == 0ull) atomicExch(A.error, 3);  // every row admits the empty set
    if (g1 != g2) s_anytie = 1;
  }
  __syncthreads();
  if (s_anytie) {
    for (int s = 0; s < cnt; ++s)
      if (s_tie[s]) {
        const uint32_t g =
            resolve_tie(A, s_item[s].v, s_item[s].cpred, s_key[s], s_ppos, s_cand, &s_tflag);
        if (tid == 0) {
          s_g[s] = g;
          s_tie[s] = s_tflag;  // now: exact fp64 tie at the maximum
        }
      }
    __syncthreads();
  }
  // Exact-tie status of the proposed graph: rescanned rows take their fresh
  // status (a unique fp32 maximum is a unique fp64 maximum), others keep theirs.
  if (tid == 0 && !A.score_only) {
    uint64_t tnew = s_tied;
    for (int s = 0; s < cnt; ++s) {
      const uint64_t b = 1ull << s_item[s].v;
      tnew = s_tie[s] ? (tnew | b) : (tnew & ~b);
    }
    s_tied_new = tnew;
  }
  if (tid < cnt) {
    const int v = s_item[tid].v;
    const uint32_t g = s_g[tid];
    const uint64_t nm = cand_to_nodes(A.tie.cmask[g], v);
    s_pm[v] = nm;
    s_pb[v] = A.tie.ls[(uint64_t)v * A.tie.S + g] + ppf_sum(A.tie.w, n, v, nm);
  }
  __syncthreads();
  // 2. proposed total, ascending node order (engine.cpp:95-96).
  if (tid == 0) {
    double t = 0.0;
    for (int i = 0; i < n; ++i) t += s_pb[i];
    s_total = t;
  }
  __syncthreads();
  if (A.score_only) {
    if (tid < n) {
      if (A.out_masks) A.out_masks[(uint64_t)c * n + tid] = s_pm[tid];
      if (A.out_best) A.out_best[(uint64_t)c * n + tid] = s_pb[tid];
    }
    if (tid == 0 && A.out_total) A.out_total[c] = s_total;
    return;
  }
  const uint64_t t = s_iter;
  const double proposed = s_total;
  // mh_accept (sampler.cpp:54-56): log10(u) < new - old; the initial order is
  // adopted as the current state without a draw.
  const bool accepted = t == 0 ? true : (A.thr[c * (A.iters + 1) + t] < proposed - s_cur_total);
  // 3. BestGraphTracker::update (sampler.cpp:32-41).
  const bool offer = (t == 0) || accepted || !A.strict;
  double* tt = A.ttotals + (uint64_t)c * A.K;
  if (offer)
    tracker_offer(A.tmasks + (uint64_t)c * A.K * n, A.ttotals + (uint64_t)c * A.K, A.K, n, s_pm,
                  proposed, &s_tcount, &s_go, s_stage);
  // 4. commit + trace + next proposal.
  if (accepted && tid < n) {
    st->masks[tid] = s_pm[tid];
    st->best[tid] = s_pb[tid];
    st->order[tid] = s_prop[tid];
    s_order[tid] = s_prop[tid];
  }
  if (tid == 0) {
    if (accepted) {
      st->total = proposed;
      st->tied = s_tied_new;
      s_tied = s_tied_new;
      if (t > 0) st->accepted += 1;
    }
    st->tcount = s_tcount;
    if (t > 0) {
      const uint64_t o = (uint64_t)c * A.iters + (t - 1);
      A.tr_prop[o] = proposed;
      A.tr_acc[o] = accepted ? 1 : 0;
      A.tr_best[o] = tt[0];
    }
    atomicAdd(A.stat_rows, (unsigned long long)cnt);
    st->iter = t + 1;
  }
  __syncthreads();
  const uint64_t nt = t + 1;
  if (nt > A.iters) {
    if (tid == 0) {
      st->done = 1;
      A.counts[c] = 0;
    }
    return;
  }
  // propose_swap (sampler.cpp:43-52): positions drawn by the setup kernel.
  const int pa = A.props[2 * (c * (A.iters + 1) + nt)];
  const int pb = A.props[2 * (c * (A.iters + 1) + nt) + 1];
  if (tid < n) {
    const int src = tid == pa ? pb : (tid == pb ? pa : tid);
    s_prop[tid] = s_order[src];
    st->prop[tid] = s_order[src];
  }
  if (tid == 0) {
    st->a = pa;
    st->b = pb;
  }
  __syncthreads();
  if (warp == 0) prepare_items_warp(A, c, s_prop, min(pa, pb), max(pa, pb), s_tied, (int)(t & 1));
}

// Setup (one thread per chain): initial order = shuffle of the split(1)
// stream (sampler.cpp:83-86), proposal positions of every iteration from the
// split(2) stream (propose_swap, sampler.cpp:43-52; the proposal stream does
// not depend on acceptance).
__global__ void setup_chains_kernel(StepArgs A, const uint64_t* __restrict__ seeds, int C) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const int n = A.n;
  const Rng master{seeds[c]};
  Rng init = master.split(1);
  Rng prop = master.split(2);
  ChainState* st = A.st + c;
  uint8_t order[64];
  for (int i = 0; i < n; ++i) order[i] = (uint8_t)i;
  for (int i = n; i > 1; --i) {
    const int j = (int)init.next_below((uint64_t)i);
    const uint8_t tmp = order[i - 1];
    order[i - 1] = order[j];
    order[j] = tmp;
  }
  st->iter = 0;
  st->accepted = 0;
  st->total = 0.0;
  st->done = 0;
  st->tcount = 0;
  st->a = st->b = -1;
  st->tied = 0;
  for (int i = 0; i < 64; ++i) {
    st->order[i] = i < n ? order[i] : 0;
    st->prop[i] = i < n ? order[i] : 0;
    st->masks[i] = 0;
    st->best[i] = 0.0;
  }
  uint8_t* pp = const_cast<uint8_t*>(A.props) + 2ull * c * (A.iters + 1);
  pp[0] = pp[1] = 0;
  for (uint64_t t = 1; t <= A.iters; ++t) {
    const int a = (int)prop.next_below((uint64_t)n);
    int b = (int)prop.next_below((uint64_t)(n - 1));
    if (b >= a) ++b;
    pp[2 * t] = (uint8_t)a;
    pp[2 * t + 1] = (uint8_t)b;
  }
}

// Initial pairs (every row of each order) into bucket 1; sel = 1. One CTA of
// 64 threads per order. The buckets' counters and the cells must be zero.
__global__ void setup_items_kernel(StepArgs A, const int* __restrict__ perms, int C) {
  const int c = blockIdx.x;
  __shared__ uint8_t s_prop[64];
  if (threadIdx.x < A.n)
    s_prop[threadIdx.x] =
        perms ? (uint8_t)perms[(uint64_t)c * A.n + threadIdx.x] : A.st[c].order[threadIdx.x];
  __syncthreads();
  if (threadIdx.x < 32) prepare_items_warp(A, c, s_prop, 0, A.n - 1, 0ull, 1);
  if (c == 0 && threadIdx.x == 0) *A.sel = 1;
}

// Diagnostics: pairs for positions lo..hi of each order (bnmc_gpu_bench_scan).
__global__ void setup_items_range_kernel(StepArgs A, const int* __restrict__ perms, int C, int lo,
                                         int hi) {
  const int c = blockIdx.x;
  __shared__ uint8_t s_prop[64];
  if (threadIdx.x < A.n) s_prop[threadIdx.x] = (uint8_t)perms[(uint64_t)c * A.n + threadIdx.x];
  __syncthreads();
  if (threadIdx.x < 32) prepare_items_warp(A, c, s_prop, lo, hi, 0ull, 1);
  if (c == 0 && threadIdx.x == 0) *A.sel = 1;
}

}  // namespace bnmc_dev
