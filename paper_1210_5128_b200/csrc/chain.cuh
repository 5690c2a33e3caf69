// K3 — device-resident MCMC step (sm_100a): one CTA per chain.
//
// Restates run_mcmc's loop body (sampler.cpp:92-111) on the device:
//   reduce the K2 partial cells of every rescanned row (argmax_reduce,
//   engine.cpp:15-22, 85-93) -> proposed per-node bests and parent sets;
//   total in ascending node order (engine.cpp:95-96); mh_accept
//   (sampler.cpp:54-56) against the host-precomputed glibc log10(u_t) of the
//   acceptance stream; BestGraphTracker::update (sampler.cpp:32-41); commit;
//   trace row; then prepare the next proposal's rescan items.
// Only rows at positions min(a,b)..max(a,b) of the proposed order change their
// predecessor sets, so only those are rescanned (the reference rescans all n,
// engine.cpp:71-76; results are identical).
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
  uint8_t order[64];   // current order: order[pos] = node
  uint8_t prop[64];    // proposed order
  uint64_t masks[64];  // current graph (parent masks by node)
  double best[64];     // current per-node effective bests
};

struct StepArgs {
  ChainState* st;           // [C]
  Item* items;              // [C][n]
  int* counts;              // [C]
  uint8_t* ppos;            // [C][64]
  const void* partials;     // [C][n][G]
  const uint8_t* props;     // [C][iters+1][2] proposal positions (a,b)
  const double* thr;        // [C][iters+1] log10(u_t) of the acceptance stream
  uint64_t* tmasks;         // [C][K][n] tracker graphs
  double* ttotals;          // [C][K]
  double* tr_prop;          // [C][iters]
  uint8_t* tr_acc;          // [C][iters]
  double* tr_best;          // [C][iters]
  unsigned long long* stat_rows;  // rows rescanned (sum)
  uint64_t iters;
  int n, G, K, strict;
  int score_only;           // bnmc_gpu_score_orders: write graphs, no chain logic
  uint64_t* out_masks;      // score_only outputs [C][n]
  double* out_best;         // [C][n]
  double* out_total;        // [C]
  TieCtx tie;
};

// precedes (sampler.cpp:16-19): total desc, then Dag operator< (lexicographic
// over the parent masks, types.hpp:140-142).
__device__ __forceinline__ bool dag_less(const uint64_t* a, const uint64_t* b, int n) {
  for (int i = 0; i < n; ++i)
    if (a[i] != b[i]) return a[i] < b[i];
  return false;
}

// Prepare the rescan items of the proposed order `prop` for positions lo..hi.
__device__ void prepare_items(const StepArgs& A, int c, const uint8_t* prop, int lo, int hi) {
  uint64_t pred = 0;
  Item* items = A.items + (uint64_t)c * A.n;
  for (int p = 0; p < hi + 1; ++p) {
    const int v = prop[p];
    if (p >= lo) {
      Item it;
      it.cpred = nodes_to_cand(pred, v);
      it.v = (uint32_t)v;
      it.pad = 0;
      items[p - lo] = it;
    }
    pred |= 1ull << v;
  }
  for (int p = 0; p < A.n; ++p) A.ppos[64 * c + prop[p]] = (uint8_t)p;
  A.counts[c] = hi - lo + 1;
}

template <typename K>
__global__ void __launch_bounds__(256) step_kernel(StepArgs A) {
  const int c = blockIdx.x;
  ChainState* st = A.st + c;
  __shared__ uint64_t s_newm[64];
  __shared__ double s_newb[64];
  __shared__ uint64_t s_pm[64];
  __shared__ double s_pb[64];
  __shared__ uint8_t s_prop[64];
  __shared__ uint8_t s_ppos[64];
  __shared__ int s_v[64];
  __shared__ double s_total;
  __shared__ int s_insert, s_dup;
  if (!A.score_only && st->done) return;
  const int n = A.n;
  const int cnt = A.counts[c];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < 64) {
    if (!A.score_only) s_prop[threadIdx.x] = st->prop[threadIdx.x];
    s_ppos[threadIdx.x] = A.ppos[64 * c + threadIdx.x];
  }
  __syncthreads();
  const Partial<K>* parts = static_cast<const Partial<K>*>(A.partials);
  // 1. argmax_reduce over the G CTA cells of every rescanned row.
  for (int s = warp; s < cnt; s += blockDim.x >> 5) {
    const int v = A.items[(uint64_t)c * n + s].v;
    K k = (K)-INFINITY;
    uint32_t g = kNoIdx;
    for (int b = lane; b < A.G; b += 32) {
      const Partial<K> p = parts[((uint64_t)c * n + s) * A.G + b];
      if (better<K>(A.tie, v, p.k, p.g, k, g, s_ppos)) {
        k = p.k;
        g = p.g;
      }
    }
    warp_argmax<K>(A.tie, v, k, g, s_ppos);
    if (lane == 0) {
      const uint64_t nm = cand_to_nodes(A.tie.cmask[g], v);
      s_newm[s] = nm;
      s_newb[s] = A.tie.ls[(uint64_t)v * A.tie.S + g] + ppf_sum(A.tie.w, n, v, nm);
      s_v[s] = v;
    }
  }
  __syncthreads();
  // 2. proposed graph and total (ascending node order, engine.cpp:95-96).
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) {  // score_only: every row is rescanned below
      s_pm[i] = A.score_only ? 0ull : st->masks[i];
      s_pb[i] = A.score_only ? 0.0 : st->best[i];
    }
    for (int s = 0; s < cnt; ++s) {
      s_pm[s_v[s]] = s_newm[s];
      s_pb[s_v[s]] = s_newb[s];
    }
    double t = 0.0;
    for (int i = 0; i < n; ++i) t += s_pb[i];
    s_total = t;
  }
  __syncthreads();
  if (A.score_only) {
    if (threadIdx.x < n) {
      if (A.out_masks) A.out_masks[(uint64_t)c * n + threadIdx.x] = s_pm[threadIdx.x];
      if (A.out_best) A.out_best[(uint64_t)c * n + threadIdx.x] = s_pb[threadIdx.x];
    }
    if (threadIdx.x == 0 && A.out_total) A.out_total[c] = s_total;
    return;
  }
  const uint64_t t = st->iter;
  const double proposed = s_total;
  bool accepted;
  if (t == 0) {
    accepted = true;  // initial order: becomes the current state
  } else {
    // mh_accept (sampler.cpp:54-56): log10(u) < new - old
    accepted = A.thr[c * (A.iters + 1) + t] < proposed - st->total;
  }
  // 3. BestGraphTracker::update (sampler.cpp:32-41), warp 0.
  const bool offer = (t == 0) || accepted || !A.strict;
  if (warp == 0 && offer) {
    const int K_ = A.K;
    uint64_t* tm = A.tmasks + (uint64_t)c * K_ * n;
    double* tt = A.ttotals + (uint64_t)c * K_;
    const int count = st->tcount;
    const bool full = count == K_;
    // A full tracker rejects totals <= its minimum whether or not the graph
    // is a duplicate, so that test may run first.
    bool go = !(full && proposed <= tt[count - 1]);
    if (go) {
      if (lane == 0) s_dup = 0;
      __syncwarp();
      for (int e = lane; e < count; e += 32) {
        bool eq = true;
        for (int i = 0; i < n && eq; ++i) eq = tm[(uint64_t)e * n + i] == s_pm[i];
        if (eq) s_dup = 1;
      }
      __syncwarp();
      go = !s_dup;
    }
    if (go) {
      // lower_bound with `precedes`: first entry that does not precede g.
      if (lane == 0) {
        int pos = 0;
        while (pos < count) {
          const double et = tt[pos];
          const bool prec = (et != proposed) ? (et > proposed)
                                             : dag_less(tm + (uint64_t)pos * n, s_pm, n);
          if (!prec) break;
          ++pos;
        }
        s_insert = pos;
      }
      __syncwarp();
      const int pos = s_insert;
      const int last = full ? count - 1 : count;
      for (int e = last; e > pos; --e) {
        for (int i = lane; i < n; i += 32) tm[(uint64_t)e * n + i] = tm[(uint64_t)(e - 1) * n + i];
        if (lane == 0) tt[e] = tt[e - 1];
        __syncwarp();
      }
      for (int i = lane; i < n; i += 32) tm[(uint64_t)pos * n + i] = s_pm[i];
      if (lane == 0) {
        tt[pos] = proposed;
        if (!full) st->tcount = count + 1;
      }
    }
  }
  __syncthreads();
  // 4. commit + trace + next proposal.
  if (threadIdx.x == 0) {
    if (accepted) {
      for (int i = 0; i < n; ++i) {
        st->masks[i] = s_pm[i];
        st->best[i] = s_pb[i];
        st->order[i] = s_prop[i];
      }
      st->total = proposed;
      if (t > 0) st->accepted += 1;
    }
    if (t > 0) {
      const uint64_t o = (uint64_t)c * A.iters + (t - 1);
      A.tr_prop[o] = proposed;
      A.tr_acc[o] = accepted ? 1 : 0;
      A.tr_best[o] = A.ttotals[(uint64_t)c * A.K];
    }
    atomicAdd(A.stat_rows, (unsigned long long)cnt);
    const uint64_t nt = t + 1;
    st->iter = nt;
    if (nt > A.iters) {
      st->done = 1;
      A.counts[c] = 0;
    } else {
      // propose_swap (sampler.cpp:43-52): positions drawn by the setup kernel.
      const int pa = A.props[2 * (c * (A.iters + 1) + nt)];
      const int pb = A.props[2 * (c * (A.iters + 1) + nt) + 1];
      uint8_t* prop = st->prop;
      for (int i = 0; i < n; ++i) prop[i] = st->order[i];
      const uint8_t tmp = prop[pa];
      prop[pa] = prop[pb];
      prop[pb] = tmp;
      st->a = pa;
      st->b = pb;
      prepare_items(A, c, prop, min(pa, pb), max(pa, pb));
    }
  }
}

// Setup (one thread per chain): initial order = shuffle of the split(1)
// stream (sampler.cpp:83-86), proposal positions of every iteration from the
// split(2) stream (propose_swap, sampler.cpp:43-52; the proposal stream does
// not depend on acceptance), initial items = every row of the initial order.
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
  prepare_items(A, c, order, 0, n - 1);
}

// Setup for bnmc_gpu_score_orders: items = every row of each given order.
__global__ void setup_orders_kernel(StepArgs A, const int* __restrict__ perms, int C) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  uint8_t order[64];
  for (int i = 0; i < A.n; ++i) order[i] = (uint8_t)perms[(uint64_t)c * A.n + i];
  prepare_items(A, c, order, 0, A.n - 1);
}

}  // namespace bnmc_dev
