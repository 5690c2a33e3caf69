// bnmc_gpu.cu — C-ABI (include/bnmc_gpu.h) over the sm_100a kernels.
//
// Device layout of a table:
//   d_cmask[Sp]      u64 candidate-position mask of global index g, shared by
//                    every row (global_index order, combinatorics.cpp:61-76);
//                    padding entries = ~0 (never admissible)
//   d_ls[n][S]       fp64 local scores, BNSC body order (scoring.cpp:194-238)
//   d_key32[n][Sp]   fp32 scan keys fl32(ls + PpfTable::sum), padding -inf
//   d_w[n][n]        PPF weights (scoring.cpp:150-155)
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/bnmc_gpu.h"
#include <cub/device/device_radix_sort.cuh>

#include "chain.cuh"
#include "walk.cuh"
#include "common.cuh"
#include "host_util.hpp"
#include "precompute.cuh"
#include "nccl_dyn.hpp"

using namespace bnmc_dev;
using bnmc_host::raise;
using bnmc_host::Status;
using bnmc_host::cuda_check;
using bnmc_host::precompute;
using bnmc_host::K1Range;
using bnmc_host::K1Report;
using bnmc_host::count_statistics_device;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return BNMC_OK;
  } catch (const Status& s) {
    g_err = s.msg;
    return s.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return BNMC_CAPACITY;
  } catch (const std::exception& e) {
    g_err = e.what();
    return BNMC_ERR;
  }
}

uint64_t h_binom[65][65];
bool h_binom_ready = false;
void host_binom_init() {
  if (h_binom_ready) return;
  for (int n = 0; n <= 64; ++n) {
    h_binom[n][0] = 1;
    for (int k = 1; k <= n; ++k) h_binom[n][k] = h_binom[n - 1][k - 1] + h_binom[n - 1][k];
    for (int k = n + 1; k <= 64; ++k) h_binom[n][k] = 0;
  }
  h_binom_ready = true;
}
uint64_t hbinom(int n, int k) {
  host_binom_init();
  return (k < 0 || n < 0 || k > n) ? 0 : h_binom[n][k];
}
uint64_t bounded_count(int c, int s) {
  uint64_t t = 0;
  for (int j = 0; j <= s; ++j) t += hbinom(c, j);
  return t;
}

// One-time per device: binomial table into constant memory; sm_100 check.
void ensure_device(int dev) {
  int count = 0;
  CK(cudaGetDeviceCount(&count));
  if (dev < 0 || dev >= count)
    raise(BNMC_CUDA, "CUDA device " + std::to_string(dev) + " not available (" +
                         std::to_string(count) + " visible)");
  CK(cudaSetDevice(dev));
  static bool ready[64] = {false};
  if (!ready[dev]) {
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, dev));
    if (p.major != 10)
      raise(BNMC_CUDA, std::string("bnmc_gpu is built for sm_100a (B200); device is ") + p.name);
    host_binom_init();
    CK(cudaMemcpyToSymbol(c_binom, h_binom, sizeof(h_binom)));
    ready[dev] = true;
  }
}

void validate_params(const bnmc_score_params* p) {
  if (!p) raise(BNMC_USAGE, "null score params");
  // RunConfig::validate (types.cpp:111-121), scoring fields
  if (p->max_parents < 0 || p->max_parents > 8) raise(BNMC_USAGE, "max-parents must lie in [0,8]");
  if (!(p->gamma > 0.0 && p->gamma <= 1.0)) raise(BNMC_USAGE, "gamma must lie in (0,1]");
  if (!(p->ess > 0.0)) raise(BNMC_USAGE, "ess must be positive");
  if (p->alpha_mode != BNMC_ALPHA_BDEU && p->alpha_mode != BNMC_ALPHA_K2)
    raise(BNMC_USAGE, "alpha_mode must be BDeu (0) or K2 (1)");
  if (p->n_gpus < 0 || p->n_gpus > 64) raise(BNMC_USAGE, "n_gpus must lie in [0,64]");
}

// ppf (scoring.cpp:143-148) and PpfTable (scoring.cpp:150-155).
std::vector<double> ppf_weights(const double* r, int n) {
  std::vector<double> w(static_cast<size_t>(n) * n, 0.0);
  if (!r) return w;
  for (int i = 0; i < n * n; ++i)
    if (!(r[i] >= 0.0 && r[i] <= 1.0)) raise(BNMC_DATA, "prior matrix entries must lie in [0,1]");
  for (int i = 0; i < n; ++i)
    for (int m = 0; m < n; ++m)
      if (i != m) {
        const double d = r[i * n + m] - 0.5;
        w[i * n + m] = 100.0 * d * d * d;
      }
  return w;
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  void alloc(size_t count) {
    if (count <= n && p) return;
    release();
    if (count == 0) return;
    cuda_check(cudaMalloc(&p, count * sizeof(T)), "cudaMalloc");
    n = count;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { release(); }
};

}  // namespace

// One rank of a multi-process NCCL communicator (bnmc_gpu_comm_init).
struct bnmc_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1, dev = 0;
  cudaStream_t stream = nullptr;
  ~bnmc_comm() {
    if (comm) bnmc_host::nccl().CommDestroy(comm);
    if (stream) cudaStreamDestroy(stream);
  }
};

static uint64_t env_u64(const char* name, uint64_t dflt) {
  const char* e = std::getenv(name);
  return e && *e ? std::strtoull(e, nullptr, 10) : dflt;
}

struct bnmc_table {
  int dev = 0;
  int n = 0, s = 0;
  uint64_t S = 0, Sp = 0;
  double gamma = 0.1, ess = 1.0;
  int alpha = 0;
  cudaStream_t stream = nullptr;
  DevBuf<uint64_t> cmask;
  DevBuf<double> ls;
  DevBuf<float> key32;
  DevBuf<double> w;
  std::vector<double> h_w;
  // sorted rows for the walk path (K2W): eff desc + candidate masks, built
  // lazily after the priors are folded; PST of small predecessor counts.
  // Sorted entries are 16-byte (eff bits, candidate mask) pairs: one 128-bit
  // load per entry and lane in the walk.
  DevBuf<ulonglong2> srow;  // [n][Sw]
  DevBuf<double> eff;  // eff = ls + PpfTable::sum in global-index order
  uint64_t Sw = 0;     // sorted row stride
  DevBuf<ulonglong2> yrow;  // delta-walk lists [n][n-1][Syw]
  uint64_t Sy = 0, Syw = 0;
  bool ylists = false;
  // exclusion lists: row v's sorted entries without its strongest parent
  // (candidate bit xbit[v]); walked instead of the row when that parent is
  // not a predecessor [n][Sxw]
  // level j = 1..xlev excludes the row's j strongest parents (nested)
  DevBuf<ulonglong2> xrow;
  DevBuf<uint64_t> xbit;  // [n][kXLevels] candidate bits of the strongest parents
  uint64_t Sx[kXLevels + 1] = {}, Sxw[kXLevels + 1] = {}, xoff[kXLevels + 1] = {};
  int xlev = 0;
  int ylist_mode = -1;  // -1 auto (when they fit), 0 off, 1 on
  bool sorted_valid = false;
  float sort_ms = 0.f;
  DevBuf<uint64_t> pst;
  DevBuf<uint32_t> pst_off;
  DevBuf<uint64_t> pst2;
  DevBuf<uint32_t> pst2_off;
  int pe = -1;
  int pc = -1;  // rows with S(p,s) <= walk_cap: capped walk, then enumeration
  bool pst_ready = false;
  uint64_t enum_max = kEnumMax;  // enumerate rows with S(p,s) <= enum_max, walk the others
  uint64_t walk_cap = env_u64("BNMC_WALK_CAP", 0);  // 0: S(n-1,s) / kWalkCapDiv
  uint32_t walk_budget = static_cast<uint32_t>(env_u64("BNMC_WALK_BUDGET", kWalkBudget));
  int walk_deep = -1;  // 8 entries per lane per deep walk round: -1 auto (long rows), 0 off, 1 on
  int scan_mode = 0;  // default for score_orders: 0 auto (walk), 1 full-row scan
  DevBuf<int> d_fo, d_tc;
  DevBuf<unsigned long long> d_acc;
  DevBuf<double> d_fs;
  float build_ms = 0.f, fold_ms = 0.f;
  uint64_t wide_entries = 0, p_lo = 0, p_hi = 0;  // last K1 run (stats)
  // chain / order-scoring workspace
  DevBuf<ChainState> st;
  DevBuf<Item> items;
  DevBuf<int> counts;
  DevBuf<uint8_t> ppos;
  DevBuf<PairRec> buckets;
  DevBuf<int> rowcnt;
  DevBuf<unsigned long long> cell;
  DevBuf<uint8_t> props;
  DevBuf<double> thr;
  DevBuf<uint64_t> tmasks;
  DevBuf<double> ttotals;
  DevBuf<uint64_t> thash;
  DevBuf<uint64_t> smasks, shash;  // slot tracker storage (track_top <= kTrackSlots)
  DevBuf<double> stotals;
  DevBuf<double> tr_prop, tr_best;
  DevBuf<uint8_t> tr_acc;
  DevBuf<unsigned long long> stat;
  DevBuf<uint64_t> seeds;
  DevBuf<int> perms;
  DevBuf<uint64_t> out_masks;
  DevBuf<double> out_best, out_total;
  uint64_t last_rescans = 0, last_sectors = 0, last_launches = 0, last_scan_samples = 0;
  uint64_t last_walked = 0, last_enumerated = 0;
  int last_team = 0, last_wu = 0, last_spec = 0;
  uint64_t last_replayed = 0;
  uint64_t last_drift_it = 0;  // debug_recheck: first iteration whose rescore differed
  DevBuf<int> d_amb;
  float last_scan_ms = 0.f, last_total_ms = 0.f;
  int last_G = 0;
  // Multi-GPU table (n_gpus > 1): full replicas on the other devices, owned.
  std::vector<bnmc_table*> replicas;
  cudaStream_t stream2 = nullptr;  // second launch stream of pipelined chain blocks
  ~bnmc_table() {
    for (bnmc_table* r : replicas) {
      cudaSetDevice(r->dev);
      delete r;
    }
    cudaSetDevice(dev);
    if (stream2) cudaStreamDestroy(stream2);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

constexpr int kMaxChainsPerLaunch = 64;

struct ScanGeom {
  int G, sectors;
};

// K2 (scan2_kernel): CTA (x, y) owns kScan2Threads x kScan2Per consecutive
// global indices of the step's rows y, y + 8, ...
ScanGeom scan_geometry(const bnmc_table* t, int max_pairs) {
  ScanGeom g;
  (void)max_pairs;
  g.sectors = static_cast<int>(t->Sp / 8);
  const uint64_t slots = (static_cast<uint64_t>(g.sectors) * 8 + kScan2Per - 1) / kScan2Per;
  g.G = static_cast<int>((slots + kScan2Threads - 1) / kScan2Threads);
  return g;
}

void launch_scan(const ScanGeom& g, ScanArgs a, int max_pairs, cudaStream_t s, bool pdl) {
  a.sectors = g.sectors;
  (void)max_pairs;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(g.G, kScan2RowGroups);
  cfg.blockDim = dim3(kScan2Threads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, scan2_kernel, a));
}

void launch_step(int C, const StepArgs& A, cudaStream_t s, bool pdl) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kStepThreads);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, step_kernel, A));
}

// Candidate masks in global-index order (device unrank, combinatorics.cpp:8-39,
// 78-90): sizes s..0, lexicographic within a size.
__global__ void build_cmask_kernel(uint64_t* out, uint64_t S, uint64_t Sp, int c, int s) {
  const uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (g >= Sp) return;
  if (g >= S) {
    out[g] = ~0ull;
    return;
  }
  uint64_t r = g;
  int k = s < c ? s : c;
  for (; k >= 0; --k) {
    const uint64_t block = binom(c, k);
    if (r < block) break;
    r -= block;
  }
  uint64_t mask = 0;
  int x = 0;
  for (int i = 0; i < k; ++i) {
    for (;;) {
      const uint64_t cnt = binom(c - x - 1, k - i - 1);
      if (r < cnt) {
        mask |= 1ull << x;
        ++x;
        break;
      }
      r -= cnt;
      ++x;
    }
  }
  out[g] = mask;
}

// PPF fold: key = fl(ls + PpfTable::sum) in the scan's association
// (engine.cpp:50-51) rounded to fp32; padding -inf.
__global__ void fold_kernel(const double* __restrict__ ls, const uint64_t* __restrict__ cmask,
                            const double* __restrict__ w, float* key32, int n,
                            uint64_t S, uint64_t Sp) {
  const int v = blockIdx.y;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < Sp;
       g += (uint64_t)gridDim.x * blockDim.x) {
    double e = -INFINITY;
    if (g < S) e = ls[(uint64_t)v * S + g] + ppf_sum(w, n, v, cand_to_nodes(cmask[g], v));
    key32[(uint64_t)v * Sp + g] = __double2float_rn(e);
  }
}

void table_init(bnmc_table* t, int n, const bnmc_score_params* p) {
  validate_params(p);
  if (n < 1 || n > 64) raise(BNMC_DATA, "dataset must have between 1 and 64 variables");
  ensure_device(p->device);
  t->dev = p->device;
  t->n = n;
  t->s = p->max_parents;
  t->gamma = p->gamma;
  t->ess = p->ess;
  t->alpha = p->alpha_mode;
  t->S = bounded_count(n - 1, t->s);
  t->Sp = (t->S + 31) / 32 * 32;
  const uint64_t est = static_cast<uint64_t>(n) * t->S * 8;  // estimate_bytes
  if (est > p->memory_cap_bytes)
    raise(BNMC_CAPACITY, "score cache estimate " + std::to_string(est) +
                             " bytes exceeds cap of " + std::to_string(p->memory_cap_bytes));
  CK(cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking));
  t->cmask.alloc(t->Sp);
  t->ls.alloc(static_cast<size_t>(n) * t->S);
  t->key32.alloc(static_cast<size_t>(n) * t->Sp);
  t->w.alloc(static_cast<size_t>(n) * n);
  const unsigned blocks = static_cast<unsigned>((t->Sp + 255) / 256);
  build_cmask_kernel<<<blocks, 256, 0, t->stream>>>(t->cmask.p, t->S, t->Sp, n - 1, t->s);
  CK(cudaGetLastError());
}

void set_priors(bnmc_table* t, const double* prior_r) {
  t->h_w = ppf_weights(prior_r, t->n);
  CK(cudaMemcpyAsync(t->w.p, t->h_w.data(), t->h_w.size() * 8, cudaMemcpyHostToDevice, t->stream));
}

void fold(bnmc_table* t) {
  t->sorted_valid = false;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const unsigned bx = static_cast<unsigned>(std::min<uint64_t>((t->Sp + 255) / 256, 4096));
  CK(cudaEventRecord(e0, t->stream));
  fold_kernel<<<dim3(bx, t->n), 256, 0, t->stream>>>(t->ls.p, t->cmask.p, t->w.p, t->key32.p,
                                                       t->n, t->S,
                                                       t->Sp);
  CK(cudaGetLastError());
  CK(cudaEventRecord(e1, t->stream));
  CK(cudaEventSynchronize(e1));
  CK(cudaEventElapsedTime(&t->fold_ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

// OrderScorer::scan_slice (engine.cpp:43-58) on the device: PST index g of
// the node at `position` is the global-index subset of POSITIONS 0..p-1
// (subset_at, combinatorics.cpp:78-90) mapped through the order
// (apply_candidates), looked up in the node's row (index_of) plus
// PpfTable::sum. The reference keeps the first maximum in ascending g; the
// (score desc, g asc) reduction below selects the same entry. One CTA.
constexpr int kSliceThreads = 512;
__global__ void __launch_bounds__(kSliceThreads)
    slice_kernel(const double* __restrict__ ls, const double* __restrict__ w, uint64_t S, int n,
                 int s, const int* __restrict__ perm, int position, uint64_t lo, uint64_t hi,
                 double* out_score, uint64_t* out_idx) {
  __shared__ int s_perm[64];
  __shared__ double s_best[kSliceThreads];
  __shared__ uint64_t s_idx[kSliceThreads];
  if (threadIdx.x < n) s_perm[threadIdx.x] = perm[threadIdx.x];
  __syncthreads();
  const int node = s_perm[position];
  double best = -INFINITY;
  uint64_t bi = ~0ull;
  for (uint64_t g = lo + threadIdx.x; g < hi; g += kSliceThreads) {
    int size = 0;
    const uint64_t pos_mask = unrank_global(g, position, s, &size);
    uint64_t nodes = 0;
    for (uint64_t m = pos_mask; m; m &= m - 1) nodes |= 1ull << s_perm[__ffsll((long long)m) - 1];
    const uint64_t gi = global_index_dev(nodes_to_cand(nodes, node), n - 1, s);
    const double eff = ls[(uint64_t)node * S + gi] + ppf_sum(w, n, node, nodes);
    if (eff > best) {  // ascending g within the thread: strict > keeps the first
      best = eff;
      bi = g;
    }
  }
  s_best[threadIdx.x] = best;
  s_idx[threadIdx.x] = bi;
  __syncthreads();
  for (int half = kSliceThreads / 2; half > 0; half >>= 1) {
    if (threadIdx.x < half) {
      const double b2 = s_best[threadIdx.x + half];
      const uint64_t i2 = s_idx[threadIdx.x + half];
      if (i2 != ~0ull && (b2 > s_best[threadIdx.x] ||
                          (b2 == s_best[threadIdx.x] && i2 < s_idx[threadIdx.x]))) {
        s_best[threadIdx.x] = b2;
        s_idx[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *out_score = s_best[0];
    *out_idx = s_idx[0];
  }
}

TieCtx tie_ctx(const bnmc_table* t) {
  TieCtx c;
  c.ls = t->ls.p;
  c.cmask = t->cmask.p;
  c.w = t->w.p;
  c.S = t->S;
  c.n = t->n;
  return c;
}

// eff = ls + PpfTable::sum in the scan's association (engine.cpp:50-51), fp64,
// with each entry's candidate mask: the input of the per-row sort.
// Delta-walk lists: for row v and candidate q, the entries of the sorted row
// that contain q, in sorted order (ordered stream compaction, one CTA per
// (q, v)), padded with never-admissible entries. Each list holds S(n-2, s-1)
// entries; *err is set on a count mismatch.
// Exclusion lists (xbit != null): one CTA per row v keeps the sorted entries
// WITHOUT candidate bit xbit[v] (S(n-2, s) of them) into list v.
constexpr int kYThreads = 256, kYItems = 4;
__global__ void __launch_bounds__(kYThreads) ylist_build_kernel(
    const double* __restrict__ seff, const uint64_t* __restrict__ scm, uint64_t S, uint64_t Sw,
    int n, ulonglong2* yrow, uint64_t Sy, uint64_t Syw, int* err,
    const uint64_t* __restrict__ xbit = nullptr) {
  const int q = blockIdx.x, v = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ uint32_t s_warp[kYThreads / 32 + 1];
  const double* re = seff + (uint64_t)v * Sw;
  const uint64_t* rc = scm + (uint64_t)v * Sw;
  const uint64_t lo = xbit ? (uint64_t)v * Syw : ((uint64_t)v * (n - 1) + q) * Syw;
  ulonglong2* orow = yrow + lo;
  const uint64_t bit = xbit ? xbit[v] : 1ull << q;
  const uint64_t want = xbit ? 0ull : bit;  // keep entries whose (m & bit) == want
  uint64_t out = 0;
  for (uint64_t c0 = 0; c0 < S; c0 += (uint64_t)kYThreads * kYItems) {
    double e[kYItems];
    uint64_t m[kYItems];
    uint32_t cnt = 0;
#pragma unroll
    for (int k = 0; k < kYItems; ++k) {
      const uint64_t i = c0 + (uint64_t)tid * kYItems + k;
      m[k] = i < S ? rc[i] : 0;
      e[k] = i < S ? re[i] : 0.0;
      cnt += i < S && (m[k] & bit) == want ? 1u : 0u;
    }
    // exclusive prefix of the per-thread counts over the CTA (warp scan + warp sums)
    uint32_t incl = cnt;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += x;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (tid == 0) {
      uint32_t run = 0;
      for (int w = 0; w < kYThreads / 32; ++w) {
        const uint32_t t = s_warp[w];
        s_warp[w] = run;
        run += t;
      }
      s_warp[kYThreads / 32] = run;
    }
    __syncthreads();
    uint64_t pos = out + s_warp[warp] + incl - cnt;
#pragma unroll
    for (int k = 0; k < kYItems; ++k)
      if (c0 + (uint64_t)tid * kYItems + k < S && (m[k] & bit) == want) {
        if (pos < Sy) orow[pos] = make_ulonglong2((unsigned long long)__double_as_longlong(e[k]), m[k]);
        ++pos;
      }
    out += s_warp[kYThreads / 32];
    __syncthreads();
  }
  if (tid == 0 && out != Sy) atomicExch(err, 6);
  for (uint64_t i = Sy + tid; i < Syw; i += kYThreads)
    orow[i] = make_ulonglong2((unsigned long long)__double_as_longlong(-INFINITY), ~0ull);
}

// Sorted rows, SoA (CUB output) -> AoS 16-byte entries, padded with
// never-admissible entries (eff -inf, mask ~0) up to the row stride Sw.
__global__ void pack_sorted_kernel(const double* __restrict__ seff, const uint64_t* __restrict__ scm,
                                   ulonglong2* srow, uint64_t S, uint64_t Sw) {
  const uint64_t v = blockIdx.y;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < Sw;
       i += (uint64_t)gridDim.x * blockDim.x)
    srow[v * Sw + i] = i < S ? make_ulonglong2((unsigned long long)__double_as_longlong(seff[v * S + i]),
                                               scm[v * S + i])
                             : make_ulonglong2((unsigned long long)__double_as_longlong(-INFINITY), ~0ull);
}

__global__ void eff64_kernel(const double* __restrict__ ls, const uint64_t* __restrict__ cmask,
                             const double* __restrict__ w, double* eff, uint64_t* cm, int n,
                             uint64_t S) {
  const int v = blockIdx.y;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < S;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t m = cmask[g];
    eff[(uint64_t)v * S + g] = ls[(uint64_t)v * S + g] + ppf_sum(w, n, v, cand_to_nodes(m, v));
    cm[(uint64_t)v * S + g] = m;
  }
}

// PST of predecessor count p (enumerate_bounded_position_sets order,
// combinatorics.hpp:83-101) for every p with S(p,s) <= kEnumMax: the walk
// path enumerates those rows instead of walking them.
void build_pst_table(int n, int s, int pmax, std::vector<uint64_t>& masks, std::vector<uint32_t>& off) {
  masks.clear();
  off.assign(1, 0);
  for (int p = 0; p <= pmax; ++p) {
    const uint64_t cnt = s < 0 ? 0 : bounded_count(p, s);
    for (uint64_t j = 0; j < cnt; ++j) {
      uint64_t r = j;
      int k = std::min(s, p);
      for (; k >= 0; --k) {
        const uint64_t block = hbinom(p, k);
        if (r < block) break;
        r -= block;
      }
      uint64_t m = 0;
      for (int i = 0, x = 0; i < k; ++i, ++x) {
        for (uint64_t c; r >= (c = hbinom(p - x - 1, k - i - 1)); ++x) r -= c;
        m |= 1ull << x;
      }
      masks.push_back(m);
    }
    off.push_back(static_cast<uint32_t>(masks.size()));
  }
  (void)n;
}

// PST of predecessor count p (enumerate_bounded_position_sets order,
// combinatorics.hpp:83-101) for every p with S(p,s) <= kEnumMax: the walk
// path enumerates those rows instead of walking them; plus PST(p, s-1) for
// p < pe (the sets containing one given position, for delta rescans).
void build_pst_small(bnmc_table* t) {
  int pe = -1;
  for (int p = 0; p < t->n && bounded_count(p, t->s) <= t->enum_max; ++p) pe = p;
  t->pe = pe;
  int pc = pe;
  const uint64_t cap = t->walk_cap ? t->walk_cap : std::max<uint64_t>(kEnumMax, t->S / kWalkCapDiv);
  if (t->walk_budget > 0)
    for (int p = pe + 1; p < t->n && bounded_count(p, t->s) <= cap; ++p) pc = p;
  t->pc = pc;
  std::vector<uint64_t> m1, m2;
  std::vector<uint32_t> o1, o2;
  build_pst_table(t->n, t->s, pc, m1, o1);
  build_pst_table(t->n, t->s - 1, std::max(pe - 1, 0), m2, o2);
  t->pst.alloc(std::max<size_t>(m1.size(), 1));
  t->pst_off.alloc(o1.size());
  t->pst2.alloc(std::max<size_t>(m2.size(), 1));
  t->pst2_off.alloc(o2.size());
  if (!m1.empty()) CK(cudaMemcpyAsync(t->pst.p, m1.data(), m1.size() * 8, cudaMemcpyHostToDevice, t->stream));
  CK(cudaMemcpyAsync(t->pst_off.p, o1.data(), o1.size() * 4, cudaMemcpyHostToDevice, t->stream));
  if (!m2.empty()) CK(cudaMemcpyAsync(t->pst2.p, m2.data(), m2.size() * 8, cudaMemcpyHostToDevice, t->stream));
  CK(cudaMemcpyAsync(t->pst2_off.p, o2.data(), o2.size() * 4, cudaMemcpyHostToDevice, t->stream));
  CK(cudaStreamSynchronize(t->stream));  // host vectors die here
}

// Sorted rows (descending eff, CUB radix sort per row; stable, so equal
// values keep ascending g). Rebuilt after every fold.
void ensure_sorted(bnmc_table* t) {
  // PST tables first: set_walk_cap / set_walk_params invalidate them without
  // touching the sorted rows
  if (!t->pst_ready) {
    build_pst_small(t);
    t->pst_ready = true;
  }
  if (t->sorted_valid) return;
  const uint64_t N = static_cast<uint64_t>(t->n) * t->S;
  // sorted rows padded with never-admissible entries so walk rounds need no
  // bounds checks: row stride Sw >= S + one full round
  t->Sw = (t->S + 32 * kWalkPadRound + 31) / 32 * 32;
  const uint64_t NW = static_cast<uint64_t>(t->n) * t->Sw;
  // CUB sorts into SoA temporaries (row stride S); the lists are built from
  // them, then they are packed into the 16-byte entries the walk reads
  DevBuf<double> seff;
  DevBuf<uint64_t> scm;
  seff.alloc(N);
  scm.alloc(N);
  t->srow.release();
  t->eff.alloc(N);  // eff in global-index order (kept: the enumeration gathers it)
  DevBuf<uint64_t> vals;
  vals.alloc(N);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, t->stream));
  const unsigned bx = static_cast<unsigned>(std::min<uint64_t>((t->S + 255) / 256, 4096));
  eff64_kernel<<<dim3(bx, t->n), 256, 0, t->stream>>>(t->ls.p, t->cmask.p, t->w.p, t->eff.p, vals.p,
                                                        t->n, t->S);
  CK(cudaGetLastError());
  size_t temp_bytes = 0;
  CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, temp_bytes, t->eff.p, seff.p, vals.p,
                                               scm.p, static_cast<int>(t->S), 0, 64, t->stream));
  DevBuf<uint8_t> temp;
  temp.alloc(std::max<size_t>(temp_bytes, 1));
  for (int v = 0; v < t->n; ++v) {
    const uint64_t o = static_cast<uint64_t>(v) * t->S;
    CK(cub::DeviceRadixSort::SortPairsDescending(temp.p, temp_bytes, t->eff.p + o, seff.p + o,
                                                 vals.p + o, scm.p + o, static_cast<int>(t->S),
                                                 0, 64, t->stream));
  }
  // delta-walk lists, when they fit comfortably in device memory
  t->Sy = t->s >= 1 && t->n >= 2 ? bounded_count(t->n - 2, t->s - 1) : 0;
  t->Syw = (t->Sy + 32 * kWalkPadRound + 31) / 32 * 32;
  const uint64_t ybytes = static_cast<uint64_t>(t->n) * (t->n - 1) * t->Syw * 16;
  size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  const char* ydis = std::getenv("BNMC_NO_YLISTS");
  t->ylists = t->Sy > 0 && !(ydis && ydis[0] == '1') && t->ylist_mode != 0 &&
              (ybytes < free_b / 3 || t->ylist_mode == 1);
  if (t->ylists) {
    t->yrow.alloc(static_cast<size_t>(ybytes / 16));
    ylist_build_kernel<<<dim3(t->n - 1, t->n), kYThreads, 0, t->stream>>>(
        seff.p, scm.p, t->S, t->S, t->n, t->yrow.p, t->Sy, t->Syw, t->rowcnt.p + 2 * t->n + 1);
    CK(cudaGetLastError());
  } else {
    t->yrow.release();
  }
  // exclusion lists: the row's strongest parents = the candidates most
  // frequent among its top 256 sorted entries (a heuristic: results are exact
  // for any choice, only walk lengths change); level j keeps the entries
  // without any of the j strongest, S(n-1-j, s) of them
  t->xlev = 0;
  const char* xdis = std::getenv("BNMC_XLISTS");  // levels (default kXLevels), 0 = off
  const int want_lev = std::min(kXLevels, xdis ? std::atoi(xdis) : kXLevels);
  uint64_t xtotal = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  for (int j = 1; j <= want_lev && t->s >= 1 && t->n - 1 - j >= 0; ++j) {
    const uint64_t Sx = bounded_count(t->n - 1 - j, t->s);
    const uint64_t Sxw = (Sx + 32 * kWalkPadRound + 31) / 32 * 32;
    const uint64_t add = static_cast<uint64_t>(t->n) * Sxw;
    if ((xtotal + add) * 16 >= free_b / 3) break;
    t->Sx[j] = Sx;
    t->Sxw[j] = Sxw;
    t->xoff[j] = xtotal;
    xtotal += add;
    t->xlev = j;
  }
  if (t->xlev > 0) {
    const int top = static_cast<int>(std::min<uint64_t>(256, t->S));
    std::vector<uint64_t> tops(static_cast<size_t>(t->n) * top);
    std::vector<uint64_t> bits(static_cast<size_t>(t->n) * kXLevels, 0);
    std::vector<uint64_t> masks(static_cast<size_t>(t->n) * t->xlev);
    CK(cudaMemcpy2DAsync(tops.data(), top * 8, scm.p, t->S * 8, top * 8, t->n,
                         cudaMemcpyDeviceToHost, t->stream));
    CK(cudaStreamSynchronize(t->stream));
    for (int v = 0; v < t->n; ++v) {
      int cnt[64] = {0};
      for (int i = 0; i < top; ++i)
        for (uint64_t m = tops[static_cast<size_t>(v) * top + i]; m; m &= m - 1)
          ++cnt[__builtin_ctzll(m)];
      uint64_t acc = 0;
      for (int j = 0; j < t->xlev; ++j) {
        int best = -1;  // most frequent candidate not taken yet (ties: lowest)
        for (int q = 0; q < t->n - 1; ++q)
          if (!((acc >> q) & 1) && (best < 0 || cnt[q] > cnt[best])) best = q;
        bits[static_cast<size_t>(v) * kXLevels + j] = 1ull << best;
        acc |= 1ull << best;
        masks[static_cast<size_t>(j) * t->n + v] = acc;
      }
    }
    t->xbit.alloc(bits.size());
    t->xrow.alloc(xtotal);
    DevBuf<uint64_t> d_masks;
    d_masks.alloc(masks.size());
    CK(cudaMemcpyAsync(t->xbit.p, bits.data(), 8 * bits.size(), cudaMemcpyHostToDevice, t->stream));
    CK(cudaMemcpyAsync(d_masks.p, masks.data(), 8 * masks.size(), cudaMemcpyHostToDevice,
                       t->stream));
    for (int j = 1; j <= t->xlev; ++j) {
      ylist_build_kernel<<<dim3(1, t->n), kYThreads, 0, t->stream>>>(
          seff.p, scm.p, t->S, t->S, t->n, t->xrow.p + t->xoff[j], t->Sx[j], t->Sxw[j],
          t->rowcnt.p + 2 * t->n + 1, d_masks.p + (j - 1) * t->n);
      CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(t->stream));  // host vectors and d_masks die here
  } else {
    t->xrow.release();
    t->xbit.release();
  }
  // pack the sorted rows (the SoA temporaries are freed on return)
  t->srow.alloc(NW);
  {
    const unsigned px = static_cast<unsigned>(std::min<uint64_t>((t->Sw + 255) / 256, 4096));
    pack_sorted_kernel<<<dim3(px, t->n), 256, 0, t->stream>>>(seff.p, scm.p, t->srow.p, t->S, t->Sw);
    CK(cudaGetLastError());
  }
  CK(cudaEventRecord(e1, t->stream));
  CK(cudaEventSynchronize(e1));
  CK(cudaEventElapsedTime(&t->sort_ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  t->sorted_valid = true;
}

// Team size: warps per chain (8 = one chain per CTA, 1 = one chain per warp).
// 0 = auto: whole-CTA chains while they fill the GPU at 4 CTAs per SM,
// otherwise one warp per chain.
void launch_walk(bnmc_table* t, const WalkArgs& A, int C, int team_warps = 0,
                 cudaStream_t st = nullptr) {
  if (!st) st = t->stream;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, t->dev);
  int tw = team_warps;
  if (tw == 0)
    tw = C <= sms ? 32 : (C <= 4 * sms ? 8 : (C <= 8 * sms ? 4 : (C <= 16 * sms ? 2 : 1)));
  const int cta = tw == 1 ? kWalkThreads1 : std::max(kWalkThreads, 32 * tw);
  const int per = cta / (32 * tw);
  const unsigned grid = static_cast<unsigned>((C + per - 1) / per);
  static const bool no_spec = [] {
    const char* e = std::getenv("BNMC_NO_SPEC");
    return e && e[0] == '1';
  }();
  // speculation pays once chains settle (lower acceptance): long runs only
  if (tw == 32 && A.perms == nullptr && !no_spec && A.iters >= 1000 && !A.recheck) {
    // few chains: one 1024-thread CTA per chain evaluating kSpecD proposals per round
    walk_spec_kernel<<<C, 1024, 0, st>>>(A);
    CK(cudaGetLastError());
    t->last_team = 32;
    t->last_wu = 8;
    t->last_spec = 1;
    return;
  }
  // deep rows (long walks): 8 entries per lane per round for small teams
  const bool deep = t->walk_deep < 0 ? t->S > kDeepRowEntries : t->walk_deep == 1;
  if (A.recheck) {  // debug_recheck variants (results are identical for every team size)
    const int rtw = tw >= 16 ? 32 : (tw >= 8 ? 8 : 1);
    const int rcta = rtw == 1 ? kWalkThreads1 : std::max(kWalkThreads, 32 * rtw);
    const int rper = rcta / (32 * rtw);
    const unsigned rgrid = static_cast<unsigned>((C + rper - 1) / rper);
    if (rtw == 32) walk_chain_kernel<32, 8, true><<<rgrid, rcta, 0, st>>>(A);
    else if (rtw == 8) walk_chain_kernel<8, 8, true><<<rgrid, rcta, 0, st>>>(A);
    else walk_chain_kernel<1, kWalkUnroll, true><<<rgrid, rcta, 0, st>>>(A);
    CK(cudaGetLastError());
    t->last_team = rtw;
    t->last_wu = rtw >= 8 ? 8 : kWalkUnroll;
    t->last_spec = 0;
    return;
  }
  switch (tw) {
    case 32: walk_chain_kernel<32><<<grid, cta, 0, st>>>(A); break;
    case 16: walk_chain_kernel<16><<<grid, cta, 0, st>>>(A); break;
    case 8: walk_chain_kernel<8><<<grid, cta, 0, st>>>(A); break;
    case 4:
      if (deep) walk_chain_kernel<4, 8><<<grid, cta, 0, st>>>(A);
      else walk_chain_kernel<4><<<grid, cta, 0, st>>>(A);
      break;
    case 2:
      if (deep) walk_chain_kernel<2, 8><<<grid, cta, 0, st>>>(A);
      else walk_chain_kernel<2><<<grid, cta, 0, st>>>(A);
      break;
    case 1:
      if (deep) walk_chain_kernel<1, 8><<<grid, cta, 0, st>>>(A);
      else walk_chain_kernel<1><<<grid, cta, 0, st>>>(A);
      break;
    default: raise(BNMC_USAGE, "team_warps must be 0, 1, 2, 4, 8, 16 or 32");
  }
  CK(cudaGetLastError());
  t->last_team = tw;
  t->last_wu = tw >= 8 || deep ? 8 : kWalkUnroll;
  t->last_spec = 0;
}

WalkArgs walk_args(bnmc_table* t) {
  WalkArgs A{};
  A.srow = t->srow.p;
  A.eff = t->eff.p;
  A.Sw = t->Sw;
  A.yrow = t->ylists ? t->yrow.p : nullptr;
  A.Sy = t->Sy;
  A.Syw = t->Syw;
  A.xrow = t->xlev ? t->xrow.p : nullptr;
  A.xbit = t->xlev ? t->xbit.p : nullptr;
  A.xlev = t->xlev;
  for (int j = 0; j <= kXLevels; ++j) {
    A.xoff[j] = t->xoff[j];
    A.Sx32[j] = static_cast<uint32_t>(t->Sx[j]);
    A.Sxw32[j] = static_cast<uint32_t>(t->Sxw[j]);
  }
  A.ls = t->ls.p;
  A.w = t->w.p;
  A.pst = t->pst.p;
  A.pst_off = t->pst_off.p;
  A.pst2 = t->pst2.p;
  A.pst2_off = t->pst2_off.p;
  A.pe = t->pe;
  A.pc = t->pc;
  A.wbud = t->walk_budget;
  A.S = t->S;
  if (t->Sw > 0xFFFFFFFFull || t->Syw > 0xFFFFFFFFull)
    raise(BNMC_CAPACITY, "sorted rows longer than 2^32 entries");
  A.S32 = static_cast<uint32_t>(t->S);
  A.Sw32 = static_cast<uint32_t>(t->Sw);
  A.Syw32 = static_cast<uint32_t>(t->Syw);
  A.n = t->n;
  A.s = t->s;
  A.stat = t->stat.p;
  A.error = t->rowcnt.p + 2 * t->n + 1;
  return A;
}

// Accept thresholds: log10(next_unit_open()) of the split(3) stream with the
// host's glibc log10 — exactly mh_accept's left-hand side (sampler.cpp:54-56).
// The acceptance stream draws once per iteration whatever the outcome, so it
// is state-independent and can be materialised before the device loop.
void accept_thresholds(const uint64_t* seeds, int C, uint64_t iters, std::vector<double>& out) {
  out.assign(static_cast<size_t>(C) * (iters + 1), 0.0);
#pragma omp parallel for schedule(static)
  for (int c = 0; c < C; ++c) {
    Rng acc = Rng{seeds[c]}.split(3);
    double* o = out.data() + static_cast<size_t>(c) * (iters + 1);
    for (uint64_t t = 1; t <= iters; ++t) o[t] = std::log10(acc.next_unit_open());
  }
}

void ensure_workspace(bnmc_table* t, int C, uint64_t iters, int K) {
  const int n = t->n;
  t->st.alloc(C);
  t->items.alloc(static_cast<size_t>(C) * 64);
  t->counts.alloc(C);
  t->ppos.alloc(static_cast<size_t>(C) * 64);
  t->buckets.alloc(2ull * n * kMaxChains);
  t->rowcnt.alloc(2ull * n + 2);  // + sel + error
  t->cell.alloc(2ull * C * n);
  t->stat.alloc(4);
  if (iters) {
    t->props.alloc(static_cast<size_t>(C) * (iters + 1) * 2);
    t->thr.alloc(static_cast<size_t>(C) * (iters + 1));
    t->tmasks.alloc(static_cast<size_t>(C) * K * n);
    t->ttotals.alloc(static_cast<size_t>(C) * K);
    t->tr_prop.alloc(static_cast<size_t>(C) * iters);
    t->tr_best.alloc(static_cast<size_t>(C) * iters);
    t->tr_acc.alloc(static_cast<size_t>(C) * iters);
  }
  // clean buckets, cells, sel, error flag
  CK(cudaMemsetAsync(t->rowcnt.p, 0, sizeof(int) * (2ull * n + 2), t->stream));
  CK(cudaMemsetAsync(t->cell.p, 0, 16ull * C * n, t->stream));
  CK(cudaMemsetAsync(t->stat.p, 0, 32, t->stream));
}

StepArgs step_args(bnmc_table* t) {
  StepArgs A{};
  A.st = t->st.p;
  A.items = t->items.p;
  A.counts = t->counts.p;
  A.ppos = t->ppos.p;
  A.buckets = t->buckets.p;
  A.rowcnt = t->rowcnt.p;
  A.sel = t->rowcnt.p + 2 * t->n;
  A.error = t->rowcnt.p + 2 * t->n + 1;
  A.cell = t->cell.p;
  A.keys = t->key32.p;
  A.Sp = t->Sp;
  A.stat_rows = t->stat.p;
  A.n = t->n;
  A.tie = tie_ctx(t);
  return A;
}

ScanArgs scan_args(const bnmc_table* t, const ScanGeom& g) {
  ScanArgs sa{};
  sa.keys = t->key32.p;
  sa.Sp = t->Sp;
  sa.buckets = t->buckets.p;
  sa.rowcnt = t->rowcnt.p;
  sa.sel = t->rowcnt.p + 2 * t->n;
  sa.ppos = t->ppos.p;
  sa.cell = t->cell.p;
  sa.n = t->n;
  sa.sectors = g.sectors;
  sa.tie = tie_ctx(t);
  sa.sector_loads = t->stat.p + 1;
  return sa;
}

int read_error(bnmc_table* t);

// OrderScorer::score for `count` orders through the walk kernel (one CTA per
// order, every row rescanned).
void score_orders_walk(bnmc_table* t, const int* perms, int count, uint64_t* masks_out,
                       double* best_out, double* totals_out) {
  const int n = t->n;
  ensure_workspace(t, 1, 0, 0);
  ensure_sorted(t);
  t->perms.alloc(static_cast<size_t>(count) * n);
  t->out_masks.alloc(static_cast<size_t>(count) * n);
  t->out_best.alloc(static_cast<size_t>(count) * n);
  t->out_total.alloc(count);
  CK(cudaMemcpyAsync(t->perms.p, perms, sizeof(int) * count * n, cudaMemcpyHostToDevice, t->stream));
  WalkArgs A = walk_args(t);
  A.C = count;
  A.perms = t->perms.p;
  A.out_masks = t->out_masks.p;
  A.out_best = t->out_best.p;
  A.out_total = t->out_total.p;
  launch_walk(t, A, count);
  CK(cudaGetLastError());
  if (masks_out)
    CK(cudaMemcpyAsync(masks_out, t->out_masks.p, 8ull * count * n, cudaMemcpyDeviceToHost, t->stream));
  if (best_out)
    CK(cudaMemcpyAsync(best_out, t->out_best.p, 8ull * count * n, cudaMemcpyDeviceToHost, t->stream));
  if (totals_out)
    CK(cudaMemcpyAsync(totals_out, t->out_total.p, 8ull * count, cudaMemcpyDeviceToHost, t->stream));
  CK(cudaStreamSynchronize(t->stream));
}

// One launch of the fused walk kernel over chains `seeds[0..C)`; outputs to the
// host pointers (any may be null). host_thr: glibc thresholds from the host
// (exact), else device log10 with ambiguity flags returned in *amb_out.
void walk_launch(bnmc_table* t, const uint64_t* seeds, int C, const bnmc_chain_params* params,
                 bool host_thr, double* trace_proposed, uint8_t* trace_accepted, double* trace_best,
                 int* final_order, double* final_score, uint64_t* accepted, int* tracker_count,
                 uint64_t* tracker_masks, double* tracker_totals, float* device_ms,
                 std::vector<int>* amb_out) {
  const int n = t->n, K = params->track_top;
  const uint64_t iters = params->iterations;
  ensure_workspace(t, 1, 0, 0);  // error flag + stats
  ensure_sorted(t);
  t->seeds.alloc(C);
  t->tmasks.alloc(static_cast<size_t>(C) * K * n);
  t->ttotals.alloc(static_cast<size_t>(C) * K);
  t->thash.alloc(static_cast<size_t>(C) * K);
  const bool slots = K <= kTrackSlots;  // slot tracker (walk.cuh tracker_insert_slots)
  if (slots) {
    t->smasks.alloc(static_cast<size_t>(C) * K * n);
    t->stotals.alloc(static_cast<size_t>(C) * K);
    t->shash.alloc(static_cast<size_t>(C) * K);
  }
  t->tr_prop.alloc(static_cast<size_t>(C) * iters);
  t->tr_best.alloc(static_cast<size_t>(C) * iters);
  t->tr_acc.alloc(static_cast<size_t>(C) * iters);
  t->d_fo.alloc(static_cast<size_t>(C) * n);
  t->d_tc.alloc(C);
  t->d_acc.alloc(C);
  t->d_fs.alloc(C);
  t->d_amb.alloc(C);
  CK(cudaMemcpyAsync(t->seeds.p, seeds, 8ull * C, cudaMemcpyHostToDevice, t->stream));
  std::vector<double> thr;
  if (host_thr) {
    t->thr.alloc(static_cast<size_t>(C) * (iters + 1));
    accept_thresholds(seeds, C, iters, thr);
    CK(cudaMemcpyAsync(t->thr.p, thr.data(), thr.size() * 8, cudaMemcpyHostToDevice, t->stream));
  }
  WalkArgs A = walk_args(t);
  A.C = C;
  A.iters = iters;
  A.K = K;
  A.strict = params->strict;
  A.seeds = t->seeds.p;
  A.thr = host_thr ? t->thr.p : nullptr;
  A.accept_tol = std::ldexp(1.0, params->accept_tol_log2 ? params->accept_tol_log2 : -48);
  A.ambiguous = t->d_amb.p;
  A.tmasks = t->tmasks.p;
  A.ttotals = t->ttotals.p;
  A.thash = t->thash.p;
  A.tcount = t->d_tc.p;
  A.smasks = slots ? t->smasks.p : nullptr;
  A.stotals = slots ? t->stotals.p : nullptr;
  A.shash = slots ? t->shash.p : nullptr;
  A.tr_prop = t->tr_prop.p;
  A.tr_acc = t->tr_acc.p;
  A.tr_best = t->tr_best.p;
  A.final_order = t->d_fo.p;
  A.final_score = t->d_fs.p;
  A.accepted = t->d_acc.p;
  A.recheck = params->debug_recheck != 0;
  // test hook (tests/test_gpu_headline.py): the sequential draw path that
  // next_below rejections take, forced for every batch
  A.seq_draws = env_u64("BNMC_SEQ_DRAWS", 0) != 0;
  // Chain blocks: with page-locked result buffers and many chains the chains
  // run as kBlocks launches alternating over two streams, and each block's
  // results are copied to the host while the next block computes (its CTAs
  // fill the SMs as the previous block's retire, so the split costs no tail).
  // Chains are independent and every result is the reference's bit for bit
  // whatever the launch split.
  static const int kBlocks = static_cast<int>(std::max<uint64_t>(1, env_u64("BNMC_CHAIN_BLOCKS", 4)));
  constexpr int kBlockMinChains = 4096;
  cudaPointerAttributes pa{};
  const bool pinned = trace_proposed && cudaPointerGetAttributes(&pa, trace_proposed) == cudaSuccess &&
                      pa.type == cudaMemoryTypeHost;
  cudaGetLastError();  // a pageable pointer may leave an error behind on old drivers
  const int B = pinned && C >= kBlocks * kBlockMinChains && !A.recheck ? kBlocks : 1;
  if (B > 1 && !t->stream2) CK(cudaStreamCreateWithFlags(&t->stream2, cudaStreamNonBlocking));
  std::vector<cudaEvent_t> ev(B + 1);
  for (auto& e : ev) CK(cudaEventCreate(&e));
  CK(cudaEventRecord(ev[0], t->stream));
  if (B > 1) CK(cudaStreamWaitEvent(t->stream2, ev[0], 0));
  for (int b = 0; b < B; ++b) {
    const int c0 = static_cast<int>(static_cast<int64_t>(C) * b / B);
    const int c1 = static_cast<int>(static_cast<int64_t>(C) * (b + 1) / B);
    const int Cb = c1 - c0;
    const uint64_t o = static_cast<uint64_t>(c0);
    cudaStream_t st = b % 2 == 0 ? t->stream : t->stream2;
    WalkArgs Ab = A;
    Ab.C = Cb;
    Ab.seeds = A.seeds + o;
    if (A.thr) Ab.thr = A.thr + o * (iters + 1);
    Ab.ambiguous = A.ambiguous + o;
    Ab.tmasks = A.tmasks + o * K * n;
    Ab.ttotals = A.ttotals + o * K;
    Ab.thash = A.thash + o * K;
    Ab.tcount = A.tcount + o;
    if (slots) {
      Ab.smasks = A.smasks + o * K * n;
      Ab.stotals = A.stotals + o * K;
      Ab.shash = A.shash + o * K;
    }
    Ab.tr_prop = A.tr_prop + o * iters;
    Ab.tr_acc = A.tr_acc + o * iters;
    Ab.tr_best = A.tr_best + o * iters;
    Ab.final_order = A.final_order + o * n;
    Ab.final_score = A.final_score + o;
    Ab.accepted = A.accepted + o;
    launch_walk(t, Ab, Cb, params->team_warps, st);
    CK(cudaEventRecord(ev[b + 1], st));
    auto d2h = [&](auto* dst, const auto* src, uint64_t per) {
      if (dst)
        CK(cudaMemcpyAsync(dst + o * per, src + o * per, sizeof(*src) * per * Cb,
                           cudaMemcpyDeviceToHost, st));
    };
    d2h(trace_proposed, t->tr_prop.p, iters);
    d2h(trace_accepted, t->tr_acc.p, iters);
    d2h(trace_best, t->tr_best.p, iters);
    d2h(tracker_masks, t->tmasks.p, static_cast<uint64_t>(K) * n);
    d2h(tracker_totals, t->ttotals.p, static_cast<uint64_t>(K));
    d2h(final_order, t->d_fo.p, static_cast<uint64_t>(n));
    d2h(final_score, t->d_fs.p, 1);
    d2h(accepted, reinterpret_cast<const uint64_t*>(t->d_acc.p), 1);
    d2h(tracker_count, t->d_tc.p, 1);
  }
  if (B > 1) {  // join: the primary stream waits for the second one
    cudaEvent_t j;
    CK(cudaEventCreate(&j));
    CK(cudaEventRecord(j, t->stream2));
    CK(cudaStreamWaitEvent(t->stream, j, 0));
    cudaEventDestroy(j);
  }
  std::vector<int> amb(C, 0);
  if (!host_thr)
    CK(cudaMemcpyAsync(amb.data(), t->d_amb.p, sizeof(int) * C, cudaMemcpyDeviceToHost, t->stream));
  unsigned long long stats[4] = {0, 0, 0, 0};
  CK(cudaMemcpyAsync(stats, t->stat.p, 32, cudaMemcpyDeviceToHost, t->stream));
  CK(cudaStreamSynchronize(t->stream));
  float ms = 0.f;
  for (int b = 1; b <= B; ++b) {  // device time: first launch to the last block's end
    float x = 0.f;
    CK(cudaEventElapsedTime(&x, ev[0], ev[b]));
    ms = std::max(ms, x);
  }
  for (auto& e : ev) cudaEventDestroy(e);
  if (device_ms) *device_ms = ms;
  if (amb_out) {
    amb_out->clear();
    for (int c = 0; c < C; ++c)
      if (amb[c]) amb_out->push_back(c);
  }
  t->last_drift_it = stats[3];
  t->last_rescans = stats[0];
  t->last_sectors = stats[1] + stats[2];  // walk path: entries visited (walked + enumerated)
  t->last_walked = stats[1];
  t->last_enumerated = stats[2];
  t->last_launches = B;
  t->last_total_ms = ms;
  t->last_scan_ms = ms;
  t->last_scan_samples = 1;
  t->last_G = C;
}

// run_chains through the fused walk kernel: one launch for all chains and
// iterations. Acceptance uses the device's log10 unless the caller asks for
// host thresholds; chains whose decisions came within the glibc/CUDA log10
// bound of the threshold are replayed with host glibc thresholds, so every
// trace is the reference's bit for bit.
void run_chains_walk(bnmc_table* t, const uint64_t* seeds, int C, const bnmc_chain_params* params,
                     double* trace_proposed, uint8_t* trace_accepted, double* trace_best,
                     int* final_order, double* final_score, uint64_t* accepted, int* tracker_count,
                     uint64_t* tracker_masks, double* tracker_totals, float* device_ms) {
  const bool host_thr = params->exact_accept == 1;
  std::vector<int> amb;
  walk_launch(t, seeds, C, params, host_thr, trace_proposed, trace_accepted, trace_best,
              final_order, final_score, accepted, tracker_count, tracker_masks, tracker_totals,
              device_ms, &amb);
  const uint64_t keep[4] = {t->last_rescans, t->last_walked, t->last_enumerated, t->last_sectors};
  const float keep_ms = t->last_scan_ms;
  const uint64_t keep_launches = t->last_launches;
  t->last_replayed = amb.size();
  if (amb.empty()) return;
  const int R = static_cast<int>(amb.size()), n = t->n, K = params->track_top;
  const uint64_t it = params->iterations;
  std::vector<uint64_t> rs(R);
  for (int i = 0; i < R; ++i) rs[i] = seeds[amb[i]];
  std::vector<double> tp(R * it), tb(R * it), fs(R), tt(static_cast<size_t>(R) * K);
  std::vector<uint8_t> ta(R * it);
  std::vector<int> fo(static_cast<size_t>(R) * n), tc(R);
  std::vector<uint64_t> acc(R), tm(static_cast<size_t>(R) * K * n);
  float replay_ms = 0.f;
  walk_launch(t, rs.data(), R, params, true, tp.data(), ta.data(), tb.data(), fo.data(), fs.data(),
              acc.data(), tc.data(), tm.data(), tt.data(), &replay_ms, nullptr);
  if (device_ms) *device_ms += replay_ms;  // the replay is part of the call's device time
  for (int i = 0; i < R; ++i) {
    const size_t c = static_cast<size_t>(amb[i]);
    if (trace_proposed) std::copy_n(tp.data() + i * it, it, trace_proposed + c * it);
    if (trace_accepted) std::copy_n(ta.data() + i * it, it, trace_accepted + c * it);
    if (trace_best) std::copy_n(tb.data() + i * it, it, trace_best + c * it);
    if (final_order) std::copy_n(fo.data() + static_cast<size_t>(i) * n, n, final_order + c * n);
    if (final_score) final_score[c] = fs[i];
    if (accepted) accepted[c] = acc[i];
    if (tracker_count) tracker_count[c] = tc[i];
    if (tracker_masks)
      std::copy_n(tm.data() + static_cast<size_t>(i) * K * n, static_cast<size_t>(K) * n,
                  tracker_masks + c * K * n);
    if (tracker_totals) std::copy_n(tt.data() + static_cast<size_t>(i) * K, K, tracker_totals + c * K);
  }
  t->last_rescans = keep[0];
  t->last_walked = keep[1];
  t->last_enumerated = keep[2];
  t->last_sectors = keep[3];
  t->last_scan_ms = keep_ms + replay_ms;
  t->last_launches = keep_launches + t->last_launches;
}

void validate_cards(const int* cards, int n) {
  for (int i = 0; i < n; ++i)
    if (cards[i] < 2 || cards[i] > 256)
      raise(BNMC_DATA, "cardinality of variable " + std::to_string(i) + " out of range [2,256]");
}

// Dataset validation (types.cpp:8-26).
void validate_dataset(const uint8_t* cells, const int* cards, uint64_t m, int n) {
  if (n < 1 || n > 64) raise(BNMC_DATA, "dataset must have between 1 and 64 variables");
  validate_cards(cards, n);
  for (uint64_t r = 0; r < m; ++r)
    for (int i = 0; i < n; ++i)
      if (cells[r * n + i] >= cards[i])
        raise(BNMC_DATA, "state out of range at row " + std::to_string(r) + ", column " +
                             std::to_string(i));
}

// K1 (+ K1W) for a prefix / row range of the table's local scores.
void run_k1(bnmc_table* t, const uint8_t* cells, const int* cards, uint64_t m, const K1Range& R) {
  K1Report rep;
  precompute(t->stream, t->ls.p, t->S, cells, cards, m, t->n, t->s, t->gamma, t->ess, t->alpha, R,
             &rep);
  t->build_ms = rep.ms;
  t->wide_entries = rep.wide_entries;
  const uint64_t total = bnmc_host::prefix_total(t->n, t->s);
  t->p_lo = std::min(R.p_lo, total);
  t->p_hi = std::min(R.p_hi, total);
}

template <class F>
void for_each_replica(bnmc_table* t, F&& f) {
  f(t);
  for (bnmc_table* r : t->replicas) f(r);
}

// Run f(g) on one host thread per device g (each thread binds its device);
// the first exception is rethrown on the caller's thread.
template <class F>
void on_devices(const std::vector<bnmc_table*>& ts, F&& f) {
  if (ts.size() == 1) {
    CK(cudaSetDevice(ts[0]->dev));
    f(0);
    return;
  }
  std::vector<std::exception_ptr> errs(ts.size());
  std::vector<std::thread> th;
  for (size_t g = 0; g < ts.size(); ++g)
    th.emplace_back([&, g] {
      try {
        CK(cudaSetDevice(ts[g]->dev));
        f(static_cast<int>(g));
      } catch (...) {
        errs[g] = std::current_exception();
      }
    });
  for (auto& x : th) x.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

// Devices of an n_gpus table: device .. device+G-1. BNMC_DEVICES="a,b,..."
// overrides the list (development: several parts on one GPU).
std::vector<int> device_list(int first, int G) {
  std::vector<int> d;
  if (const char* e = std::getenv("BNMC_DEVICES")) {
    for (const char* p = e; *p;) {
      d.push_back(static_cast<int>(std::strtol(p, const_cast<char**>(&p), 10)));
      while (*p == ',' || *p == ' ') ++p;
    }
    if (static_cast<int>(d.size()) < G) raise(BNMC_USAGE, "BNMC_DEVICES lists fewer than n_gpus devices");
    d.resize(G);
    return d;
  }
  int count = 0;
  CK(cudaGetDeviceCount(&count));
  if (first + G > count)
    raise(BNMC_CUDA, std::to_string(G) + " GPUs requested from device " + std::to_string(first) +
                         ", " + std::to_string(count) + " visible");
  for (int g = 0; g < G; ++g) d.push_back(first + g);
  return d;
}

__global__ void add_i64_kernel(unsigned long long* __restrict__ dst,
                               const unsigned long long* __restrict__ src, uint64_t count) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] += src[i];
}

// Complete a table from its parts: every local-score word is written by
// exactly one part and zero elsewhere, so an integer sum of the 64-bit words
// is the bitwise union. Distinct devices: ncclAllReduce(int64, sum) in place
// over NVLink (one group call). Shared devices (BNMC_DEVICES): peer copies +
// an add kernel on the first table, then copies back.
void combine_parts(const std::vector<bnmc_table*>& ts) {
  const size_t words = static_cast<size_t>(ts[0]->n) * ts[0]->S;
  bool distinct = true;
  for (size_t i = 0; i < ts.size(); ++i)
    for (size_t j = 0; j < i; ++j) distinct &= ts[i]->dev != ts[j]->dev;
  if (distinct) {
    const auto& N = bnmc_host::nccl();
    std::vector<int> devs;
    for (auto* t : ts) devs.push_back(t->dev);
    std::vector<ncclComm_t> comms(ts.size());
    NK(N.CommInitAll(comms.data(), static_cast<int>(ts.size()), devs.data()));
    NK(N.GroupStart());
    for (size_t g = 0; g < ts.size(); ++g) {
      CK(cudaSetDevice(ts[g]->dev));
      NK(N.AllReduce(ts[g]->ls.p, ts[g]->ls.p, words, ncclInt64, ncclSum, comms[g], ts[g]->stream));
    }
    NK(N.GroupEnd());
    for (size_t g = 0; g < ts.size(); ++g) {
      CK(cudaSetDevice(ts[g]->dev));
      CK(cudaStreamSynchronize(ts[g]->stream));
      N.CommDestroy(comms[g]);
    }
    CK(cudaSetDevice(ts[0]->dev));
    return;
  }
  bnmc_table* t0 = ts[0];
  CK(cudaSetDevice(t0->dev));
  DevBuf<unsigned long long> tmp;
  tmp.alloc(words);
  auto* dst = reinterpret_cast<unsigned long long*>(t0->ls.p);
  for (size_t g = 1; g < ts.size(); ++g) {
    CK(cudaMemcpyPeerAsync(tmp.p, t0->dev, ts[g]->ls.p, ts[g]->dev, words * 8, t0->stream));
    add_i64_kernel<<<148 * 8, 256, 0, t0->stream>>>(dst, tmp.p, words);
    CK(cudaGetLastError());
  }
  for (size_t g = 1; g < ts.size(); ++g)
    CK(cudaMemcpyPeerAsync(ts[g]->ls.p, ts[g]->dev, t0->ls.p, t0->dev, words * 8, t0->stream));
  CK(cudaStreamSynchronize(t0->stream));
}

// ScoreCache::build over G devices of this process (bnmc_score_params::n_gpus).
bnmc_table* build_multi(const uint8_t* cells, const int* cards, uint64_t m, int n,
                        const bnmc_score_params* params, const double* prior_r) {
  const int G = params->n_gpus;
  const std::vector<int> devs = device_list(params->device, G);
  std::vector<std::unique_ptr<bnmc_table>> own;
  std::vector<bnmc_table*> ts;
  for (int g = 0; g < G; ++g) {
    bnmc_score_params p = *params;
    p.device = devs[g];
    p.n_gpus = 1;
    own.emplace_back(new bnmc_table);
    table_init(own.back().get(), n, &p);
    set_priors(own.back().get(), prior_r);
    CK(cudaMemsetAsync(own.back()->ls.p, 0, static_cast<size_t>(n) * own.back()->S * 8,
                       own.back()->stream));
    ts.push_back(own.back().get());
  }
  const std::vector<uint64_t> cut = bnmc_host::k1_partition(cards, n, params->max_parents, m, G);
  on_devices(ts, [&](int g) {
    K1Range R;
    R.p_lo = cut[g];
    R.p_hi = cut[g + 1];
    run_k1(ts[g], cells, cards, m, R);
    CK(cudaStreamSynchronize(ts[g]->stream));
  });
  combine_parts(ts);
  on_devices(ts, [&](int g) { fold(ts[g]); });
  bnmc_table* t = own[0].release();
  float k1 = t->build_ms;
  uint64_t wide = t->wide_entries;
  for (int g = 1; g < G; ++g) {
    k1 = std::max(k1, own[g]->build_ms);
    wide += own[g]->wide_entries;
    t->replicas.push_back(own[g].release());
  }
  t->build_ms = k1;  // the slowest part
  t->wide_entries = wide;
  t->p_lo = 0;
  t->p_hi = cut[G];
  CK(cudaSetDevice(t->dev));
  return t;
}

int read_error(bnmc_table* t) {
  int err = 0;
  CK(cudaMemcpy(&err, t->rowcnt.p + 2 * t->n + 1, sizeof(int), cudaMemcpyDeviceToHost));
  return err;
}

}  // namespace

// ------------------------------------------------------------------ C-ABI
extern "C" {

const char* bnmc_gpu_last_error_message(void) { return g_err.c_str(); }
int bnmc_gpu_version(void) { return 10000; }

int bnmc_gpu_device_count(int* out) {
  return guarded([&] {
    int count = 0;
    const cudaError_t e = cudaGetDeviceCount(&count);
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) {
      cudaGetLastError();
      *out = 0;
      return;
    }
    CK(e);
    int ok = 0;
    for (int d = 0; d < count; ++d) {
      cudaDeviceProp p;
      CK(cudaGetDeviceProperties(&p, d));
      if (p.major == 10) ++ok;
    }
    *out = ok;
  });
}

int bnmc_gpu_host_alloc(uint64_t bytes, void** out) {
  return guarded([&] {
    if (!out) raise(BNMC_USAGE, "null output pointer");
    *out = nullptr;
    int count = 0;
    CK(cudaGetDeviceCount(&count));
    if (bytes == 0) return;
    CK(cudaHostAlloc(out, bytes, cudaHostAllocPortable));
  });
}

int bnmc_gpu_host_free(void* p) {
  return guarded([&] {
    if (p) CK(cudaFreeHost(p));
  });
}

uint64_t bnmc_gpu_table_estimate_bytes(int n, int s) {
  return static_cast<uint64_t>(n) * bounded_count(n - 1, s) * 8;
}
uint64_t bnmc_gpu_bounded_subset_count(int c, int s) { return bounded_count(c, s); }

int bnmc_gpu_table_upload(const double* table, int n, const bnmc_score_params* params,
                          const double* prior_r, bnmc_table** out) {
  return guarded([&] {
    auto t = std::make_unique<bnmc_table>();
    table_init(t.get(), n, params);
    CK(cudaMemcpyAsync(t->ls.p, table, static_cast<size_t>(n) * t->S * 8, cudaMemcpyHostToDevice,
                       t->stream));
    set_priors(t.get(), prior_r);
    fold(t.get());
    *out = t.release();
  });
}

int bnmc_gpu_table_build(const uint8_t* cells, const int* cards, uint64_t m, int n,
                         const bnmc_score_params* params, const double* prior_r,
                         bnmc_table** out) {
  if (params && params->n_gpus > 1)
    return guarded([&] {
      *out = nullptr;
      validate_params(params);
      validate_dataset(cells, cards, m, n);
      *out = build_multi(cells, cards, m, n, params, prior_r);
    });
  int st = bnmc_gpu_table_build_rows(cells, cards, m, n, params, prior_r, 0, n, out);
  if (st != BNMC_OK) return st;
  st = bnmc_gpu_table_finalize(*out);
  if (st != BNMC_OK) {
    const std::string keep = g_err;
    bnmc_gpu_table_free(*out);
    *out = nullptr;
    g_err = keep;
  }
  return st;
}

int bnmc_gpu_table_build_rows(const uint8_t* cells, const int* cards, uint64_t m, int n,
                              const bnmc_score_params* params, const double* prior_r,
                              int row_begin, int row_end, bnmc_table** out) {
  return guarded([&] {
    *out = nullptr;
    validate_dataset(cells, cards, m, n);
    if (row_begin < 0 || row_end > n || row_begin > row_end) raise(BNMC_USAGE, "bad row range");
    auto t = std::make_unique<bnmc_table>();
    table_init(t.get(), n, params);
    set_priors(t.get(), prior_r);
    K1Range R;
    R.row_begin = row_begin;
    R.row_end = row_end;
    run_k1(t.get(), cells, cards, m, R);
    *out = t.release();
  });
}

int bnmc_gpu_k1_partition(const int* cards, uint64_t m, int n, int s, int nparts,
                          uint64_t* cuts) {
  return guarded([&] {
    if (n < 1 || n > 64) raise(BNMC_DATA, "dataset must have between 1 and 64 variables");
    if (s < 0 || s > 8) raise(BNMC_USAGE, "max-parents must lie in [0,8]");
    if (nparts < 1) raise(BNMC_USAGE, "nparts must be >= 1");
    validate_cards(cards, n);
    const std::vector<uint64_t> c = bnmc_host::k1_partition(cards, n, s, m, nparts);
    std::copy(c.begin(), c.end(), cuts);
  });
}

int bnmc_gpu_table_build_part(const uint8_t* cells, const int* cards, uint64_t m, int n,
                              const bnmc_score_params* params, const double* prior_r, int part,
                              int nparts, bnmc_table** out) {
  return guarded([&] {
    *out = nullptr;
    validate_dataset(cells, cards, m, n);
    if (nparts < 1 || part < 0 || part >= nparts) raise(BNMC_USAGE, "bad part index");
    auto t = std::make_unique<bnmc_table>();
    table_init(t.get(), n, params);
    set_priors(t.get(), prior_r);
    const std::vector<uint64_t> cut =
        bnmc_host::k1_partition(cards, n, t->s, m, nparts);
    CK(cudaMemsetAsync(t->ls.p, 0, static_cast<size_t>(n) * t->S * 8, t->stream));
    K1Range R;
    R.p_lo = cut[part];
    R.p_hi = cut[part + 1];
    run_k1(t.get(), cells, cards, m, R);
    *out = t.release();
  });
}

int bnmc_gpu_table_k1_stats(const bnmc_table* t, float* k1_ms, uint64_t* wide_entries,
                            uint64_t* prefix_lo, uint64_t* prefix_hi) {
  return guarded([&] {
    if (!t) raise(BNMC_USAGE, "null table");
    if (k1_ms) *k1_ms = t->build_ms;
    if (wide_entries) *wide_entries = t->wide_entries;
    if (prefix_lo) *prefix_lo = t->p_lo;
    if (prefix_hi) *prefix_hi = t->p_hi;
  });
}

int bnmc_gpu_table_rows_buffer(bnmc_table* t, void** dev_ptr, uint64_t* bytes,
                               uint64_t* row_stride_elems) {
  return guarded([&] {
    if (!t) raise(BNMC_USAGE, "null table");
    *dev_ptr = t->ls.p;
    *bytes = static_cast<uint64_t>(t->n) * t->S * 8;
    *row_stride_elems = t->S;
  });
}

int bnmc_gpu_table_finalize(bnmc_table* t) {
  return guarded([&] {
    if (!t) raise(BNMC_USAGE, "null table");
    CK(cudaSetDevice(t->dev));
    fold(t);
  });
}

int bnmc_gpu_table_set_priors(bnmc_table* t, const double* prior_r) {
  return guarded([&] {
    if (!t) raise(BNMC_USAGE, "null table");
    for_each_replica(t, [&](bnmc_table* r) {
      CK(cudaSetDevice(r->dev));
      set_priors(r, prior_r);
      fold(r);
    });
    CK(cudaSetDevice(t->dev));
  });
}

// ------------------------------------------------------------ communicators
int bnmc_gpu_comm_unique_id(uint8_t* id128) {
  return guarded([&] {
    if (!id128) raise(BNMC_USAGE, "null id buffer");
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
    ncclUniqueId id;
    NK(bnmc_host::nccl().GetUniqueId(&id));
    std::memcpy(id128, &id, sizeof(id));
  });
}

int bnmc_gpu_comm_init(const uint8_t* id128, int nranks, int rank, int device, bnmc_comm** out) {
  return guarded([&] {
    *out = nullptr;
    if (!id128) raise(BNMC_USAGE, "null id");
    if (nranks < 1 || rank < 0 || rank >= nranks) raise(BNMC_USAGE, "bad rank / nranks");
    ensure_device(device);
    const auto& N = bnmc_host::nccl();
    auto c = std::make_unique<bnmc_comm>();
    c->rank = rank;
    c->nranks = nranks;
    c->dev = device;
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    NK(N.CommInitRank(&c->comm, nranks, id, rank));
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    *out = c.release();
  });
}

int bnmc_gpu_comm_free(bnmc_comm* c) {
  return guarded([&] {
    if (!c) return;
    cudaSetDevice(c->dev);
    delete c;
  });
}

int bnmc_gpu_table_build_comm(const uint8_t* cells, const int* cards, uint64_t m, int n,
                              const bnmc_score_params* params, const double* prior_r,
                              bnmc_comm* comm, bnmc_table** out) {
  return guarded([&] {
    *out = nullptr;
    if (!comm) raise(BNMC_USAGE, "null communicator");
    validate_params(params);
    if (params->device != comm->dev)
      raise(BNMC_USAGE, "params->device must be the communicator's device");
    validate_dataset(cells, cards, m, n);
    auto t = std::make_unique<bnmc_table>();
    table_init(t.get(), n, params);
    set_priors(t.get(), prior_r);
    const size_t words = static_cast<size_t>(n) * t->S;
    CK(cudaMemsetAsync(t->ls.p, 0, words * 8, t->stream));
    const std::vector<uint64_t> cut =
        bnmc_host::k1_partition(cards, n, t->s, m, comm->nranks);
    K1Range R;
    R.p_lo = cut[comm->rank];
    R.p_hi = cut[comm->rank + 1];
    run_k1(t.get(), cells, cards, m, R);
    // every word has one writer (zero elsewhere): the int64 sum is the union
    NK(bnmc_host::nccl().AllReduce(t->ls.p, t->ls.p, words, ncclInt64, ncclSum, comm->comm,
                                   t->stream));
    CK(cudaStreamSynchronize(t->stream));
    fold(t.get());
    *out = t.release();
  });
}

int bnmc_gpu_comm_allgather(bnmc_comm* c, const void* send, uint64_t bytes, void* recv) {
  return guarded([&] {
    if (!c) raise(BNMC_USAGE, "null communicator");
    CK(cudaSetDevice(c->dev));
    DevBuf<uint8_t> d;
    d.alloc(bytes * (c->nranks + 1) + 1);
    uint8_t* dsend = d.p + bytes * c->nranks;
    CK(cudaMemcpyAsync(dsend, send, bytes, cudaMemcpyHostToDevice, c->stream));
    NK(bnmc_host::nccl().AllGather(dsend, d.p, bytes, ncclUint8, c->comm, c->stream));
    CK(cudaMemcpyAsync(recv, d.p, bytes * c->nranks, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int bnmc_gpu_comm_allreduce_max(bnmc_comm* c, double* values, int count) {
  return guarded([&] {
    if (!c) raise(BNMC_USAGE, "null communicator");
    if (count < 1) return;
    CK(cudaSetDevice(c->dev));
    DevBuf<double> d;
    d.alloc(count);
    CK(cudaMemcpyAsync(d.p, values, 8ull * count, cudaMemcpyHostToDevice, c->stream));
    NK(bnmc_host::nccl().AllReduce(d.p, d.p, count, ncclFloat64, ncclMax, c->comm, c->stream));
    CK(cudaMemcpyAsync(values, d.p, 8ull * count, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int bnmc_gpu_table_devices(const bnmc_table* t, int* count, int* devices) {
  return guarded([&] {
    if (!t) raise(BNMC_USAGE, "null table");
    if (count) *count = 1 + static_cast<int>(t->replicas.size());
    if (devices) {
      devices[0] = t->dev;
      for (size_t g = 0; g < t->replicas.size(); ++g) devices[g + 1] = t->replicas[g]->dev;
    }
  });
}

int bnmc_gpu_table_info(const bnmc_table* t, int* n, int* s, uint64_t* per_node) {
  return guarded([&] {
    if (!t) raise(BNMC_USAGE, "null table");
    if (n) *n = t->n;
    if (s) *s = t->s;
    if (per_node) *per_node = t->S;
  });
}

int bnmc_gpu_table_download(const bnmc_table* t, double* out) {
  return guarded([&] {
    if (!t) raise(BNMC_USAGE, "null table");
    CK(cudaSetDevice(t->dev));
    CK(cudaMemcpyAsync(out, t->ls.p, static_cast<size_t>(t->n) * t->S * 8, cudaMemcpyDeviceToHost,
                       t->stream));
    CK(cudaStreamSynchronize(t->stream));
  });
}

int bnmc_gpu_table_build_ms(const bnmc_table* t, float* count_score_ms, float* fold_ms) {
  return guarded([&] {
    if (!t) raise(BNMC_USAGE, "null table");
    if (count_score_ms) *count_score_ms = t->build_ms;
    if (fold_ms) *fold_ms = t->fold_ms;
  });
}

int bnmc_gpu_table_free(bnmc_table* t) {
  return guarded([&] {
    if (!t) return;
    cudaSetDevice(t->dev);
    delete t;
  });
}

int bnmc_gpu_count_statistics(const uint8_t* cells, const int* cards, uint64_t m, int n, int count,
                              const int* nodes, const uint64_t* psets, const uint64_t* offsets,
                              uint32_t* out, uint64_t* configs_out, int device) {
  return guarded([&] {
    ensure_device(device);
    count_statistics_device(cells, cards, m, n, count, nodes, psets, offsets, out, configs_out);
  });
}

int bnmc_gpu_count_statistics_sparse(const uint8_t* cells, const int* cards, uint64_t m, int n,
                                     int node, uint64_t pset, uint64_t* configs_out,
                                     uint32_t* counts_out, uint64_t* n_active, int device) {
  return guarded([&] {
    ensure_device(device);
    bnmc_host::count_statistics_sparse_device(cells, cards, m, n, node, pset, configs_out,
                                              counts_out, n_active);
  });
}

int bnmc_gpu_score_orders(bnmc_table* t, const int* perms, int count, uint64_t* masks_out,
                          double* best_out, double* totals_out) {
  return guarded([&] {
    if (!t) raise(BNMC_USAGE, "null table");
    if (count < 1) return;
    const int n = t->n;
    for (int c = 0; c < count; ++c) {  // Order::Order validation (types.cpp:28-38)
      std::vector<bool> seen(n, false);
      for (int i = 0; i < n; ++i) {
        const int v = perms[static_cast<size_t>(c) * n + i];
        if (v < 0 || v >= n || seen[v]) raise(BNMC_DATA, "order is not a permutation of 0..n-1");
        seen[v] = true;
      }
    }
    CK(cudaSetDevice(t->dev));
    if (t->scan_mode != 1) {
      score_orders_walk(t, perms, count, masks_out, best_out, totals_out);
      if (const int err = read_error(t))
        raise(BNMC_ERR, "walk consistency check failed (" + std::to_string(err) + ")");
      return;
    }
    const ScanGeom g = scan_geometry(t, kMaxChainsPerLaunch * n);
    t->perms.alloc(static_cast<size_t>(kMaxChainsPerLaunch) * n);
    t->out_masks.alloc(static_cast<size_t>(count) * n);
    t->out_best.alloc(static_cast<size_t>(count) * n);
    t->out_total.alloc(count);
    ensure_workspace(t, kMaxChainsPerLaunch, 0, 0);
    for (int c0 = 0; c0 < count; c0 += kMaxChainsPerLaunch) {
      const int cc = std::min(kMaxChainsPerLaunch, count - c0);
      CK(cudaMemcpyAsync(t->perms.p, perms + static_cast<size_t>(c0) * n, sizeof(int) * cc * n,
                         cudaMemcpyHostToDevice, t->stream));
      CK(cudaMemsetAsync(t->rowcnt.p, 0, sizeof(int) * 2ull * n, t->stream));
      StepArgs A = step_args(t);
      A.score_only = 1;
      A.out_masks = t->out_masks.p + static_cast<size_t>(c0) * n;
      A.out_best = t->out_best.p + static_cast<size_t>(c0) * n;
      A.out_total = t->out_total.p + c0;
      setup_items_kernel<<<cc, 64, 0, t->stream>>>(A, t->perms.p, cc);
      CK(cudaGetLastError());
      launch_scan(g, scan_args(t, g), cc * n, t->stream, false);
      launch_step(cc, A, t->stream, false);
    }
    if (masks_out)
      CK(cudaMemcpyAsync(masks_out, t->out_masks.p, 8ull * count * n, cudaMemcpyDeviceToHost,
                         t->stream));
    if (best_out)
      CK(cudaMemcpyAsync(best_out, t->out_best.p, 8ull * count * n, cudaMemcpyDeviceToHost,
                         t->stream));
    if (totals_out)
      CK(cudaMemcpyAsync(totals_out, t->out_total.p, 8ull * count, cudaMemcpyDeviceToHost,
                         t->stream));
    CK(cudaStreamSynchronize(t->stream));
    if (const int err = read_error(t))
      raise(BNMC_ERR, "scan consistency check failed (" + std::to_string(err) + ")");
  });
}

int bnmc_gpu_bench_scan(bnmc_table* t, const int* perms, int count, int lo, int hi, int reps,
                        int flush_l2, float* ms_per_launch, uint64_t* key_bytes_per_launch) {
  return guarded([&] {
    if (!t) raise(BNMC_USAGE, "null table");
    if (count < 1 || count > kMaxChainsPerLaunch) raise(BNMC_USAGE, "count must lie in [1,64]");
    const int n = t->n;
    if (lo < 0 || hi >= n || lo > hi) raise(BNMC_USAGE, "bad position range");
    CK(cudaSetDevice(t->dev));
    const ScanGeom g = scan_geometry(t, count * n);
    t->perms.alloc(static_cast<size_t>(count) * n);
    ensure_workspace(t, count, 0, 0);
    CK(cudaMemcpyAsync(t->perms.p, perms, sizeof(int) * count * n, cudaMemcpyHostToDevice,
                       t->stream));
    StepArgs A = step_args(t);
    setup_items_range_kernel<<<count, 64, 0, t->stream>>>(A, t->perms.p, count, lo, hi);
    CK(cudaGetLastError());
    const ScanArgs sa = scan_args(t, g);
    launch_scan(g, sa, count * n, t->stream, false);  // warm-up
    DevBuf<uint32_t> scratch;  // > L2 (126 MB): every timed launch starts cold
    if (flush_l2) scratch.alloc(64ull << 20);
    CK(cudaMemsetAsync(sa.sector_loads, 0, sizeof(unsigned long long), t->stream));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    double total = 0.0;
    for (int r = 0; r < std::max(1, reps); ++r) {
      if (flush_l2) CK(cudaMemsetAsync(scratch.p, r & 0xff, 256ull << 20, t->stream));
      CK(cudaEventRecord(e0, t->stream));
      launch_scan(g, sa, count * n, t->stream, false);
      CK(cudaEventRecord(e1, t->stream));
      CK(cudaEventSynchronize(e1));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      total += ms;
    }
    *ms_per_launch = static_cast<float>(total / std::max(1, reps));
    if (key_bytes_per_launch) {
      unsigned long long slots = 0;
      CK(cudaMemcpy(&slots, sa.sector_loads, sizeof(slots), cudaMemcpyDeviceToHost));
      *key_bytes_per_launch = slots * 16ull / static_cast<uint64_t>(std::max(1, reps));
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

int bnmc_gpu_score_order(bnmc_table* t, const int* perm, uint64_t* masks_out, double* best_out,
                         double* total_out) {
  return bnmc_gpu_score_orders(t, perm, 1, masks_out, best_out, total_out);
}

void run_chains_one(bnmc_table* t, const uint64_t* seeds, int n_chains,
                    const bnmc_chain_params* params, double* trace_proposed,
                    uint8_t* trace_accepted, double* trace_best, int* final_order,
                    double* final_score, uint64_t* accepted, int* tracker_count,
                    uint64_t* tracker_masks, double* tracker_totals, float* device_ms);

int bnmc_gpu_run_chains(bnmc_table* t, const uint64_t* seeds, int n_chains,
                        const bnmc_chain_params* params, double* trace_proposed,
                        uint8_t* trace_accepted, double* trace_best, int* final_order,
                        double* final_score, uint64_t* accepted, int* tracker_count,
                        uint64_t* tracker_masks, double* tracker_totals, float* device_ms) {
  return guarded([&] {
    if (!t) raise(BNMC_USAGE, "null table");
    if (!params) raise(BNMC_USAGE, "null chain params");
    if (t->replicas.empty() || n_chains < 2 || params->scan_mode == 1) {
      run_chains_one(t, seeds, n_chains, params, trace_proposed, trace_accepted, trace_best,
                     final_order, final_score, accepted, tracker_count, tracker_masks,
                     tracker_totals, device_ms);
      return;
    }
    // Multi-GPU table: contiguous chain blocks per device, outputs written in
    // place (chain order preserved); device time = the slowest device.
    std::vector<bnmc_table*> ts{t};
    for (bnmc_table* r : t->replicas) ts.push_back(r);
    const int G = static_cast<int>(std::min<size_t>(ts.size(), n_chains));
    ts.resize(G);
    const uint64_t I = params->iterations;
    const int n = t->n, K = params->track_top;
    std::vector<float> ms(G, 0.f);
    on_devices(ts, [&](int g) {
      const int c0 = static_cast<int>(static_cast<int64_t>(n_chains) * g / G);
      const int c1 = static_cast<int>(static_cast<int64_t>(n_chains) * (g + 1) / G);
      auto off = [&](auto* p, uint64_t per) { return p ? p + static_cast<uint64_t>(c0) * per : p; };
      run_chains_one(ts[g], seeds + c0, c1 - c0, params, off(trace_proposed, I),
                     off(trace_accepted, I), off(trace_best, I), off(final_order, n),
                     off(final_score, 1), off(accepted, 1), off(tracker_count, 1),
                     off(tracker_masks, static_cast<uint64_t>(K) * n), off(tracker_totals, K),
                     &ms[g]);
    });
    CK(cudaSetDevice(t->dev));
    if (device_ms) *device_ms = *std::max_element(ms.begin(), ms.end());
    for (int g = 1; g < G; ++g) {  // walk statistics of the whole call on the primary
      t->last_walked += ts[g]->last_walked;
      t->last_enumerated += ts[g]->last_enumerated;
      t->last_rescans += ts[g]->last_rescans;
      t->last_replayed += ts[g]->last_replayed;
    }
  });
}

void run_chains_one(bnmc_table* t, const uint64_t* seeds, int n_chains,
                    const bnmc_chain_params* params, double* trace_proposed,
                    uint8_t* trace_accepted, double* trace_best, int* final_order,
                    double* final_score, uint64_t* accepted, int* tracker_count,
                    uint64_t* tracker_masks, double* tracker_totals, float* device_ms) {
  {
    if (!t) raise(BNMC_USAGE, "null table");
    if (!params) raise(BNMC_USAGE, "null chain params");
    if (params->iterations < 1) raise(BNMC_USAGE, "iterations must be >= 1");
    if (params->track_top < 1) raise(BNMC_USAGE, "tracker capacity must be >= 1");
    if (t->n < 2) raise(BNMC_USAGE, "swap proposal needs at least two nodes");
    const int mode = params->scan_mode;
    if (mode < 0 || mode > 2) raise(BNMC_USAGE, "scan_mode must be 0, 1 or 2");
    if (n_chains < 1 || (mode == 1 && n_chains > kMaxChainsPerLaunch))
      raise(BNMC_USAGE, "n_chains must lie in [1," + std::to_string(kMaxChainsPerLaunch) +
                            "] for scan_mode 1");
    CK(cudaSetDevice(t->dev));
    if (mode != 1) {
      run_chains_walk(t, seeds, n_chains, params, trace_proposed, trace_accepted, trace_best,
                      final_order, final_score, accepted, tracker_count, tracker_masks,
                      tracker_totals, device_ms);
      if (const int err = read_error(t)) {
        if (err == kErrDrift)  // RunConfig::debug_recheck, sampler.cpp:105-110
          raise(BNMC_ERR, "chain score drifted from recomputation at iteration " +
                              std::to_string(t->last_drift_it));
        raise(BNMC_ERR, "walk consistency check failed (" + std::to_string(err) + ")");
      }
      return;
    }
    if (params->debug_recheck)
      raise(BNMC_USAGE, "debug_recheck runs on the sorted-walk path (scan_mode 0 or 2)");
    const int n = t->n, C = n_chains, K = params->track_top;
    const uint64_t iters = params->iterations;
    const ScanGeom g = scan_geometry(t, C * n);
    ensure_workspace(t, C, iters, K);
    t->seeds.alloc(C);
    std::vector<double> thr;
    accept_thresholds(seeds, C, iters, thr);
    CK(cudaMemcpyAsync(t->seeds.p, seeds, 8ull * C, cudaMemcpyHostToDevice, t->stream));
    CK(cudaMemcpyAsync(t->thr.p, thr.data(), thr.size() * 8, cudaMemcpyHostToDevice, t->stream));
    StepArgs A = step_args(t);
    A.props = t->props.p;
    A.thr = t->thr.p;
    A.tmasks = t->tmasks.p;
    A.ttotals = t->ttotals.p;
    A.tr_prop = t->tr_prop.p;
    A.tr_acc = t->tr_acc.p;
    A.tr_best = t->tr_best.p;
    A.iters = iters;
    A.K = K;
    A.strict = params->strict;
    setup_chains_kernel<<<(C + 63) / 64, 64, 0, t->stream>>>(A, t->seeds.p, C);
    CK(cudaGetLastError());
    setup_items_kernel<<<C, 64, 0, t->stream>>>(A, nullptr, C);
    CK(cudaGetLastError());
    const ScanArgs sa = scan_args(t, g);

    // Two instances of a captured batch of (scan, step) pairs with PDL edges;
    // every `sample`-th scan is bracketed by event-record nodes so the scan's
    // device time is measured live. Instances alternate so the host harvests
    // one instance's events while the other runs. Steps past `iters` are no-ops.
    const uint64_t total_steps = iters + 1;
    const int batch = static_cast<int>(std::min<uint64_t>(total_steps, 128));
    const int sample = std::max(1, params->timing_sample > 0 ? params->timing_sample : 8);
    const uint64_t replays = (total_steps + batch - 1) / batch;
    const int ninst = replays > 1 ? 2 : 1;
    struct Inst {
      cudaGraphExec_t exec = nullptr;
      std::vector<cudaEvent_t> ev;
    } inst[2];
    for (int k = 0; k < ninst; ++k) {
      for (int i = 0; i < batch; i += sample) {
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        inst[k].ev.push_back(e0);
        inst[k].ev.push_back(e1);
      }
      cudaGraph_t graph;
      CK(cudaStreamBeginCapture(t->stream, cudaStreamCaptureModeThreadLocal));
      for (int i = 0; i < batch; ++i) {
        const bool timed = i % sample == 0;
        if (timed) CK(cudaEventRecordWithFlags(inst[k].ev[2 * (i / sample)], t->stream,
                                               cudaEventRecordExternal));
        launch_scan(g, sa, C * n, t->stream, !timed && i > 0);
        if (timed) CK(cudaEventRecordWithFlags(inst[k].ev[2 * (i / sample) + 1], t->stream,
                                               cudaEventRecordExternal));
        launch_step(C, A, t->stream, !timed);
      }
      CK(cudaStreamEndCapture(t->stream, &graph));
      CK(cudaGraphInstantiate(&inst[k].exec, graph, 0));
      cudaGraphDestroy(graph);
    }
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    double scan_ms = 0.0;
    uint64_t scan_samples = 0;
    auto harvest = [&](Inst& in) {
      for (size_t i = 0; i + 1 < in.ev.size(); i += 2) {
        float ms = 0.f;
        CK(cudaEventSynchronize(in.ev[i + 1]));
        CK(cudaEventElapsedTime(&ms, in.ev[i], in.ev[i + 1]));
        scan_ms += ms;
        ++scan_samples;
      }
    };
    CK(cudaEventRecord(e0, t->stream));
    for (uint64_t r = 0; r < replays; ++r) {
      Inst& cur = inst[r % ninst];
      if (r >= 2) harvest(cur);  // its previous launch must finish before reuse
      CK(cudaGraphLaunch(cur.exec, t->stream));
    }
    CK(cudaEventRecord(e1, t->stream));
    CK(cudaEventSynchronize(e1));
    for (uint64_t r = replays >= 2 ? replays - 2 : 0; r < replays; ++r) harvest(inst[r % ninst]);
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (device_ms) *device_ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    for (int k = 0; k < ninst; ++k) {
      for (auto e : inst[k].ev) cudaEventDestroy(e);
      cudaGraphExecDestroy(inst[k].exec);
    }
    CK(cudaGetLastError());

    // Results back to the host.
    std::vector<ChainState> hs(C);
    CK(cudaMemcpyAsync(hs.data(), t->st.p, sizeof(ChainState) * C, cudaMemcpyDeviceToHost,
                       t->stream));
    if (trace_proposed)
      CK(cudaMemcpyAsync(trace_proposed, t->tr_prop.p, 8ull * C * iters, cudaMemcpyDeviceToHost,
                         t->stream));
    if (trace_accepted)
      CK(cudaMemcpyAsync(trace_accepted, t->tr_acc.p, 1ull * C * iters, cudaMemcpyDeviceToHost,
                         t->stream));
    if (trace_best)
      CK(cudaMemcpyAsync(trace_best, t->tr_best.p, 8ull * C * iters, cudaMemcpyDeviceToHost,
                         t->stream));
    if (tracker_masks)
      CK(cudaMemcpyAsync(tracker_masks, t->tmasks.p, 8ull * C * K * n, cudaMemcpyDeviceToHost,
                         t->stream));
    if (tracker_totals)
      CK(cudaMemcpyAsync(tracker_totals, t->ttotals.p, 8ull * C * K, cudaMemcpyDeviceToHost,
                         t->stream));
    unsigned long long stats[2] = {0, 0};
    CK(cudaMemcpyAsync(stats, t->stat.p, 16, cudaMemcpyDeviceToHost, t->stream));
    CK(cudaStreamSynchronize(t->stream));
    if (const int err = read_error(t))
      raise(BNMC_ERR, "scan consistency check failed (" + std::to_string(err) + ")");
    for (int c = 0; c < C; ++c) {
      if (!hs[c].done) raise(BNMC_ERR, "chain did not finish (internal error)");
      if (final_order)
        for (int i = 0; i < n; ++i) final_order[c * n + i] = hs[c].order[i];
      if (final_score) final_score[c] = hs[c].total;
      if (accepted) accepted[c] = hs[c].accepted;
      if (tracker_count) tracker_count[c] = hs[c].tcount;
    }
    t->last_rescans = stats[0];
    t->last_sectors = stats[1];
    t->last_launches = replays * batch * 2 + 2;
    t->last_total_ms = ms;
    t->last_scan_ms = scan_samples ? static_cast<float>(scan_ms / scan_samples) : 0.f;
    t->last_scan_samples = scan_samples;
    t->last_G = g.G;
  }
}

int bnmc_gpu_scan_slice(bnmc_table* t, const int* perm, int position, uint64_t lo, uint64_t hi,
                        double* score_out, uint64_t* idx_out) {
  return guarded([&] {
    if (!t) raise(BNMC_USAGE, "null table");
    const int n = t->n;
    std::vector<bool> seen(n, false);
    for (int i = 0; i < n; ++i) {
      const int v = perm[i];
      if (v < 0 || v >= n || seen[v]) raise(BNMC_DATA, "order is not a permutation of 0..n-1");
      seen[v] = true;
    }
    if (position < 0 || position >= n) raise(BNMC_USAGE, "slice position out of range");
    const uint64_t total = bounded_count(position, t->s);
    if (lo > hi || hi > total) raise(BNMC_USAGE, "slice range outside [0, S(position, s))");
    *score_out = -INFINITY;
    *idx_out = ~0ull;
    if (lo == hi) return;
    CK(cudaSetDevice(t->dev));
    t->perms.alloc(std::max<size_t>(t->perms.n, static_cast<size_t>(n)));
    t->out_best.alloc(std::max<size_t>(t->out_best.n, 1));
    t->out_masks.alloc(std::max<size_t>(t->out_masks.n, 1));
    CK(cudaMemcpyAsync(t->perms.p, perm, sizeof(int) * n, cudaMemcpyHostToDevice, t->stream));
    slice_kernel<<<1, kSliceThreads, 0, t->stream>>>(t->ls.p, t->w.p, t->S, n, t->s, t->perms.p,
                                                     position, lo, hi, t->out_best.p,
                                                     t->out_masks.p);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(score_out, t->out_best.p, 8, cudaMemcpyDeviceToHost, t->stream));
    CK(cudaMemcpyAsync(idx_out, t->out_masks.p, 8, cudaMemcpyDeviceToHost, t->stream));
    CK(cudaStreamSynchronize(t->stream));
  });
}

int bnmc_gpu_table_set_scan_mode(bnmc_table* t, int mode) {
  return guarded([&] {
    if (!t) raise(BNMC_USAGE, "null table");
    if (mode < 0 || mode > 2) raise(BNMC_USAGE, "scan_mode must be 0, 1 or 2");
    for_each_replica(t, [&](bnmc_table* r) { r->scan_mode = mode; });
  });
}

int bnmc_gpu_table_set_walk_cap(bnmc_table* t, int64_t walk_cap, int64_t budget, int deep) {
  return guarded([&] {
    if (!t) raise(BNMC_USAGE, "null table");
    if (deep < -1 || deep > 1) raise(BNMC_USAGE, "deep must be -1, 0 or 1");
    if (budget > 0xFFFF) raise(BNMC_USAGE, "walk budget must be <= 65535");
    for_each_replica(t, [&](bnmc_table* r) {
      r->walk_deep = deep;
      r->walk_cap = walk_cap < 0 ? 0 : static_cast<uint64_t>(walk_cap);
      r->walk_budget =
          budget < 0 ? static_cast<uint32_t>(kWalkBudget) : static_cast<uint32_t>(budget);
      r->pst_ready = false;
    });
  });
}

int bnmc_gpu_table_set_walk_params(bnmc_table* t, int64_t enum_max, int ylists) {
  return guarded([&] {
    if (!t) raise(BNMC_USAGE, "null table");
    for_each_replica(t, [&](bnmc_table* r) {
      r->enum_max = enum_max < 0 ? kEnumMax : static_cast<uint64_t>(enum_max);
      r->pst_ready = false;
      r->ylist_mode = ylists;
      r->sorted_valid = false;
    });
  });
}

int bnmc_gpu_last_walk_stats(const bnmc_table* t, uint64_t* pairs, uint64_t* walked,
                             uint64_t* enumerated, float* sort_ms) {
  return guarded([&] {
    if (!t) raise(BNMC_USAGE, "null table");
    if (pairs) *pairs = t->last_rescans;
    if (walked) *walked = t->last_walked;
    if (enumerated) *enumerated = t->last_enumerated;
    if (sort_ms) *sort_ms = t->sort_ms;
  });
}

int bnmc_gpu_last_walk_variant(const bnmc_table* t, int* team_warps, int* entries_per_lane,
                               int* speculative) {
  return guarded([&] {
    if (!t) raise(BNMC_USAGE, "null table");
    if (team_warps) *team_warps = t->last_team;
    if (entries_per_lane) *entries_per_lane = t->last_wu;
    if (speculative) *speculative = t->last_spec;
  });
}

int bnmc_gpu_last_replayed(const bnmc_table* t, uint64_t* chains) {
  return guarded([&] {
    if (!t) raise(BNMC_USAGE, "null table");
    *chains = t->last_replayed;
  });
}

int bnmc_gpu_last_scan_stats(const bnmc_table* t, uint64_t* row_rescans, uint64_t* sectors,
                             float* scan_ms_avg, uint64_t* kernel_launches) {
  return guarded([&] {
    if (!t) raise(BNMC_USAGE, "null table");
    if (row_rescans) *row_rescans = t->last_rescans;
    if (sectors) *sectors = t->last_sectors;
    if (scan_ms_avg) *scan_ms_avg = t->last_scan_ms;
    if (kernel_launches) *kernel_launches = t->last_launches;
  });
}

}  // extern "C"
