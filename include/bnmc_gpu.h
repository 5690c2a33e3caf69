/* bnmc_gpu.h — C-ABI of the B200-native order-MCMC hot path.
 *
 * Drop-in boundary for the reference's hot path (arXiv:1210.5128 order-space
 * MCMC, reference project "bnmc", paths relative to /root/reference/proj):
 *
 *   reference interface                                   replaced by
 *   ---------------------------------------------------   ----------------------------------
 *   ScoreCache::build(const Dataset&, const RunConfig&)   bnmc_gpu_table_build
 *     (include/bnmc/scoring.hpp:126, src/scoring.cpp:162-192)
 *   count_statistics(const Dataset&, int, ParentSet)      bnmc_gpu_count_statistics
 *     (include/bnmc/scoring.hpp:79, src/scoring.cpp:82-109)
 *   ScoreCache::estimate_bytes (scoring.hpp:123)          bnmc_gpu_table_estimate_bytes
 *   ScoreCache::load / prebuilt cache (scoring.hpp:153,   bnmc_gpu_table_upload
 *     sampler.hpp:63-65 `prebuilt`)
 *   ScoreCache::save / at / lookup (scoring.hpp:141-152)  bnmc_gpu_table_download
 *   OrderScorer::OrderScorer(cache, priors, EngineConfig) bnmc_gpu_table_set_priors
 *     (include/bnmc/engine.hpp:77-78; PpfTable scoring.hpp:96-112)
 *   OrderScorer::score(const Order&) (engine.hpp:80,      bnmc_gpu_score_order(s)
 *     src/engine.cpp:60-98); score_order (scoring.cpp:261-289)
 *   OrderScorer::scan_slice (engine.hpp:83,               bnmc_gpu_scan_slice
 *     src/engine.cpp:43-58)
 *   run_mcmc(data, cfg, priors, prebuilt)                 bnmc_gpu_run_chains
 *     (include/bnmc/sampler.hpp:63-65, src/sampler.cpp:58-116)
 *
 * Conventions:
 *   * Every function returns a status: 0 ok, 2 usage (reference UsageError),
 *     3 data (DataError), 4 capacity (CapacityError), 5 CUDA, 6 NCCL, 1 other. The
 *     message of the last failure on the calling thread is returned by
 *     bnmc_gpu_last_error_message().
 *   * The caller owns every host buffer; the library owns device memory through
 *     the opaque handle. Calls are synchronous at return. One handle must not be
 *     used from two threads at once.
 *   * There is no CPU fallback: without a usable sm_100 device every compute
 *     entry point fails with status 5.
 *   * Layouts: datasets are row-major uint8 m x n (Dataset::cells, types.hpp:77-79);
 *     prior matrices are row-major double n x n with r[child*n + parent]
 *     (PriorMatrix, types.hpp:149-163), NULL = neutral; tables are double
 *     n x S(n-1,s) in (node, global index) order — the BNSC body order
 *     (scoring.hpp:148-153, scoring.cpp:194-238); parent sets are u64 node masks.
 */
#ifndef BNMC_GPU_H
#define BNMC_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  BNMC_OK = 0,
  BNMC_ERR = 1,
  BNMC_USAGE = 2,
  BNMC_DATA = 3,
  BNMC_CAPACITY = 4,
  BNMC_CUDA = 5,
  BNMC_NCCL = 6
};

enum { BNMC_ALPHA_BDEU = 0, BNMC_ALPHA_K2 = 1 };

typedef struct bnmc_table bnmc_table;
typedef struct bnmc_comm bnmc_comm;

/* The scoring fields of RunConfig (types.hpp:167-183) that the table depends on. */
typedef struct {
  int max_parents;           /* s, RunConfig::max_parents, in [0,8] */
  double gamma;              /* per-parent penalty, (0,1] */
  double ess;                /* equivalent sample size, > 0 */
  int alpha_mode;            /* BNMC_ALPHA_BDEU | BNMC_ALPHA_K2 */
  uint64_t memory_cap_bytes; /* RunConfig::memory_cap_bytes (checked like estimate_bytes) */
  int device;                /* CUDA ordinal this table lives on (the first of n_gpus) */
  int n_gpus;                /* 0 or 1: one device. G > 1: one process drives devices
                                device .. device+G-1 — the precompute is split into G
                                work-balanced parts (bnmc_gpu_k1_partition), one per
                                GPU, combined by an NCCL all-reduce over NVLink; every
                                GPU keeps a full replica and bnmc_gpu_run_chains spreads
                                chains over them (contiguous blocks, chain order kept) */
} bnmc_score_params;

const char* bnmc_gpu_last_error_message(void);
/* Library/ABI version, e.g. 10000 for 1.0.0. */
int bnmc_gpu_version(void);
/* Number of usable sm_100 devices (0 when none; status 5 when the runtime fails). */
int bnmc_gpu_device_count(int* out);

/* Page-locked (pinned) host memory for result buffers: device->host copies of
 * run_chains outputs into it run at full PCIe/C2C bandwidth and need no
 * staging. bytes == 0 yields NULL. Free with bnmc_gpu_host_free. */
int bnmc_gpu_host_alloc(uint64_t bytes, void** out);
int bnmc_gpu_host_free(void* p);

/* S(n-1,s) * 8: ScoreCache::estimate_bytes (scoring.cpp:157-160). */
uint64_t bnmc_gpu_table_estimate_bytes(int n, int s);
/* S(c,s) = sum_{j<=s} C(c,j): bounded_subset_count (combinatorics.hpp:32-36). */
uint64_t bnmc_gpu_bounded_subset_count(int c, int s);

/* ScoreCache::build on the device: joint-state count tables + BD local scores
 * for every (node, parent set |pi|<=s), then the PPF fold for prior_r.
 * Bit-exact with the reference's canonical build. */
int bnmc_gpu_table_build(const uint8_t* cells, const int* cards, uint64_t m, int n,
                         const bnmc_score_params* params, const double* prior_r,
                         bnmc_table** out);

/* Node-row-sharded build (multi-GPU precompute): allocate the full
 * table but compute only rows [row_begin, row_end). The caller exchanges rows
 * (e.g. an NCCL all-gather over the buffer from bnmc_gpu_table_rows_buffer)
 * and then calls bnmc_gpu_table_finalize. */
int bnmc_gpu_table_build_rows(const uint8_t* cells, const int* cards, uint64_t m, int n,
                              const bnmc_score_params* params, const double* prior_r,
                              int row_begin, int row_end, bnmc_table** out);
/* Work-balanced partition of the precompute into `nparts` parts (host only, no
 * device needed). K1 works per prefix P (|P| <= s) in the global-index order of
 * subsets of the n variables; part g owns prefix indices [cuts[g], cuts[g+1])
 * (cuts: nparts + 1 values) and with them every entry (v, pi) whose joint set
 * pi + {v} minus its largest member is such a prefix — the parts' entries are
 * disjoint and cover the table. Replaces the reference's OpenMP row loop over
 * nodes (src/scoring.cpp:179-190) as the unit of parallel work. */
int bnmc_gpu_k1_partition(const int* cards, uint64_t m, int n, int s, int nparts,
                          uint64_t* cuts);

/* Multi-GPU precompute, one part per GPU: allocate the full table, zero it and
 * compute the entries of part `part` of bnmc_gpu_k1_partition(nparts). The
 * parts combine by an integer (bitwise-exact) sum of the 64-bit table words,
 * e.g. ncclAllReduce(ncclInt64, ncclSum) over bnmc_gpu_table_rows_buffer, or
 * bnmc_gpu_table_build_comm which does this internally; then
 * bnmc_gpu_table_finalize. */
int bnmc_gpu_table_build_part(const uint8_t* cells, const int* cards, uint64_t m, int n,
                              const bnmc_score_params* params, const double* prior_r, int part,
                              int nparts, bnmc_table** out);

/* Multi-process multi-GPU (one process per GPU, e.g. under torchrun): an
 * NCCL communicator over NVLink/NVSwitch. Rank 0 creates the unique id
 * (NCCL_UNIQUE_ID_BYTES = 128 bytes) and ships it to the other ranks out of
 * band (e.g. torch.distributed broadcast); every rank then calls
 * bnmc_gpu_comm_init with its rank and CUDA device. Collective calls below
 * must be made by every rank in the same order. NCCL is loaded at first use
 * (libnccl.so.2; BNMC_NCCL_LIB overrides); failures are status 6. */
int bnmc_gpu_comm_unique_id(uint8_t* id128);
int bnmc_gpu_comm_init(const uint8_t* id128, int nranks, int rank, int device, bnmc_comm** out);
int bnmc_gpu_comm_free(bnmc_comm* comm);
/* ScoreCache::build over a communicator: rank r computes part r of nranks
 * (bnmc_gpu_k1_partition), an in-place ncclAllReduce(int64, sum) of the table
 * words completes it on every rank (bit-exact: each entry has one writer),
 * then the PPF fold. params->device must be the communicator's device. */
int bnmc_gpu_table_build_comm(const uint8_t* cells, const int* cards, uint64_t m, int n,
                              const bnmc_score_params* params, const double* prior_r,
                              bnmc_comm* comm, bnmc_table** out);
/* All-gather of `bytes` of host data per rank (e.g. fixed-size chain records)
 * through device buffers: recv receives nranks * bytes in rank order. */
int bnmc_gpu_comm_allgather(bnmc_comm* comm, const void* send, uint64_t bytes, void* recv);
/* Element-wise max over ranks of `count` doubles, in place (timings). */
int bnmc_gpu_comm_allreduce_max(bnmc_comm* comm, double* values, int count);
/* Devices a table spans (1 unless built with n_gpus > 1) and their ordinals. */
int bnmc_gpu_table_devices(const bnmc_table* t, int* count, int* devices /* >= count */);

/* Last precompute run on this table: K1 + K1W device time (ms), entries scored
 * by the wide path (joint spaces beyond the dense counter) and the prefix
 * index range computed. */
int bnmc_gpu_table_k1_stats(const bnmc_table* t, float* k1_ms, uint64_t* wide_entries,
                            uint64_t* prefix_lo, uint64_t* prefix_hi);

/* Device pointer and byte size of the fp64 local-score rows (n x S doubles,
 * contiguous, row stride S). Valid until bnmc_gpu_table_free. */
int bnmc_gpu_table_rows_buffer(bnmc_table* t, void** dev_ptr, uint64_t* bytes,
                               uint64_t* row_stride_elems);
/* Rebuild the derived scan table after rows were written externally. */
int bnmc_gpu_table_finalize(bnmc_table* t);

/* Prebuilt cache: host table in BNSC body order (e.g. from ScoreCache::load). */
int bnmc_gpu_table_upload(const double* table, int n, const bnmc_score_params* params,
                          const double* prior_r, bnmc_table** out);
/* Replace the pairwise prior (re-folds the PPF into the scan table). */
int bnmc_gpu_table_set_priors(bnmc_table* t, const double* prior_r);
int bnmc_gpu_table_info(const bnmc_table* t, int* n, int* s, uint64_t* entries_per_node);
/* Local scores (no PPF) back to the host in BNSC body order: n * S doubles. */
int bnmc_gpu_table_download(const bnmc_table* t, double* out);
/* Device-side timings of the last build: count+score kernel and PPF fold, ms. */
int bnmc_gpu_table_build_ms(const bnmc_table* t, float* count_score_ms, float* fold_ms);
int bnmc_gpu_table_free(bnmc_table* t);

/* count_statistics for `count` (node, pset) pairs on the device (same kernel
 * code as the build). out receives, for entry e, r_e * cards[node_e] u32 cells
 * at out + offsets[e] (offsets computed by the caller as the prefix sum of
 * r_e * card, configs_out[e] = r_e). */
int bnmc_gpu_count_statistics(const uint8_t* cells, const int* cards, uint64_t m, int n,
                              int count, const int* nodes, const uint64_t* psets,
                              const uint64_t* offsets, uint32_t* out,
                              uint64_t* configs_out, int device);

/* count_statistics as the reference's CountTable iterates it (for_each_active,
 * scoring.hpp:55-67; dense or ordered-map storage, scoring.cpp:53-80): the
 * active parent configurations of (node, pset) ascending, written to
 * configs_out (capacity m), with their card(node) state counts in counts_out
 * (capacity m * card(node)); *n_active receives their number. No limit on the
 * configuration space other than the reference's 64-bit overflow check
 * (status 4, "parent configuration space overflows 64 bits"). */
int bnmc_gpu_count_statistics_sparse(const uint8_t* cells, const int* cards, uint64_t m, int n,
                                     int node, uint64_t pset, uint64_t* configs_out,
                                     uint32_t* counts_out, uint64_t* n_active, int device);

/* OrderScorer::score for `count` orders (perms: count x n positions->node).
 * Outputs per order: parent masks (n, indexed by node), per-node effective
 * best (n, by node) and the total summed in ascending node order. Any output
 * pointer may be NULL. Bit-exact with the reference (tie rule included). */
int bnmc_gpu_score_orders(bnmc_table* t, const int* perms, int count, uint64_t* masks_out,
                          double* best_out, double* totals_out);
int bnmc_gpu_score_order(bnmc_table* t, const int* perm, uint64_t* masks_out,
                         double* best_out, double* total_out);

/* OrderScorer::scan_slice (engine.hpp:83, engine.cpp:43-58): argmax of the
 * effective score (lookup + PpfTable::sum, with the table's bound priors) over
 * PST indices [lo, hi) of the subsets of positions 0..position-1 of `perm`
 * (the node at `position`); ties keep the smallest index. An empty slice
 * yields score -inf and idx UINT64_MAX (the ArgmaxCell identity). */
int bnmc_gpu_scan_slice(bnmc_table* t, const int* perm, int position, uint64_t lo, uint64_t hi,
                        double* score_out, uint64_t* idx_out);

/* run_mcmc parameters (RunConfig fields of the sampler). */
typedef struct {
  uint64_t iterations; /* >= 1 */
  int track_top;       /* BestGraphTracker capacity, >= 1 */
  int strict;          /* RunConfig::strict_paper_tracker */
  int scan_mode;       /* 0 = auto (= 2); 1 = full-row scan: fp32 keys streamed per
                          rescanned row + exact fp64 resolve, CUDA-Graph loop, <= 64
                          chains per call; 2 = sorted-row walk: fused device-resident
                          chains, one CTA per chain, any number of chains */
  int timing_sample;   /* every k-th scan launch is bracketed by CUDA events (0 = 8) */
  int team_warps;      /* sorted walk: warps per chain (0 auto, 1, 2, 4, 8) */
  int exact_accept;    /* sorted walk: 0 = device log10 for mh_accept, chains with a
                          decision inside the CUDA/glibc log10 error bound replayed
                          with host glibc thresholds; 1 = host glibc thresholds only */
  int accept_tol_log2; /* relative bound of that test as a power of two (0 = -48) */
  int debug_recheck;   /* RunConfig::debug_recheck (sampler.cpp:105-110): every 100
                          iterations each chain re-scores its current order from
                          scratch (full rows, no incremental state) on the device
                          and fails with status 1 ("chain score drifted ...") when
                          the total differs; sorted-walk path only */
} bnmc_chain_params;

/* Run n_chains independent chains, chain c seeded with seeds[c] exactly as
 * run_mcmc(data, cfg{seed=seeds[c]}, priors, prebuilt=table), in lockstep on
 * the device (CUDA-Graph / persistent loop, no per-iteration host round trip).
 * Host outputs (any may be NULL), chain-major:
 *   trace_proposed[c*iters + t], trace_accepted[..], trace_best[..]  (TraceRow)
 *   final_order[c*n + p], final_score[c], accepted[c]
 *   tracker_count[c], tracker_masks[(c*K + e)*n + node], tracker_totals[c*K + e]
 * device_ms (optional) receives the device time of the sampling loop. */
int bnmc_gpu_run_chains(bnmc_table* t, const uint64_t* seeds, int n_chains,
                        const bnmc_chain_params* params, double* trace_proposed,
                        uint8_t* trace_accepted, double* trace_best, int* final_order,
                        double* final_score, uint64_t* accepted, int* tracker_count,
                        uint64_t* tracker_masks, double* tracker_totals, float* device_ms);

/* Statistics of the last run_chains call: node-row rescans (summed over
 * chains and iterations), 16-byte key slots streamed by the scan kernel
 * (after batching chains per row and skipping sectors no pair can admit), the
 * average device time of one scan launch (CUDA events around every
 * timing_sample-th launch inside the loop, ms) and the number of kernel
 * launches of the loop (scan_mode 1; for the walk path sectors = entries
 * visited and scan_ms = the fused kernel's time). */
int bnmc_gpu_last_scan_stats(const bnmc_table* t, uint64_t* row_rescans, uint64_t* sectors,
                             float* scan_ms_avg, uint64_t* kernel_launches);

/* Scan algorithm used by bnmc_gpu_score_order(s) on this table (0 auto = 2
 * sorted walk, 1 full-row scan, 2 sorted walk). Results are identical. */
int bnmc_gpu_table_set_scan_mode(bnmc_table* t, int mode);

/* Sorted-walk tuning (results are identical for every setting): rows whose
 * predecessor count p has S(p,s) <= enum_max are enumerated in PST order, the
 * others walked (enum_max < 0: default 64); ylists -1 auto / 0 off / 1 on
 * selects the per-(row, node) lists used by delta walks. */
int bnmc_gpu_table_set_walk_params(bnmc_table* t, int64_t enum_max, int ylists);

/* Capped walks (results are identical for every setting): rows with
 * enum_max < S(p,s) <= walk_cap walk at most budget * S(p,s) sorted entries
 * and then enumerate PST(p) (bounds the deep walks of rows with few
 * predecessors). walk_cap < 0: default S(n-1,s) / 512; budget < 0: default
 * 16; budget 0 disables the cap. deep: entries per lane per deep walk round
 * for chains of fewer than 8 warps, -1 auto (8 for rows longer than 2^21
 * entries, else 4), 0 -> 4, 1 -> 8. */
int bnmc_gpu_table_set_walk_cap(bnmc_table* t, int64_t walk_cap, int64_t budget, int deep);

/* Statistics of the last sorted-walk run_chains call: (chain, row) pairs
 * rescanned, sorted entries walked, PST entries enumerated (small predecessor
 * counts), and the device time of the last per-row sort build (ms). */
int bnmc_gpu_last_walk_stats(const bnmc_table* t, uint64_t* pairs, uint64_t* walked,
                             uint64_t* enumerated, float* sort_ms);

/* Kernel variant of the last sorted-walk launch (run_chains or score_orders):
 * warps per chain, entries per lane in a deep walk round (4 or 8), and
 * whether the speculative single-chain kernel ran (walk_spec_kernel). */
int bnmc_gpu_last_walk_variant(const bnmc_table* t, int* team_warps, int* entries_per_lane,
                               int* speculative);

/* Chains of the last sorted-walk run_chains call that were replayed with host
 * glibc acceptance thresholds (an mh_accept decision fell inside the bound). */
int bnmc_gpu_last_replayed(const bnmc_table* t, uint64_t* chains);

/* Diagnostics: time the order-scan kernel (K2) alone on the rows at positions
 * lo..hi of `count` (<= 64) orders: `reps` launches, each timed with CUDA
 * events and, when flush_l2 != 0, preceded by a 256 MiB write (cold L2).
 * Outputs the mean launch time (ms) and the key bytes streamed per launch
 * (16-byte slots actually loaded x 16; may be NULL). */
int bnmc_gpu_bench_scan(bnmc_table* t, const int* perms, int count, int lo, int hi, int reps,
                        int flush_l2, float* ms_per_launch, uint64_t* key_bytes_per_launch);

#ifdef __cplusplus
}
#endif
#endif
