/* TEST INFRASTRUCTURE — plain-C restatement of the reference hot path.
 *
 * This is the parity CHECKER for the B200 product, not part of it: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 * Each function restates one reference symbol (file:line cited at the
 * definition, paths relative to /root/reference/proj). Parity of this port
 * with the reference itself is pinned by tests/test_oracle.py against golden
 * vectors that oracle/_ref (the unmodified reference) generated
 * (tests/golden/make_golden.py).
 */
#ifndef BNMC_ORACLE_H
#define BNMC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_USAGE = 2, ORC_DATA = 3, ORC_CAPACITY = 4 };

const char* orc_last_error(void);

/* rng.hpp:14-45, 86-90 */
typedef struct { uint64_t state; } orc_rng;
orc_rng orc_rng_make(uint64_t seed);
orc_rng orc_rng_split(const orc_rng* r, uint64_t tag);
uint64_t orc_next_u64(orc_rng* r);
double orc_next_unit(orc_rng* r);
double orc_next_unit_open(orc_rng* r);
uint64_t orc_next_below(orc_rng* r, uint64_t bound);
void orc_shuffle_int(int* v, int len, orc_rng* r);

/* combinatorics.hpp:14-36, combinatorics.cpp:61-90 */
uint64_t orc_binomial(int n, int k);
uint64_t orc_bounded_subset_count(int n, int s);
uint64_t orc_global_index(uint64_t mask, int candidates, int s);
uint64_t orc_subset_at(uint64_t index, int candidates, int s);
/* enumerate_bounded_position_sets order (combinatorics.hpp:83-101) */
void orc_build_pst(int candidates, int s, uint64_t* out);

/* scoring.cpp:82-135 */
int orc_count_statistics(const uint8_t* cells, const int* cards, int n, uint64_t m,
                         int node, uint64_t pset, uint32_t* out, uint64_t cap,
                         uint64_t* configs_out);
int orc_local_score(const uint8_t* cells, const int* cards, int n, uint64_t m,
                    int node, uint64_t pset, double gamma, double ess, int k2,
                    double* out);
double orc_ppf(double r);
/* ScoreCache::build (scoring.cpp:162-192): table[n * S(n-1,s)] in BNSC order */
int orc_cache_build(const uint8_t* cells, const int* cards, int n, uint64_t m,
                    int s, double gamma, double ess, int k2, int threads,
                    double* table);
/* ScoreCache::index_of (scoring.hpp:133-139) */
uint64_t orc_index_of(int n, int s, int node, uint64_t pset);

/* score_order (scoring.cpp:261-289): per-node parent masks, per-node
 * effective bests, total (ascending node order). prior_r may be NULL. */
int orc_score_order(const double* table, int n, int s, const double* prior_r,
                    const int* perm, uint64_t* masks_out, double* best_out,
                    double* total_out);

/* run_mcmc (sampler.cpp:58-116) on a prebuilt table. */
typedef struct {
  uint64_t iterations, seed;
  int track_top, strict;
} orc_mcmc_cfg;
int orc_run_mcmc(const double* table, int n, int s, const double* prior_r,
                 const orc_mcmc_cfg* cfg, double* trace_proposed,
                 uint8_t* trace_accepted, double* trace_best, int* final_order,
                 double* final_score, uint64_t* accepted, int* tracker_count,
                 uint64_t* tracker_masks, double* tracker_totals);

#ifdef __cplusplus
}
#endif
#endif
