/* TEST INFRASTRUCTURE — plain-C restatement of the reference hot path.
 * See bnmc_oracle.h. Paths cited are relative to /root/reference/proj.
 * Compiled with -ffp-contract=off and no -march so that, like the reference's
 * canonical Release build, no FMA contraction changes floating-point bits.
 */
#include "bnmc_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ RNG */
/* Rng::mix (rng.hpp:77-81) */
static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

orc_rng orc_rng_make(uint64_t seed) {
  orc_rng r = {seed};
  return r;
}

/* Rng::split (rng.hpp:21-23) */
orc_rng orc_rng_split(const orc_rng* r, uint64_t tag) {
  orc_rng c = {mix64(r->state + 0x9E3779B97F4A7C15ull * (tag + 1))};
  return c;
}

/* Rng::next_u64 (rng.hpp:25-28) */
uint64_t orc_next_u64(orc_rng* r) {
  r->state += 0x9E3779B97F4A7C15ull;
  return mix64(r->state);
}

/* rng.hpp:31 */
double orc_next_unit(orc_rng* r) { return (double)(orc_next_u64(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:35-37 */
double orc_next_unit_open(orc_rng* r) {
  return ((double)(orc_next_u64(r) >> 11) + 0.5) * 0x1.0p-53;
}

/* rng.hpp:40-45: rejection below 2^64 mod bound */
uint64_t orc_next_below(orc_rng* r, uint64_t bound) {
  const uint64_t threshold = (0 - bound) % bound;
  uint64_t x;
  do {
    x = orc_next_u64(r);
  } while (x < threshold);
  return x % bound;
}

/* Fisher-Yates, rng.hpp:86-90 */
void orc_shuffle_int(int* v, int len, orc_rng* r) {
  for (int i = len; i > 1; --i) {
    const uint64_t j = orc_next_below(r, (uint64_t)i);
    const int t = v[i - 1];
    v[i - 1] = v[j];
    v[j] = t;
  }
}

/* -------------------------------------------------------- combinatorics */
static uint64_t g_pascal[65][65];
static int g_pascal_ready = 0;

static void pascal_init(void) {
  if (g_pascal_ready) return;
  for (int n = 0; n <= 64; ++n) {
    g_pascal[n][0] = 1;
    for (int k = 1; k <= n; ++k) g_pascal[n][k] = g_pascal[n - 1][k - 1] + g_pascal[n - 1][k];
  }
  g_pascal_ready = 1;
}

/* binomial (combinatorics.hpp:27-29) */
uint64_t orc_binomial(int n, int k) {
  pascal_init();
  return (k < 0 || k > n || n < 0) ? 0 : g_pascal[n][k];
}

/* bounded_subset_count (combinatorics.hpp:32-36) */
uint64_t orc_bounded_subset_count(int n, int s) {
  uint64_t t = 0;
  for (int j = 0; j <= s; ++j) t += orc_binomial(n, j);
  return t;
}

/* global_index (combinatorics.cpp:61-76): descending size, then the 0-based
 * lexicographic CNS rank of the mask within its size. */
uint64_t orc_global_index(uint64_t mask, int candidates, int s) {
  const int k = __builtin_popcountll(mask);
  uint64_t offset = 0;
  for (int j = k + 1; j <= s; ++j) offset += orc_binomial(candidates, j);
  uint64_t rank = 0;
  int prev = 0, pos = 1;
  for (uint64_t m = mask; m != 0; m &= m - 1, ++pos) {
    const int a = __builtin_ctzll(m) + 1;
    rank += orc_binomial(candidates - prev, k - pos + 1) -
            orc_binomial(candidates - a + 1, k - pos + 1);
    prev = a;
  }
  return offset + rank;
}

/* unrank_combination (combinatorics.cpp:8-39), 1-based elements → bitmask of
 * 0-based positions (subset_at, combinatorics.cpp:78-90). */
static uint64_t unrank_mask(int n, int k, uint64_t l) {
  const int total = k;
  uint64_t mask = 0;
  int low = 0;
  for (int pos = 0; pos + 1 < total; ++pos) {
    uint64_t sum = 0;
    int shift = 1;
    for (; shift <= n; ++shift) {
      const uint64_t block = orc_binomial(n - shift, k - 1);
      if (sum + block < l)
        sum += block;
      else
        break;
    }
    const int e = low + shift;
    mask |= 1ull << (e - 1);
    n -= shift;
    k -= 1;
    l -= sum;
    low = e;
  }
  if (total > 0) mask |= 1ull << (low + (int)l - 1);
  return mask;
}

uint64_t orc_subset_at(uint64_t index, int candidates, int s) {
  for (int k = s < candidates ? s : candidates; k >= 0; --k) {
    const uint64_t block = orc_binomial(candidates, k);
    if (index < block) return unrank_mask(candidates, k, index + 1);
    index -= block;
  }
  return ~0ull; /* out of range */
}

/* enumerate_bounded_position_sets (combinatorics.hpp:83-101): sizes
 * min(s,c)..1 by the lexicographic successor rule, then the empty set. */
void orc_build_pst(int candidates, int s, uint64_t* out) {
  uint64_t g = 0;
  int a[64];
  for (int k = s < candidates ? s : candidates; k >= 1; --k) {
    for (int i = 0; i < k; ++i) a[i] = i;
    for (;;) {
      uint64_t p = 0;
      for (int i = 0; i < k; ++i) p |= 1ull << a[i];
      out[g++] = p;
      int i = k - 1;
      while (i >= 0 && a[i] == candidates - k + i) --i;
      if (i < 0) break;
      ++a[i];
      for (int j = i + 1; j < k; ++j) a[j] = a[j - 1] + 1;
    }
  }
  out[g] = 0;
}

/* ScoreCache::index_of (scoring.hpp:133-139) */
uint64_t orc_index_of(int n, int s, int node, uint64_t pset) {
  const uint64_t low = pset & ((1ull << node) - 1);
  const uint64_t high = node + 1 < 64 ? (pset >> (node + 1)) << node : 0;
  return orc_global_index(low | high, n - 1, s);
}

/* --------------------------------------------------------------- scoring */
static double log10_gamma(double x) { return lgamma(x) * 0.43429448190325182765; }

/* Parent-configuration space r = prod card(parent), scoring.cpp:89-95. */
static int config_space(const int* cards, uint64_t pset, uint64_t* r_out) {
  uint64_t r = 1;
  for (uint64_t m = pset; m; m &= m - 1) {
    const uint64_t card = (uint64_t)cards[__builtin_ctzll(m)];
    if (r > UINT64_MAX / card) return fail(ORC_CAPACITY, "parent configuration space overflows 64 bits");
    r *= card;
  }
  *r_out = r;
  return ORC_OK;
}

/* Mixed-radix configuration index, lowest parent least significant
 * (scoring.cpp:99-105). */
static uint64_t config_of(const uint8_t* row, const int* cards, uint64_t pset) {
  uint64_t k = 0, radix = 1;
  for (uint64_t m = pset; m; m &= m - 1) {
    const int p = __builtin_ctzll(m);
    k += radix * row[p];
    radix *= (uint64_t)cards[p];
  }
  return k;
}

int orc_count_statistics(const uint8_t* cells, const int* cards, int n, uint64_t m,
                         int node, uint64_t pset, uint32_t* out, uint64_t cap,
                         uint64_t* configs_out) {
  if ((pset >> node) & 1u) return fail(ORC_DATA, "node cannot appear in its own parent set");
  uint64_t r;
  int st = config_space(cards, pset, &r);
  if (st) return st;
  const int card = cards[node];
  if (r > cap / (uint64_t)card) return fail(ORC_CAPACITY, "count table larger than buffer");
  *configs_out = r;
  memset(out, 0, sizeof(uint32_t) * r * card);
  for (uint64_t t = 0; t < m; ++t) {
    const uint8_t* row = cells + t * (uint64_t)n;
    out[config_of(row, cards, pset) * card + row[node]]++;
  }
  return ORC_OK;
}

typedef struct {
  uint64_t cfg;
  uint32_t state;
} cfg_state;

static int cmp_cfg_state(const void* a, const void* b) {
  const cfg_state* x = (const cfg_state*)a;
  const cfg_state* y = (const cfg_state*)b;
  if (x->cfg != y->cfg) return x->cfg < y->cfg ? -1 : 1;
  return (int)x->state - (int)y->state;
}

/* local_score_from_counts (scoring.cpp:111-135) over the active configs in
 * ascending order. The per-config body is restated exactly: inner accumulates
 * lG(c + a_cell) - lG(a_cell) over states with c > 0, then
 * score += (lG(a_row) - lG(a_row + N_ik)) + inner. */
static void score_config(const uint32_t* counts, int card, double a_cell, double a_row,
                         double lg_row, double lg_cell, double* score) {
  uint32_t n_ik = 0;
  double inner = 0.0;
  for (int j = 0; j < card; ++j) {
    const uint32_t c = counts[j];
    if (c > 0) {
      inner += log10_gamma((double)c + a_cell) - lg_cell;
      n_ik += c;
    }
  }
  *score += lg_row - log10_gamma(a_row + (double)n_ik) + inner;
}

int orc_local_score(const uint8_t* cells, const int* cards, int n, uint64_t m,
                    int node, uint64_t pset, double gamma, double ess, int k2,
                    double* out) {
  if ((pset >> node) & 1u) return fail(ORC_DATA, "node cannot appear in its own parent set");
  uint64_t r;
  int st = config_space(cards, pset, &r);
  if (st) return st;
  const int card = cards[node];
  /* Hyperparams::alpha_cell (scoring.hpp:27-31) */
  const double a_cell = k2 ? 1.0 : ess / ((double)r * card);
  if (!(a_cell > 0.0)) return fail(ORC_USAGE, "Dirichlet hyperparameter must be positive");
  const double a_row = a_cell * card;
  const double lg_row = log10_gamma(a_row);
  const double lg_cell = log10_gamma(a_cell);
  double score = (double)__builtin_popcountll(pset) * log10(gamma);

  /* CountTable: dense up to 2^22 cells (scoring.cpp:13, 53-57), else sparse;
   * either way configs are visited ascending and empty ones skipped. */
  if (r <= (1ull << 22) / (uint64_t)card) {
    uint32_t* cnt = (uint32_t*)calloc(r * card, sizeof(uint32_t));
    if (!cnt) return fail(ORC_CAPACITY, "out of memory");
    for (uint64_t t = 0; t < m; ++t) {
      const uint8_t* row = cells + t * (uint64_t)n;
      cnt[config_of(row, cards, pset) * card + row[node]]++;
    }
    for (uint64_t k = 0; k < r; ++k) {
      const uint32_t* c = cnt + k * card;
      uint32_t rowsum = 0;
      for (int j = 0; j < card; ++j) rowsum += c[j];
      if (rowsum > 0) score_config(c, card, a_cell, a_row, lg_row, lg_cell, &score);
    }
    free(cnt);
  } else {
    cfg_state* ks = (cfg_state*)malloc(sizeof(cfg_state) * (m ? m : 1));
    uint32_t* c = (uint32_t*)calloc((size_t)card, sizeof(uint32_t));
    if (!ks || !c) return fail(ORC_CAPACITY, "out of memory");
    for (uint64_t t = 0; t < m; ++t) {
      const uint8_t* row = cells + t * (uint64_t)n;
      ks[t].cfg = config_of(row, cards, pset);
      ks[t].state = row[node];
    }
    qsort(ks, m, sizeof(cfg_state), cmp_cfg_state);
    for (uint64_t t = 0; t < m;) {
      uint64_t u = t;
      memset(c, 0, sizeof(uint32_t) * card);
      while (u < m && ks[u].cfg == ks[t].cfg) c[ks[u++].state]++;
      score_config(c, card, a_cell, a_row, lg_row, lg_cell, &score);
      t = u;
    }
    free(ks);
    free(c);
  }
  *out = score;
  return ORC_OK;
}

/* ppf (scoring.cpp:143-148) */
double orc_ppf(double r) {
  const double d = r - 0.5;
  return 100.0 * d * d * d;
}

static int validate_cfg(int s, double gamma, double ess) {
  /* RunConfig::validate (types.cpp:111-121), the fields the build reads */
  if (s < 0 || s > 8) return fail(ORC_USAGE, "max-parents must lie in [0,8]");
  if (!(gamma > 0.0 && gamma <= 1.0)) return fail(ORC_USAGE, "gamma must lie in (0,1]");
  if (!(ess > 0.0)) return fail(ORC_USAGE, "ess must be positive");
  return ORC_OK;
}

/* ScoreCache::build (scoring.cpp:162-192) */
int orc_cache_build(const uint8_t* cells, const int* cards, int n, uint64_t m,
                    int s, double gamma, double ess, int k2, int threads,
                    double* table) {
  int st = validate_cfg(s, gamma, ess);
  if (st) return st;
  const uint64_t per = orc_bounded_subset_count(n - 1, s);
  uint64_t* pst = (uint64_t*)malloc(sizeof(uint64_t) * per);
  if (!pst) return fail(ORC_CAPACITY, "out of memory");
  orc_build_pst(n - 1, s, pst);
  int err = 0;
#pragma omp parallel for num_threads(threads > 0 ? threads : 1) schedule(dynamic)
  for (int node = 0; node < n; ++node) {
    int cand[64], c = 0;
    for (int v = 0; v < n; ++v)
      if (v != node) cand[c++] = v;
    for (uint64_t g = 0; g < per; ++g) {
      uint64_t pset = 0;
      for (uint64_t pm = pst[g]; pm; pm &= pm - 1) pset |= 1ull << cand[__builtin_ctzll(pm)];
      if (orc_local_score(cells, cards, n, m, node, pset, gamma, ess, k2,
                          &table[(uint64_t)node * per + g]) != ORC_OK)
        err = 1;
    }
  }
  free(pst);
  return err ? ORC_CAPACITY : ORC_OK;
}

/* ---------------------------------------------------------------- orders */
static void ppf_table(const double* prior_r, int n, double* w) {
  /* PpfTable (scoring.cpp:150-155); zero diagonal */
  for (int i = 0; i < n; ++i)
    for (int m = 0; m < n; ++m)
      w[i * n + m] = (prior_r && i != m) ? orc_ppf(prior_r[i * n + m]) : 0.0;
}

/* PpfTable::sum (scoring.hpp:103-107): ascending parents, from 0.0 */
static double ppf_sum(const double* w, int n, int child, uint64_t pset) {
  double t = 0.0;
  for (uint64_t m = pset; m; m &= m - 1) t += w[child * n + __builtin_ctzll(m)];
  return t;
}

/* One order scan with a prebuilt PST for every predecessor count. */
typedef struct {
  int n, s;
  uint64_t per;
  const double* table;
  double* w;
  uint64_t** pst; /* pst[p] = build_pst(p, s) */
  uint64_t* pst_len;
} scorer_t;

static int scorer_init(scorer_t* sc, const double* table, int n, int s, const double* prior_r) {
  sc->n = n;
  sc->s = s;
  sc->per = orc_bounded_subset_count(n - 1, s);
  sc->table = table;
  sc->w = (double*)malloc(sizeof(double) * n * n);
  sc->pst = (uint64_t**)calloc(n, sizeof(uint64_t*));
  sc->pst_len = (uint64_t*)calloc(n, sizeof(uint64_t));
  if (!sc->w || !sc->pst || !sc->pst_len) return fail(ORC_CAPACITY, "out of memory");
  ppf_table(prior_r, n, sc->w);
  for (int p = 0; p < n; ++p) {
    sc->pst_len[p] = orc_bounded_subset_count(p, s);
    sc->pst[p] = (uint64_t*)malloc(sizeof(uint64_t) * sc->pst_len[p]);
    if (!sc->pst[p]) return fail(ORC_CAPACITY, "out of memory");
    orc_build_pst(p, s, sc->pst[p]);
  }
  return ORC_OK;
}

static void scorer_free(scorer_t* sc) {
  for (int p = 0; p < sc->n; ++p) free(sc->pst[p]);
  free(sc->pst);
  free(sc->pst_len);
  free(sc->w);
}

/* score_order (scoring.cpp:261-289): predecessor subsets streamed in
 * global-index order over the predecessor POSITIONS; strict '>' keeps the
 * first maximum (the tie rule of SURVEY §8.1.2). */
static void scorer_score(const scorer_t* sc, const int* perm, uint64_t* masks, double* best_by_node,
                         double* total) {
  const int n = sc->n;
  for (int p = 0; p < n; ++p) {
    const int node = perm[p];
    double best = -INFINITY;
    uint64_t best_set = 0;
    for (uint64_t g = 0; g < sc->pst_len[p]; ++g) {
      uint64_t pset = 0; /* apply_candidates (combinatorics.hpp:73-79) */
      for (uint64_t pm = sc->pst[p][g]; pm; pm &= pm - 1) pset |= 1ull << perm[__builtin_ctzll(pm)];
      const double eff = sc->table[(uint64_t)node * sc->per + orc_index_of(n, sc->s, node, pset)] +
                         ppf_sum(sc->w, n, node, pset);
      if (eff > best) {
        best = eff;
        best_set = pset;
      }
    }
    masks[node] = best_set;
    best_by_node[node] = best;
  }
  double t = 0.0; /* ascending node order (scoring.cpp:285-286) */
  for (int i = 0; i < n; ++i) t += best_by_node[i];
  *total = t;
}

int orc_score_order(const double* table, int n, int s, const double* prior_r,
                    const int* perm, uint64_t* masks_out, double* best_out,
                    double* total_out) {
  scorer_t sc;
  int st = scorer_init(&sc, table, n, s, prior_r);
  if (st) return st;
  double* best = best_out ? best_out : (double*)malloc(sizeof(double) * n);
  scorer_score(&sc, perm, masks_out, best, total_out);
  if (!best_out) free(best);
  scorer_free(&sc);
  return ORC_OK;
}

/* --------------------------------------------------------------- sampler */
typedef struct {
  int cap, count, n;
  uint64_t* masks; /* cap * n */
  double* totals;
} tracker_t;

/* Dag operator< : lexicographic over the n parent masks (types.hpp:140-142) */
static int dag_less(const uint64_t* a, const uint64_t* b, int n) {
  for (int i = 0; i < n; ++i)
    if (a[i] != b[i]) return a[i] < b[i];
  return 0;
}

/* precedes (sampler.cpp:16-19) */
static int precedes(double ta, const uint64_t* a, double tb, const uint64_t* b, int n) {
  if (ta != tb) return ta > tb;
  return dag_less(a, b, n);
}

/* BestGraphTracker::update (sampler.cpp:32-41) */
static int tracker_update(tracker_t* t, const uint64_t* masks, double total) {
  const int n = t->n;
  for (int e = 0; e < t->count; ++e)
    if (memcmp(t->masks + (uint64_t)e * n, masks, sizeof(uint64_t) * n) == 0) return 0;
  const int full = t->count == t->cap;
  if (full && total <= t->totals[t->count - 1]) return 0;
  int pos = 0; /* lower_bound: first entry that does not precede g */
  while (pos < t->count && precedes(t->totals[pos], t->masks + (uint64_t)pos * n, total, masks, n))
    ++pos;
  const int last = full ? t->count - 1 : t->count;
  for (int e = last; e > pos; --e) {
    t->totals[e] = t->totals[e - 1];
    memcpy(t->masks + (uint64_t)e * n, t->masks + (uint64_t)(e - 1) * n, sizeof(uint64_t) * n);
  }
  t->totals[pos] = total;
  memcpy(t->masks + (uint64_t)pos * n, masks, sizeof(uint64_t) * n);
  if (!full) t->count++;
  return 1;
}

/* run_mcmc (sampler.cpp:58-116) with a prebuilt cache: streams split(1)
 * initial order, split(2) proposals, split(3) acceptance. */
int orc_run_mcmc(const double* table, int n, int s, const double* prior_r,
                 const orc_mcmc_cfg* cfg, double* trace_proposed,
                 uint8_t* trace_accepted, double* trace_best, int* final_order,
                 double* final_score, uint64_t* accepted, int* tracker_count,
                 uint64_t* tracker_masks, double* tracker_totals) {
  if (cfg->iterations < 1) return fail(ORC_USAGE, "iterations must be >= 1");
  if (cfg->track_top < 1) return fail(ORC_USAGE, "tracker capacity must be >= 1");
  if (n < 2) return fail(ORC_USAGE, "swap proposal needs at least two nodes");
  scorer_t sc;
  int st = scorer_init(&sc, table, n, s, prior_r);
  if (st) return st;
  tracker_t tr = {cfg->track_top, 0, n, tracker_masks, tracker_totals};
  const orc_rng master = orc_rng_make(cfg->seed);
  orc_rng init = orc_rng_split(&master, 1);
  orc_rng prop = orc_rng_split(&master, 2);
  orc_rng acc = orc_rng_split(&master, 3);

  int order[64], proposed[64];
  for (int i = 0; i < n; ++i) order[i] = i;
  orc_shuffle_int(order, n, &init);
  uint64_t cur_masks[64], new_masks[64];
  double best[64], cur_total, new_total;
  scorer_score(&sc, order, cur_masks, best, &cur_total);
  tracker_update(&tr, cur_masks, cur_total);
  uint64_t acc_count = 0;
  for (uint64_t it = 1; it <= cfg->iterations; ++it) {
    /* propose_swap (sampler.cpp:43-52) */
    const int a = (int)orc_next_below(&prop, (uint64_t)n);
    int b = (int)orc_next_below(&prop, (uint64_t)(n - 1));
    if (b >= a) ++b;
    memcpy(proposed, order, sizeof(int) * n);
    const int t = proposed[a];
    proposed[a] = proposed[b];
    proposed[b] = t;
    scorer_score(&sc, proposed, new_masks, best, &new_total);
    /* mh_accept (sampler.cpp:54-56) */
    const int ok = log10(orc_next_unit_open(&acc)) < new_total - cur_total;
    if (ok || !cfg->strict) tracker_update(&tr, new_masks, new_total);
    if (ok) {
      memcpy(order, proposed, sizeof(int) * n);
      memcpy(cur_masks, new_masks, sizeof(uint64_t) * n);
      cur_total = new_total;
      ++acc_count;
    }
    if (trace_proposed) trace_proposed[it - 1] = new_total;
    if (trace_accepted) trace_accepted[it - 1] = (uint8_t)ok;
    if (trace_best) trace_best[it - 1] = tr.totals[0];
  }
  memcpy(final_order, order, sizeof(int) * n);
  *final_score = cur_total;
  *accepted = acc_count;
  *tracker_count = tr.count;
  scorer_free(&sc);
  return ORC_OK;
}
