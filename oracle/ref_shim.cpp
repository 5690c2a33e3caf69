// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// extern "C" shim over the UNMODIFIED reference library (compiled in place from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libbnmc_ref.so).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load it. It exists so that Python tests can
//   * generate golden fixtures from the reference itself,
//   * time the reference CPU path (bench.py --impl reference), and
//   * cross-check the plain-C restatement in oracle/bnmc_oracle.c.
// Every entry point calls the reference's own public API (no logic here beyond
// marshalling): see the cited reference symbols.

#include <omp.h>

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <fstream>
#include <numeric>
#include <string>
#include <vector>

#include "bnmc/combinatorics.hpp"
#include "bnmc/engine.hpp"
#include "bnmc/evalgen.hpp"
#include "bnmc/io.hpp"
#include "bnmc/rng.hpp"
#include "bnmc/sampler.hpp"
#include "bnmc/scoring.hpp"
#include "bnmc/types.hpp"

using namespace bnmc;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const UsageError& e) {
    g_err = e.what();
    return 2;
  } catch (const DataError& e) {
    g_err = e.what();
    return 3;
  } catch (const CapacityError& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

Dataset make_dataset(const std::uint8_t* cells, const int* cards, int n,
                     std::uint64_t m) {
  std::vector<int> c(cards, cards + n);
  std::vector<std::uint8_t> rows(cells, cells + m * static_cast<std::uint64_t>(n));
  return Dataset(std::move(c), std::move(rows));
}

PriorMatrix make_priors(const double* r, int n) {
  if (!r) return PriorMatrix::neutral(n);
  return PriorMatrix(n, std::vector<double>(r, r + static_cast<std::size_t>(n) * n));
}

RunConfig make_cfg(int s, double gamma, double ess, int k2, int workers,
                   std::uint64_t mem_cap) {
  RunConfig cfg;
  cfg.max_parents = s;
  cfg.gamma = gamma;
  cfg.ess = ess;
  cfg.alpha_mode = k2 ? AlphaMode::kK2 : AlphaMode::kBdeu;
  cfg.workers = workers;
  cfg.memory_cap_bytes = mem_cap;
  return cfg;
}

struct Scorer {
  PriorMatrix priors;
  OrderScorer scorer;
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
int ref_max_threads() { return omp_get_max_threads(); }

// Synthetic instance exactly as `bnmc generate` / SURVEY §8d builds it:
// master=Rng(seed); random_dag(split(tag_dag)); random_ground_truth(split(tag_cpt));
// forward_sample(split(tag_rows)) (proj/tools/bnmc.cpp:64-73, evalgen.cpp:38-109).
int ref_generate(int n, int max_parents, double edge_prob, double concentration,
                 std::uint64_t m, const int* cards, std::uint64_t seed,
                 std::uint64_t tag_dag, std::uint64_t tag_cpt,
                 std::uint64_t tag_rows, std::uint8_t* cells_out,
                 std::uint64_t* truth_out) {
  return guarded([&] {
    const Rng master(seed);
    Rng dag_rng = master.split(tag_dag);
    Rng cpt_rng = master.split(tag_cpt);
    Rng row_rng = master.split(tag_rows);
    const Dag truth = random_dag(n, max_parents, edge_prob, dag_rng);
    const GroundTruthBn bn = random_ground_truth(
        truth, std::vector<int>(cards, cards + n), concentration, cpt_rng);
    const Dataset d = forward_sample(bn, m, row_rng);
    std::memcpy(cells_out, d.cells().data(), d.cells().size());
    for (int i = 0; i < n; ++i) truth_out[i] = truth.parents(i).mask;
  });
}

// Prior matrix of SURVEY §8d (stream tag 104 of the same master seed).
int ref_synth_priors(int n, const std::uint64_t* truth, std::uint64_t seed,
                     std::uint64_t tag, double* r_out) {
  return guarded([&] {
    PriorMatrix pm = PriorMatrix::neutral(n);
    Rng pr = Rng(seed).split(tag);
    for (int c = 0; c < n; ++c)
      for (int p = 0; p < n; ++p) {
        if (p == c) continue;
        if ((truth[c] >> p) & 1u) {
          if (pr.next_unit() < 0.3) pm.set(c, p, 0.75);
        } else {
          if (pr.next_unit() < 0.02) pm.set(c, p, 0.25);
        }
      }
    for (int c = 0; c < n; ++c)
      for (int p = 0; p < n; ++p) r_out[c * n + p] = pm.r(c, p);
  });
}

// ---- L1 combinatorics (combinatorics.cpp) ----
std::uint64_t ref_binomial(int n, int k) { return binomial(n, k); }
std::uint64_t ref_bounded_subset_count(int n, int s) {
  return bounded_subset_count(n, s);
}
std::uint64_t ref_global_index(std::uint64_t mask, int candidates, int s) {
  return global_index(ParentSet{mask}, candidates, s);
}
std::uint64_t ref_subset_at(std::uint64_t index, int candidates, int s) {
  return subset_at(index, candidates, s).mask;
}
int ref_build_pst(int candidates, int s, std::uint64_t* out) {
  return guarded([&] {
    const ParentSetTable t = build_pst(candidates, s);
    std::memcpy(out, t.masks.data(), t.masks.size() * 8);
  });
}

// ---- L0 RNG (rng.hpp) ----
// kind: 0 next_u64, 1 next_unit, 2 next_unit_open (as u64 bits), 3 next_below(arg)
int ref_rng_stream(std::uint64_t seed, std::int64_t tag, int kind,
                   std::uint64_t arg, std::uint64_t count, std::uint64_t* out) {
  return guarded([&] {
    Rng rng = tag < 0 ? Rng(seed) : Rng(seed).split(static_cast<std::uint64_t>(tag));
    for (std::uint64_t i = 0; i < count; ++i) {
      double d;
      switch (kind) {
        case 0: out[i] = rng.next_u64(); break;
        case 1: d = rng.next_unit(); std::memcpy(&out[i], &d, 8); break;
        case 2: d = rng.next_unit_open(); std::memcpy(&out[i], &d, 8); break;
        default: out[i] = rng.next_below(arg); break;
      }
    }
  });
}

int ref_shuffle_identity(int n, std::uint64_t seed, std::int64_t tag, int* out) {
  return guarded([&] {
    Rng rng = tag < 0 ? Rng(seed) : Rng(seed).split(static_cast<std::uint64_t>(tag));
    std::vector<int> perm(n);
    std::iota(perm.begin(), perm.end(), 0);
    shuffle(perm, rng);
    std::memcpy(out, perm.data(), sizeof(int) * n);
  });
}

// ---- L2 scoring (scoring.cpp) ----
int ref_count_statistics(const std::uint8_t* cells, const int* cards, int n,
                         std::uint64_t m, int node, std::uint64_t pset,
                         std::uint32_t* out, std::uint64_t out_cap,
                         std::uint64_t* configs_out) {
  return guarded([&] {
    const Dataset d = make_dataset(cells, cards, n, m);
    const CountTable t = count_statistics(d, node, ParentSet{pset});
    *configs_out = t.configs();
    const std::uint64_t cells_n = t.configs() * t.child_card();
    if (cells_n > out_cap) throw CapacityError("count table larger than buffer");
    for (std::uint64_t k = 0; k < t.configs(); ++k)
      for (int j = 0; j < t.child_card(); ++j)
        out[k * t.child_card() + j] = t.njk(k, j);
  });
}

// count_statistics as CountTable::for_each_active sees it (dense or map
// storage): active configurations ascending with their state counts.
int ref_count_statistics_active(const std::uint8_t* cells, const int* cards, int n,
                                std::uint64_t m, int node, std::uint64_t pset,
                                std::uint64_t* configs_out, std::uint32_t* counts_out,
                                std::uint64_t cap, std::uint64_t* n_active) {
  return guarded([&] {
    const Dataset d = make_dataset(cells, cards, n, m);
    const CountTable t = count_statistics(d, node, ParentSet{pset});
    std::uint64_t k = 0;
    t.for_each_active([&](std::uint64_t cfg, const std::uint32_t* row) {
      if (k >= cap) throw CapacityError("more active configurations than the buffer holds");
      configs_out[k] = cfg;
      for (int j = 0; j < t.child_card(); ++j) counts_out[k * t.child_card() + j] = row[j];
      ++k;
    });
    *n_active = k;
  });
}

int ref_local_score(const std::uint8_t* cells, const int* cards, int n,
                    std::uint64_t m, int node, std::uint64_t pset, double gamma,
                    double ess, int k2, double* out) {
  return guarded([&] {
    const Dataset d = make_dataset(cells, cards, n, m);
    const Hyperparams hp{gamma, ess, k2 ? AlphaMode::kK2 : AlphaMode::kBdeu};
    *out = local_score(node, ParentSet{pset}, d, hp);
  });
}

// local_score over `count` entries on one Dataset (built once, outside the
// timed loop), single thread: the per-entry body of ScoreCache::build
// (scoring.cpp:179-190). *seconds receives the loop's wall time.
int ref_local_score_batch(const std::uint8_t* cells, const int* cards, int n, std::uint64_t m,
                          int count, const int* nodes, const std::uint64_t* psets, double gamma,
                          double ess, int k2, double* out, double* seconds) {
  return guarded([&] {
    const Dataset d = make_dataset(cells, cards, n, m);
    const Hyperparams hp{gamma, ess, k2 ? AlphaMode::kK2 : AlphaMode::kBdeu};
    const auto t0 = std::chrono::steady_clock::now();
    for (int e = 0; e < count; ++e) out[e] = local_score(nodes[e], ParentSet{psets[e]}, d, hp);
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

int ref_ppf(double r, double* out) {
  return guarded([&] { *out = ppf(r); });
}

void* ref_cache_build(const std::uint8_t* cells, const int* cards, int n,
                      std::uint64_t m, int s, double gamma, double ess, int k2,
                      int workers, std::uint64_t mem_cap, int* status) {
  ScoreCache* out = nullptr;
  *status = guarded([&] {
    const Dataset d = make_dataset(cells, cards, n, m);
    out = new ScoreCache(
        ScoreCache::build(d, make_cfg(s, gamma, ess, k2, workers, mem_cap)));
  });
  return out;
}

void* ref_cache_load(const char* path, int s, double gamma, double ess, int k2,
                     int* status) {
  ScoreCache* out = nullptr;
  *status = guarded([&] {
    out = new ScoreCache(ScoreCache::load(
        path, make_cfg(s, gamma, ess, k2, 1, ~std::uint64_t{0})));
  });
  return out;
}

int ref_cache_save(void* h, const char* path) {
  return guarded([&] { static_cast<ScoreCache*>(h)->save(path); });
}
int ref_cache_n(void* h) { return static_cast<ScoreCache*>(h)->n(); }
std::uint64_t ref_cache_per_node(void* h) {
  return static_cast<ScoreCache*>(h)->entries_per_node();
}
void ref_cache_table(void* h, double* out) {
  const ScoreCache& c = *static_cast<ScoreCache*>(h);
  for (int v = 0; v < c.n(); ++v)
    for (std::uint64_t g = 0; g < c.entries_per_node(); ++g)
      out[v * c.entries_per_node() + g] = c.at(v, g);
}
double ref_cache_lookup(void* h, int node, std::uint64_t pset) {
  return static_cast<ScoreCache*>(h)->lookup(node, ParentSet{pset});
}
std::uint64_t ref_estimate_bytes(int n, int s) {
  return ScoreCache::estimate_bytes(n, s);
}
void ref_cache_free(void* h) { delete static_cast<ScoreCache*>(h); }

// ---- L3 engine (engine.cpp) ----
void* ref_scorer_new(void* cache, const double* prior_r, int workers,
                     int tasks_per_node, int use_pst, int* status) {
  Scorer* out = nullptr;
  *status = guarded([&] {
    const ScoreCache& c = *static_cast<ScoreCache*>(cache);
    PriorMatrix pm = make_priors(prior_r, c.n());
    EngineConfig ecfg{workers, tasks_per_node,
                      use_pst ? IndexStrategy::kPst : IndexStrategy::kUnrank};
    out = new Scorer{pm, OrderScorer(c, pm, ecfg)};
  });
  return out;
}

int ref_scorer_score(void* h, const int* perm, int n, std::uint64_t* masks_out,
                     double* total_out) {
  return guarded([&] {
    const ScoredGraph g =
        static_cast<Scorer*>(h)->scorer.score(Order(std::vector<int>(perm, perm + n)));
    for (int i = 0; i < n; ++i) masks_out[i] = g.dag.parents(i).mask;
    *total_out = g.total;
  });
}

void ref_scorer_free(void* h) { delete static_cast<Scorer*>(h); }

// Serial reference score_order (scoring.cpp:261-289).
int ref_score_order(void* cache, const double* prior_r, const int* perm, int n,
                    std::uint64_t* masks_out, double* total_out) {
  return guarded([&] {
    const ScoreCache& c = *static_cast<ScoreCache*>(cache);
    const ScoredGraph g = score_order(Order(std::vector<int>(perm, perm + n)), c,
                                      make_priors(prior_r, c.n()));
    for (int i = 0; i < n; ++i) masks_out[i] = g.dag.parents(i).mask;
    *total_out = g.total;
  });
}

int ref_score_graph(void* cache, const double* prior_r, const std::uint64_t* masks,
                    int n, double* total_out) {
  return guarded([&] {
    const ScoreCache& c = *static_cast<ScoreCache*>(cache);
    std::vector<ParentSet> ps(n);
    for (int i = 0; i < n; ++i) ps[i] = ParentSet{masks[i]};
    *total_out = score_graph(Dag(ps), c, make_priors(prior_r, c.n())).total;
  });
}

// ---- L4 sampler (sampler.cpp) ----
int ref_mh_accept(double old_s, double new_s, std::uint64_t seed, std::int64_t tag,
                  std::uint64_t count, std::uint8_t* out) {
  return guarded([&] {
    Rng rng = tag < 0 ? Rng(seed) : Rng(seed).split(static_cast<std::uint64_t>(tag));
    for (std::uint64_t i = 0; i < count; ++i) out[i] = mh_accept(old_s, new_s, rng);
  });
}

int ref_run_mcmc(const std::uint8_t* cells, const int* cards, int n,
                 std::uint64_t m, int s, double gamma, double ess, int k2,
                 std::uint64_t iterations, std::uint64_t seed, int workers,
                 int track_top, int strict, int use_pst, int tasks_per_node,
                 std::uint64_t mem_cap, int debug_recheck, const double* prior_r,
                 void* prebuilt, double* trace_proposed, std::uint8_t* trace_accepted,
                 double* trace_best, int* final_order, double* final_score,
                 std::uint64_t* accepted, int* tracker_count,
                 std::uint64_t* tracker_masks, double* tracker_totals,
                 double* preprocess_s, double* sampling_s) {
  return guarded([&] {
    const Dataset d = make_dataset(cells, cards, n, m);
    RunConfig cfg = make_cfg(s, gamma, ess, k2, workers, mem_cap);
    cfg.iterations = iterations;
    cfg.seed = seed;
    cfg.track_top = track_top;
    cfg.strict_paper_tracker = strict != 0;
    cfg.use_pst = use_pst != 0;
    cfg.tasks_per_node = tasks_per_node;
    cfg.debug_recheck = debug_recheck != 0;
    const McmcResult r = run_mcmc(d, cfg, make_priors(prior_r, n),
                                  static_cast<const ScoreCache*>(prebuilt));
    for (std::size_t i = 0; i < r.trace.size(); ++i) {
      if (trace_proposed) trace_proposed[i] = r.trace[i].proposed_score;
      if (trace_accepted) trace_accepted[i] = r.trace[i].accepted;
      if (trace_best) trace_best[i] = r.trace[i].best_score;
    }
    for (int i = 0; i < n; ++i) final_order[i] = r.final_order.node_at(i);
    *final_score = r.final_score;
    *accepted = r.accepted;
    const auto& es = r.tracker.entries();
    *tracker_count = static_cast<int>(es.size());
    for (std::size_t e = 0; e < es.size(); ++e) {
      tracker_totals[e] = es[e].total;
      for (int i = 0; i < n; ++i) tracker_masks[e * n + i] = es[e].dag.parents(i).mask;
    }
    *preprocess_s = r.preprocess_seconds;
    *sampling_s = r.sampling_seconds;
  });
}

// ---- L6 driver steps (tools/bnmc.cpp), restated with the reference's own io.cpp
// writers so CLI outputs of the B200 build can be compared byte for byte.
int ref_write_dataset_csv(const std::uint8_t* cells, const int* cards, int n, std::uint64_t m,
                          const char* path) {
  return guarded([&] { write_dataset_csv(path, make_dataset(cells, cards, n, m)); });
}

int ref_write_prior_csv(const double* r, int n, const char* path) {
  return guarded([&] { write_prior_csv(path, make_priors(r, n)); });
}

int ref_write_edge_list(const std::uint64_t* masks, int n, const char* path) {
  return guarded([&] {
    std::vector<ParentSet> ps(n);
    for (int i = 0; i < n; ++i) ps[i] = ParentSet{masks[i]};
    write_edge_list(path, Dag(ps));
  });
}

// run_learn (bnmc.cpp:100-138) without --save/--load-cache.
int ref_learn(const char* data_path, const char* priors_path, int s, double gamma, double ess,
              int k2, std::uint64_t iterations, std::uint64_t seed, int workers, int track_top,
              int strict, const char* out_prefix) {
  return guarded([&] {
    RunConfig cfg = make_cfg(s, gamma, ess, k2, workers, std::uint64_t{4} << 30);
    cfg.iterations = iterations;
    cfg.seed = seed;
    cfg.track_top = track_top;
    cfg.strict_paper_tracker = strict != 0;
    cfg.validate();
    const Dataset data = read_dataset_csv(data_path);
    if (data.rows() == 0) throw DataError(std::string(data_path) + ": no data rows");
    const PriorMatrix priors = priors_path ? read_prior_csv(priors_path, data.n())
                                           : PriorMatrix::neutral(data.n());
    const McmcResult result = run_mcmc(data, cfg, priors, nullptr);
    const std::string p = out_prefix;
    write_summary(p + ".summary.txt", cfg, result);
    write_trace_csv(p + ".trace.csv", result.trace);
    write_edge_list(p + ".best.edges", result.tracker.best().dag);
  });
}

// run_eval --sweep (bnmc.cpp:160-212), metrics CSV to out_path.
int ref_eval_sweep(const char* truth_path, const char* data_path, int s, double gamma,
                   double ess, std::uint64_t iterations, std::uint64_t seed, int workers,
                   int track_top, const char* out_path) {
  return guarded([&] {
    std::ofstream out(out_path);
    auto row = [&](const std::string& label, double hi, double lo, double fraction,
                   const ConfusionCounts& c, double best) {
      out << label << "," << format_double(hi) << "," << format_double(lo) << ","
          << format_double(fraction) << "," << c.tp << "," << c.fp << "," << c.fn << "," << c.tn
          << "," << format_double(c.tp_rate()) << "," << format_double(c.fp_rate()) << ","
          << format_double(c.f1()) << "," << format_double(best) << "\n";
    };
    out << "label,prior_hi,prior_lo,fraction,tp,fp,fn,tn,tp_rate,fp_rate,f1,best_score\n";
    const Dag truth = read_edge_list(truth_path, 0);
    const Dataset data = read_dataset_csv(data_path);
    RunConfig cfg = make_cfg(s, gamma, ess, 0, workers, std::uint64_t{4} << 30);
    cfg.iterations = iterations;
    cfg.seed = seed;
    cfg.track_top = track_top;
    cfg.validate();
    const ScoreCache cache = ScoreCache::build(data, cfg);
    const McmcResult base = run_mcmc(data, cfg, PriorMatrix::neutral(data.n()), &cache);
    const Dag& bd = base.tracker.best().dag;
    row("baseline", 0.5, 0.5, 0.0, confusion(bd, truth), base.tracker.best_score());
    const std::pair<double, double> pairs[2] = {{0.7, 0.2}, {0.8, 0.1}};
    const double fractions[2] = {0.2, 0.4};
    const Rng master(cfg.seed);
    int k = 0;
    for (const auto& pr : pairs)
      for (const double f : fractions) {
        Rng prng = master.split(201 + k++);
        const PriorMatrix priors = prior_perturbation_protocol(truth, bd, pr, f, prng);
        const McmcResult run = run_mcmc(data, cfg, priors, &cache);
        row("priors", pr.first, pr.second, f, confusion(run.tracker.best().dag, truth),
            run.tracker.best_score());
      }
  });
}

}  // extern "C"
