// C++ drop-in tests: the reference's own test cases for the hot path
// (proj/tests/test_engine.cpp, test_sampler.cpp, test_scoring.cpp, paths
// relative to /root/reference) compiled against this repo's B200-backed API
// through the reference's header names, plus bit-exact cross-checks against the
// plain-C oracle (oracle/bnmc_oracle.h — test infrastructure only).
//
//   test_dropin cpu   host-only cases (no device calls)
//   test_dropin gpu   every case (needs a B200)
#include <algorithm>
#include <filesystem>
#include <fstream>
#include <cmath>
#include <cstdio>
#include <map>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/bnmc_synth.h"
#include "../../oracle/bnmc_oracle.h"
#include "bnmc/engine.hpp"
#include "bnmc/io.hpp"
#include "bnmc/sampler.hpp"
#include "bnmc/scoring.hpp"
#include "mini_test.hpp"

using namespace bnmc;

namespace {

// The reference tests' synth(): random_dag + Dirichlet CPTs + forward
// sampling from Rng(seed).split(1/2/3) (test_engine.cpp:12-22).
Dataset synth(int n, std::size_t rows, std::uint64_t seed, int card = 2, double edge_p = 0.3,
              double conc = 1.0) {
  std::vector<int> cards(n, card);
  std::vector<std::uint8_t> cells(rows * n);
  std::vector<std::uint64_t> truth(n);
  if (bnmc_synth_instance(n, 3, edge_p, conc, rows, cards.data(), seed, 1, 2, 3, cells.data(),
                          truth.data()) != 0)
    throw Error(bnmc_synth_last_error());
  return Dataset(cards, cells);
}

std::vector<double> oracle_table(const Dataset& d, const RunConfig& cfg) {
  const std::uint64_t per = bounded_subset_count(d.n() - 1, cfg.max_parents);
  std::vector<double> t(per * d.n());
  REQUIRE(orc_cache_build(d.cells().data(), d.cardinalities().data(), d.n(), d.rows(),
                          cfg.max_parents, cfg.gamma, cfg.ess, cfg.alpha_mode == AlphaMode::kK2, 4,
                          t.data()) == 0);
  return t;
}

Order random_order(int n, Rng& rng) {
  std::vector<int> p(n);
  std::iota(p.begin(), p.end(), 0);
  shuffle(p, rng);
  return Order(p);
}

bool same_bits(double a, double b) { return std::bit_cast<std::uint64_t>(a) == std::bit_cast<std::uint64_t>(b); }

}  // namespace

// ------------------------------------------------------------ host-only
TEST_CASE("partition follows the floor rule", false) {
  const auto four = partition(57, 4);
  REQUIRE(four.size() == 4);
  CHECK((four[0] == std::pair<std::uint64_t, std::uint64_t>{0, 14}));
  CHECK((four[3] == std::pair<std::uint64_t, std::uint64_t>{42, 57}));
  const auto tiny = partition(3, 8);
  int empty = 0;
  std::uint64_t covered = 0;
  for (auto [lo, hi] : tiny) {
    empty += lo == hi;
    covered += hi - lo;
  }
  CHECK(empty == 5);
  CHECK(covered == 3);
  CHECK_THROWS_AS(partition(5, 0), UsageError);
}

TEST_CASE("argmax_reduce worked example and tie rule", false) {
  const double v[16] = {-3, -5, -9, -1, -7, -4, -2, -8, -6, -10, -12, -11, -13, -14, -15, -16};
  std::vector<ArgmaxCell> cells(16);
  for (int i = 0; i < 16; ++i) cells[i] = {v[i], static_cast<std::uint64_t>(i)};
  CHECK(argmax_reduce(cells).score == -1.0);
  CHECK(argmax_reduce(cells).idx == 3);
  std::vector<ArgmaxCell> tie{{1.0, 7}, {1.0, 2}};
  CHECK(argmax_reduce(tie).idx == 2);
  std::vector<ArgmaxCell> none{ArgmaxCell{}, ArgmaxCell{}};
  CHECK_THROWS_AS(argmax_reduce(none), UsageError);
}

TEST_CASE("global_index / subset_at agree with the oracle", false) {
  for (int c : {0, 1, 5, 11, 19, 36, 59, 63}) {
    for (int s : {0, 1, 3, 4}) {
      const std::uint64_t S = bounded_subset_count(c, s);
      CHECK(S == orc_bounded_subset_count(c, s));
      const std::uint64_t step = std::max<std::uint64_t>(1, S / 997);
      for (std::uint64_t g = 0; g < S; g += step) {
        const ParentSet p = subset_at(g, c, s);
        CHECK(p.mask == orc_subset_at(g, c, s));
        CHECK(global_index(p, c, s) == g);
      }
    }
  }
  CHECK(subset_at(bounded_subset_count(6, 3) - 1, 6, 3).empty());
}

TEST_CASE("combinatorics: combinations, PST, bounded enumeration", false) {  // test_combinatorics.cpp
  // worked values (n = 6, s = 4): {0,1,2,3} -> 0, empty set -> 56
  CHECK(global_index(ParentSet::of({0, 1, 2, 3}), 6, 4) == 0);
  CHECK(global_index(ParentSet{}, 6, 4) == 56);
  CHECK(bounded_subset_count(6, 4) == 57);
  for (int n : {1, 5, 9})
    for (int k = 0; k <= n && k <= 4; ++k)
      for (std::uint64_t l = 1; l <= binomial(n, k); ++l) {
        const Combination c = unrank_combination(n, k, l);
        CHECK(c.k() == k);
        CHECK(rank_combination(c, n) == l);
      }
  CHECK_THROWS_AS(unrank_combination(5, 2, 0), std::out_of_range);
  CHECK_THROWS_AS(unrank_combination(5, 2, 11), std::out_of_range);
  CHECK_THROWS_AS(rank_combination(Combination{{2, 2}}, 5), std::out_of_range);
  const ParentSetTable t = build_pst(12, 3);
  CHECK(t.size() == bounded_subset_count(12, 3));
  std::vector<std::uint64_t> ref(t.size());
  orc_build_pst(12, 3, ref.data());
  CHECK(t.masks == ref);
  std::uint64_t g = 0;
  const std::vector<int> cands{2, 5, 7, 11};
  bool ok = true;
  enumerate_bounded_subsets(cands, 2, [&](ParentSet p) {
    ok &= p == apply_candidates(subset_at(g++, 4, 2).mask, cands);
  });
  CHECK(ok);
  CHECK(g == bounded_subset_count(4, 2));
  CHECK(pst_bytes_upper_bound(59, 4) == 489406ull * 16);
}

TEST_CASE("DAG utilities", false) {  // test_types.cpp
  Dag d(4);
  d.add_edge(2, 0);
  d.add_edge(3, 2);
  d.add_edge(1, 0);
  CHECK(is_acyclic(d));
  CHECK(topological_order(d) == Order({1, 3, 2, 0}));
  CHECK(consistent(ParentSet::of({1, 2}), 0, Order({1, 3, 2, 0})));
  CHECK_FALSE(consistent(ParentSet::of({3}), 2, Order({2, 3, 1, 0})));
  d.add_edge(0, 3);
  CHECK_FALSE(is_acyclic(d));
  CHECK_THROWS_AS(topological_order(d), DataError);
}

TEST_CASE("propose_swap and mh_accept consume the reference streams", false) {
  Rng a(7), b(7);
  const Order o({3, 1, 0, 2, 4});
  CHECK(propose_swap(propose_swap(o, a), b) == o);
  Rng one(1);
  CHECK_THROWS_AS(propose_swap(Order({0}), one), UsageError);
  orc_rng orng = orc_rng_make(123);
  Rng rng(123);
  for (int t = 0; t < 1000; ++t) {
    const double u = orc_next_unit_open(&orng);
    CHECK(mh_accept(0.0, -0.3, rng) == (std::log10(u) < -0.3));
  }
  Rng r5(5);
  for (int t = 0; t < 10000; ++t) CHECK_FALSE(mh_accept(0.0, -300.0, r5));
}

TEST_CASE("best graph tracker", false) {
  auto g = [](std::uint64_t mask, double score) {
    Dag d(3);
    d.set_parents(2, ParentSet{mask});
    return ScoredGraph{d, score};
  };
  BestGraphTracker t(2);
  CHECK(t.empty());
  CHECK(t.update(g(1, 5.0)));
  CHECK_FALSE(t.update(g(1, 5.0)));
  CHECK(t.update(g(2, 3.0)));
  CHECK(t.update(g(3, 4.0)));
  CHECK(t.entries().size() == 2);
  CHECK(t.entries()[1].total == 4.0);
  CHECK_FALSE(t.update(g(0, 4.0)));
  CHECK_THROWS_AS(BestGraphTracker(0), UsageError);
}

TEST_CASE("value types validate like the reference", false) {
  CHECK_THROWS_AS(Dataset({}, {}), DataError);
  CHECK_THROWS_AS(Dataset({2, 1}, {}), DataError);
  CHECK_THROWS_AS(Dataset({2, 2}, {0, 2}), DataError);
  CHECK_THROWS_AS(Dataset({2, 2}, {0, 1, 1}), DataError);
  CHECK_THROWS_AS(Order({0, 0}), DataError);
  CHECK_THROWS_AS(PriorMatrix(2, {0.5, 0.5, 0.5}), DataError);
  CHECK_THROWS_AS(PriorMatrix(1, {1.5}), DataError);
  Dag d(3);
  CHECK_THROWS_AS(d.add_edge(1, 1), DataError);
  RunConfig cfg;
  cfg.max_parents = 9;
  CHECK_THROWS_AS(cfg.validate(), UsageError);
  cfg = RunConfig{};
  cfg.gamma = 0.0;
  CHECK_THROWS_AS(cfg.validate(), UsageError);
  CHECK(ScoreCache::estimate_bytes(60, 4) == 60ull * 489406ull * 8ull);
  CHECK_THROWS_AS(ScoreCache().device_table(), UsageError);
}


TEST_CASE("io: dataset / prior / edge-list round trips and errors", false) {  // test_io.cpp
  const std::string dir = "/tmp/bnmc_dropin_io";
  std::filesystem::create_directories(dir);
  const Dataset d({2, 3, 4}, {0, 1, 2, 1, 2, 3, 0, 0, 1});
  write_dataset_csv(dir + "/d.csv", d);
  CHECK(read_dataset_csv(dir + "/d.csv") == d);
  {  // cardinalities inferred without "#cards:" (max state + 1, floor 2)
    std::ofstream f(dir + "/e.csv");
    f << "a,b\n0,0\n\n1,0\r\n# comment\n";
  }
  const Dataset e = read_dataset_csv(dir + "/e.csv");
  CHECK(e.rows() == 2);
  CHECK(e.cardinality(0) == 2);
  CHECK(e.cardinality(1) == 2);
  {
    std::ofstream f(dir + "/bad.csv");
    f << "a,b\n0,1,2\n";
  }
  CHECK_THROWS_AS(read_dataset_csv(dir + "/bad.csv"), DataError);
  CHECK_THROWS_AS(read_dataset_csv(dir + "/missing.csv"), DataError);
  PriorMatrix pr = PriorMatrix::neutral(3);
  pr.set(0, 2, 0.75);
  pr.set(2, 1, 0.125);
  write_prior_csv(dir + "/p.csv", pr);
  const PriorMatrix back = read_prior_csv(dir + "/p.csv", 3);
  CHECK(back.r(0, 2) == 0.75);
  CHECK(back.r(2, 1) == 0.125);
  CHECK_THROWS_AS(read_prior_csv(dir + "/p.csv", 4), DataError);
  Dag g(5);
  g.add_edge(0, 3);
  g.add_edge(4, 3);
  g.add_edge(1, 2);
  write_edge_list(dir + "/g.edges", g);
  CHECK(read_edge_list(dir + "/g.edges") == g);  // "# nodes:" keeps isolated nodes
  CHECK(read_edge_list(dir + "/g.edges").n() == 5);
  CHECK(format_double(0.1) == "0.1");
  CHECK(format_double(-4251.749719875) == "-4251.749719875");
  const ConfusionCounts c = confusion(g, Dag(5));
  CHECK(c.fp == 3);
  CHECK(c.tn == 17);
  CHECK(c.f1() == 0.0);
}

// ------------------------------------------------------------- device
TEST_CASE("ScoreCache::build is bit-exact with the oracle", true) {
  for (const auto& [d, s] : {std::pair{synth(9, 150, 42), 4}, std::pair{synth(12, 700, 5, 3), 3},
                             std::pair{synth(7, 1, 3, 4), 2}}) {
    RunConfig cfg;
    cfg.max_parents = s;
    const ScoreCache cache = ScoreCache::build(d, cfg);
    const std::vector<double> ref = oracle_table(d, cfg);
    REQUIRE(cache.entries_per_node() * d.n() == ref.size());
    bool exact = true;
    for (std::size_t i = 0; i < ref.size(); ++i) exact &= same_bits(cache.host_table()[i], ref[i]);
    CHECK(exact);
    // lookup == index_of + at (scoring.hpp:141-146)
    CHECK(same_bits(cache.lookup(3, ParentSet::of({0, 5})), ref[3 * cache.entries_per_node() +
                                                                 orc_index_of(d.n(), s, 3, ParentSet::of({0, 5}).mask)]));
  }
  RunConfig k2;
  k2.alpha_mode = AlphaMode::kK2;
  k2.ess = 3.0;
  const Dataset d = synth(8, 300, 9);
  const ScoreCache c = ScoreCache::build(d, k2);
  const std::vector<double> ref = oracle_table(d, k2);
  bool exact = true;
  for (std::size_t i = 0; i < ref.size(); ++i) exact &= same_bits(c.host_table()[i], ref[i]);
  CHECK(exact);
}

TEST_CASE("count_statistics is bit-exact with the oracle", true) {
  const Dataset d = synth(10, 500, 17, 3);
  for (std::uint64_t mask : {0ull, 0x2ull, 0x31ull, 0x2C0ull}) {
    const CountTable t = count_statistics(d, 2, ParentSet{mask & ~4ull});
    std::vector<std::uint32_t> ref(t.configs() * t.child_card());
    std::uint64_t configs = 0;
    REQUIRE(orc_count_statistics(d.cells().data(), d.cardinalities().data(), d.n(), d.rows(), 2,
                                 mask & ~4ull, ref.data(), ref.size(), &configs) == 0);
    CHECK(configs == t.configs());
    bool same = true;
    for (std::uint64_t k = 0; k < t.configs(); ++k)
      for (int j = 0; j < t.child_card(); ++j) same &= t.njk(k, j) == ref[k * t.child_card() + j];
    CHECK(same);
    CHECK(t.samples() == d.rows());
  }
}

TEST_CASE("local_score: device counts + reference formula, bit-exact", true) {  // test_scoring.cpp:69-118
  const Dataset d = synth(9, 300, 12, 3);
  const Hyperparams bdeu{0.1, 1.0, AlphaMode::kBdeu}, k2{0.5, 2.0, AlphaMode::kK2};
  for (const Hyperparams& h : {bdeu, k2})
    for (std::uint64_t mask : {0ull, 0x4ull, 0x1A2ull, 0x14Cull}) {
      const ParentSet ps{mask & ~2ull};
      double ref = 0.0;
      REQUIRE(orc_local_score(d.cells().data(), d.cardinalities().data(), d.n(), d.rows(), 1,
                              ps.mask, h.gamma, h.ess, h.alpha_mode == AlphaMode::kK2, &ref) == 0);
      CHECK(same_bits(local_score(1, ps, d, h), ref));
    }
  // m = 0: |pi| * log10(gamma) (test_scoring.cpp:74-78)
  const Dataset empty({2, 2, 2}, {});
  CHECK(local_score(0, ParentSet::of({1, 2}), empty, bdeu) == 2 * std::log10(0.1));
}

TEST_CASE("capacity and usage errors", true) {
  const Dataset d = synth(9, 50, 1);
  RunConfig cfg;
  cfg.memory_cap_bytes = ScoreCache::estimate_bytes(9, 4) - 1;
  CHECK_THROWS_AS(ScoreCache::build(d, cfg), CapacityError);
  cfg = RunConfig{};
  cfg.ess = -1.0;
  CHECK_THROWS_AS(ScoreCache::build(d, cfg), UsageError);
  const ScoreCache c = ScoreCache::build(d, RunConfig{});
  CHECK_THROWS_AS(OrderScorer(c, PriorMatrix::neutral(8), EngineConfig{}), DataError);
  CHECK_THROWS_AS(OrderScorer(c, PriorMatrix::neutral(9), EngineConfig{0, 0, IndexStrategy::kPst}),
                  UsageError);
  const OrderScorer sc(c, PriorMatrix::neutral(9), EngineConfig{});
  CHECK_THROWS_AS(sc.score(Order::identity(8)), DataError);
}

TEST_CASE("scan_slice", true) {  // test_engine.cpp:120-152
  const Dataset data = synth(6, 80, 11);
  RunConfig cfg;
  const ScoreCache cache = ScoreCache::build(data, cfg);
  const PriorMatrix neutral = PriorMatrix::neutral(6);
  const OrderScorer scorer(cache, neutral, EngineConfig{});
  const Order order({2, 5, 0, 3, 1, 4});
  CHECK(scorer.scan_slice({3, order.node_at(3), 4, 4}, order).is_identity());
  const int p = 2;
  const std::uint64_t last = bounded_subset_count(p, cfg.max_parents) - 1;
  const ArgmaxCell only_empty = scorer.scan_slice({p, order.node_at(p), last, last + 1}, order);
  CHECK(only_empty.idx == last);
  CHECK(only_empty.score == cache.lookup(order.node_at(p), ParentSet{}));
  const ScoredGraph ref = score_order(order, cache, neutral);
  for (int q = 0; q < 6; ++q) {
    const std::uint64_t total = bounded_subset_count(q, cfg.max_parents);
    const ArgmaxCell cell = scorer.scan_slice({q, order.node_at(q), 0, total}, order);
    CHECK(cell.score == cache.lookup(order.node_at(q), ref.dag.parents(order.node_at(q))));
    const std::span<const int> preds(order.perm().data(), q);
    CHECK(apply_candidates(scorer.set_at(cell.idx, q).mask, preds) == ref.dag.parents(order.node_at(q)));
    // any partition of the range reduces to the same cell (engine.hpp:27-30)
    std::vector<ArgmaxCell> parts;
    for (auto [lo, hi] : partition(total, 3)) parts.push_back(scorer.scan_slice({q, order.node_at(q), lo, hi}, order));
    const ArgmaxCell red = argmax_reduce(parts);
    CHECK(red.idx == cell.idx);
    CHECK(red.score == cell.score);
  }
  CHECK_THROWS_AS(scorer.scan_slice({1, order.node_at(2), 0, 1}, order), UsageError);
}

TEST_CASE("parallel_score_order matches the serial oracle exactly", true) {  // test_engine.cpp:154-182
  const Dataset data = synth(9, 150, 42);
  RunConfig cfg;
  const ScoreCache cache = ScoreCache::build(data, cfg);
  Rng rng(77);
  PriorMatrix priors = PriorMatrix::neutral(9);
  priors.set(3, 1, 0.85);
  priors.set(7, 2, 0.15);
  const std::vector<double> table = oracle_table(data, cfg);
  for (int trial = 0; trial < 20; ++trial) {
    const Order order = random_order(9, rng);
    std::vector<std::uint64_t> masks(9);
    std::vector<double> best(9);
    double total = 0.0;
    REQUIRE(orc_score_order(table.data(), 9, cfg.max_parents, priors.values().data(),
                            order.perm().data(), masks.data(), best.data(), &total) == 0);
    for (const int workers : {1, 3, 8}) {
      for (const IndexStrategy st : {IndexStrategy::kPst, IndexStrategy::kUnrank}) {
        const ScoredGraph g = OrderScorer(cache, priors, EngineConfig{workers, 0, st}).score(order);
        CHECK(same_bits(g.total, total));
        for (int v = 0; v < 9; ++v) CHECK(g.dag.parents(v).mask == masks[v]);
      }
    }
    CHECK(score_order(order, cache, priors).dag == parallel_score_order(order, cache, priors, 4).dag);
  }
}

TEST_CASE("all-ties fixture keeps the first maximum in position order", true) {
  const Dataset empty(std::vector<int>(7, 3), {});
  RunConfig cfg;
  cfg.max_parents = 3;
  cfg.gamma = 1.0;
  const ScoreCache cache = ScoreCache::build(empty, cfg);
  const ScoredGraph g = OrderScorer(cache, PriorMatrix::neutral(7), EngineConfig{}).score(Order({4, 1, 6, 0, 3, 5, 2}));
  CHECK(g.total == 0.0);
  CHECK(g.dag.parents(4) == ParentSet{});
  CHECK(g.dag.parents(1) == ParentSet::of({4}));
  CHECK(g.dag.parents(6) == ParentSet::of({1, 4}));
  for (int v : {0, 3, 5, 2}) CHECK(g.dag.parents(v) == ParentSet::of({1, 4, 6}));
}

TEST_CASE("run_mcmc matches the oracle chain bit for bit", true) {
  for (const bool strict : {false, true}) {
    const Dataset data = synth(10, 400, 33, 3, 0.4, 0.5);
    RunConfig cfg;
    cfg.iterations = 600;
    cfg.seed = 1234;
    cfg.strict_paper_tracker = strict;
    cfg.debug_recheck = true;
    PriorMatrix priors = PriorMatrix::neutral(10);
    priors.set(2, 5, 0.9);
    priors.set(4, 1, 0.1);
    const McmcResult r = run_mcmc(data, cfg, priors);
    const std::vector<double> table = oracle_table(data, cfg);
    const orc_mcmc_cfg oc{cfg.iterations, cfg.seed, cfg.track_top, strict ? 1 : 0};
    std::vector<double> tp(cfg.iterations), tb(cfg.iterations), tt(cfg.track_top);
    std::vector<std::uint8_t> ta(cfg.iterations);
    std::vector<int> fo(10);
    std::vector<std::uint64_t> tm(cfg.track_top * 10);
    double fs = 0.0;
    std::uint64_t acc = 0;
    int tc = 0;
    REQUIRE(orc_run_mcmc(table.data(), 10, cfg.max_parents, priors.values().data(), &oc, tp.data(),
                         ta.data(), tb.data(), fo.data(), &fs, &acc, &tc, tm.data(), tt.data()) == 0);
    REQUIRE(r.trace.size() == cfg.iterations);
    bool trace_ok = true;
    for (std::size_t i = 0; i < r.trace.size(); ++i)
      trace_ok &= r.trace[i].iteration == i + 1 && same_bits(r.trace[i].proposed_score, tp[i]) &&
                  r.trace[i].accepted == (ta[i] != 0) && same_bits(r.trace[i].best_score, tb[i]);
    CHECK(trace_ok);
    CHECK(r.accepted == acc);
    CHECK(same_bits(r.final_score, fs));
    CHECK(r.final_order.perm() == fo);
    REQUIRE(static_cast<int>(r.tracker.entries().size()) == tc);
    for (int e = 0; e < tc; ++e) {
      CHECK(same_bits(r.tracker.entries()[e].total, tt[e]));
      for (int v = 0; v < 10; ++v) CHECK(r.tracker.entries()[e].dag.parents(v).mask == tm[e * 10 + v]);
    }
  }
}

TEST_CASE("run_mcmc determinism across worker knobs and prebuilt caches", true) {  // test_sampler.cpp:139-171
  const Dataset data = synth(6, 120, 33, 2, 0.4, 0.5);
  const PriorMatrix neutral = PriorMatrix::neutral(6);
  RunConfig cfg;
  cfg.iterations = 300;
  cfg.seed = 1234;
  const McmcResult ref = run_mcmc(data, cfg, neutral);
  const ScoreCache cache = ScoreCache::build(data, cfg);
  for (const int workers : {1, 2, 4}) {
    RunConfig c = cfg;
    c.workers = workers;
    c.use_pst = workers != 4;
    const McmcResult r = run_mcmc(data, c, neutral, workers == 2 ? &cache : nullptr);
    REQUIRE(r.trace.size() == ref.trace.size());
    bool same = true;
    for (std::size_t i = 0; i < r.trace.size(); ++i)
      same &= r.trace[i].proposed_score == ref.trace[i].proposed_score &&
              r.trace[i].accepted == ref.trace[i].accepted;
    CHECK(same);
    CHECK(r.final_order == ref.final_order);
    CHECK(r.accepted == ref.accepted);
  }
  // trace invariants (test_sampler.cpp:173-190)
  double last = -1e300;
  for (const TraceRow& row : ref.trace) {
    CHECK(row.best_score >= last);
    last = row.best_score;
  }
  CHECK(score_order(ref.final_order, cache, neutral).total == ref.final_score);
}

TEST_CASE("run_mcmc finds the exhaustive optimum on a small instance", true) {  // test_sampler.cpp:124-137
  const Dataset data = synth(3, 80, 21, 2, 0.4, 0.5);
  RunConfig cfg;
  cfg.iterations = 200;
  cfg.seed = 5;
  const PriorMatrix neutral = PriorMatrix::neutral(3);
  const ScoreCache cache = ScoreCache::build(data, cfg);
  std::vector<int> perm{0, 1, 2};
  double best = -1e300;
  do best = std::max(best, score_order(Order(perm), cache, neutral).total);
  while (std::next_permutation(perm.begin(), perm.end()));
  CHECK(run_mcmc(data, cfg, neutral).tracker.best_score() == best);
}

TEST_CASE("run_mcmc rejects bad inputs", true) {  // test_sampler.cpp:214-220
  RunConfig cfg;
  const Dataset empty({2, 2}, {});
  CHECK_THROWS_AS(run_mcmc(empty, cfg, PriorMatrix::neutral(2)), DataError);
  const Dataset ok({2, 2}, {0, 1});
  CHECK_THROWS_AS(run_mcmc(ok, cfg, PriorMatrix::neutral(3)), DataError);
}

TEST_CASE("BNSC save/load round trip and header checks", true) {
  const Dataset data = synth(8, 200, 4, 3);
  RunConfig cfg;
  cfg.max_parents = 3;
  const ScoreCache built = ScoreCache::build(data, cfg);
  const std::string path = "/tmp/bnmc_dropin_test.bnsc";
  built.save(path);
  const ScoreCache loaded = ScoreCache::load(path, cfg);
  CHECK(loaded.n() == 8);
  CHECK(loaded.host_table() == built.host_table());
  const Order o({7, 2, 5, 0, 1, 3, 6, 4});
  CHECK(score_order(o, loaded, PriorMatrix::neutral(8)).total ==
        score_order(o, built, PriorMatrix::neutral(8)).total);
  RunConfig other = cfg;
  other.ess = 2.0;
  CHECK_THROWS_AS(ScoreCache::load(path, other), DataError);
  other = cfg;
  other.max_parents = 2;
  CHECK_THROWS_AS(ScoreCache::load(path, other), DataError);
  CHECK_THROWS_AS(ScoreCache::load("/nonexistent/x.bnsc", cfg), DataError);
  std::remove(path.c_str());
}

TEST_CASE("run_chains: chain c equals run_mcmc with seed c", true) {
  const Dataset data = synth(12, 300, 8, 3);
  RunConfig cfg;
  cfg.iterations = 250;
  const ScoreCache cache = ScoreCache::build(data, cfg);
  const PriorMatrix neutral = PriorMatrix::neutral(12);
  std::vector<std::uint64_t> seeds(70);
  std::iota(seeds.begin(), seeds.end(), 1);
  const ChainResults all = run_chains(cache, neutral, cfg, seeds);
  REQUIRE(all.size() == seeds.size());
  const std::vector<McmcResult> vec = all.to_vector();
  REQUIRE(vec.size() == seeds.size());
  CHECK(vec[41].final_score == all.final_score(41));
  CHECK(vec[41].trace.size() == cfg.iterations);
  CHECK(all.trace_proposed(41)[7] == vec[41].trace[7].proposed_score);
  for (std::size_t c : {std::size_t{0}, std::size_t{41}, std::size_t{69}}) {
    RunConfig one = cfg;
    one.seed = seeds[c];
    const McmcResult r = run_mcmc(data, one, neutral, &cache);
    CHECK(r.final_order == all[c].final_order);
    CHECK(r.final_score == all[c].final_score);
    CHECK(r.tracker.best().dag == all[c].tracker.best().dag);
  }
}

int main(int argc, char** argv) { return mini::run_all(argc, argv); }
