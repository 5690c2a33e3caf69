// bnmc_b200/bnmc.hpp — the reference's C++ API for the order-MCMC hot path,
// served by the B200 (sm_100a) backend.
//
// A caller of the reference (project "bnmc", /root/reference/proj) that uses
//   ScoreCache  (include/bnmc/scoring.hpp:117-161)
//   OrderScorer (include/bnmc/engine.hpp:70-98)
//   run_mcmc    (include/bnmc/sampler.hpp:63-65)
// and the value types around them (include/bnmc/types.hpp, rng.hpp,
// combinatorics.hpp) recompiles unchanged against this header (or the
// forwarding headers include/bnmc/*.hpp of this repo) and links
// libbnmc_b200_cxx.so instead of bnmc_core. Names, argument meaning and the
// exception taxonomy (UsageError / DataError / CapacityError) follow the
// reference; every compute call goes through the thin C-ABI of
// include/bnmc_gpu.h — there is no CPU path for the precompute, the order scan
// or the chain. Differences a caller can observe:
//   * EngineConfig::workers / tasks_per_node / strategy and RunConfig::workers,
//     use_pst are validated and otherwise ignored (the device scan has no
//     worker knob); results are bit-identical for every value, as in the
//     reference (engine.hpp:70-75).
//   * ScoreCache copies share one device table (the table is immutable after
//     build, so value semantics are preserved); at()/lookup() read a host
//     mirror downloaded on first use.
//   * RunConfig::debug_recheck re-scores every chain's current order from
//     scratch on the device every 100 iterations (sampler.cpp:105-110) and
//     throws bnmc::Error("chain score drifted from recomputation at iteration
//     N") on a difference, like the reference.
//   * Extensions: RunConfig::device (CUDA ordinal), ScoreCache::upload /
//     device_table(), OrderScorer::score_many, run_chains (independent chains
//     in one device launch).
//   * Not provided (off the hot path): the generator and evaluation
//     of evalgen.hpp other than confusion / prior_perturbation_protocol (io.hpp),
//     Rng::next_normal / next_gamma, full_bitvector_scan, write_cpts, count_dags.
#ifndef BNMC_B200_BNMC_HPP
#define BNMC_B200_BNMC_HPP

#include <bit>
#include <cmath>
#include <cstdint>
#include <initializer_list>
#include <limits>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <map>
#include <vector>

#include "../bnmc_gpu.h"

namespace bnmc {

// ------------------------------------------------------------ types.hpp
inline constexpr int kMaxNodes = 64;

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct UsageError : Error {  // CLI exit code 2
  using Error::Error;
};
struct DataError : Error {  // exit code 3
  using Error::Error;
};
struct CapacityError : Error {  // exit code 4
  using Error::Error;
};

struct ParentSet {
  std::uint64_t mask = 0;

  static ParentSet of(std::initializer_list<int> nodes) {
    ParentSet p;
    for (const int v : nodes) p.add(v);
    return p;
  }
  int size() const { return std::popcount(mask); }
  bool empty() const { return mask == 0; }
  bool contains(int node) const { return ((mask >> node) & 1u) != 0; }
  void add(int node) { mask |= std::uint64_t{1} << node; }
  void remove(int node) { mask &= ~(std::uint64_t{1} << node); }
  template <class F>
  void for_each(F&& f) const {  // ascending node order
    for (std::uint64_t m = mask; m; m &= m - 1) f(std::countr_zero(m));
  }
  std::vector<int> members() const {
    std::vector<int> v;
    for_each([&](int x) { v.push_back(x); });
    return v;
  }
  friend bool operator==(ParentSet a, ParentSet b) { return a.mask == b.mask; }
  friend bool operator<(ParentSet a, ParentSet b) { return a.mask < b.mask; }
};

class Dataset {
 public:
  Dataset() = default;
  Dataset(std::vector<int> cardinalities, std::vector<std::uint8_t> rows);
  int n() const { return static_cast<int>(cards_.size()); }
  std::size_t rows() const { return m_; }
  int cardinality(int i) const { return cards_[i]; }
  const std::vector<int>& cardinalities() const { return cards_; }
  std::uint8_t state(std::size_t row, int col) const { return cells_[row * cards_.size() + col]; }
  const std::vector<std::uint8_t>& cells() const { return cells_; }
  friend bool operator==(const Dataset& a, const Dataset& b) {
    return a.cards_ == b.cards_ && a.cells_ == b.cells_;
  }

 private:
  std::vector<int> cards_;
  std::vector<std::uint8_t> cells_;
  std::size_t m_ = 0;
};

class Order {
 public:
  Order() = default;
  explicit Order(std::vector<int> perm);
  static Order identity(int n);
  int n() const { return static_cast<int>(perm_.size()); }
  int node_at(int pos) const { return perm_[pos]; }
  const std::vector<int>& perm() const { return perm_; }
  std::vector<int> positions() const;
  void swap_positions(int a, int b) { std::swap(perm_[a], perm_[b]); }
  friend bool operator==(const Order& a, const Order& b) { return a.perm_ == b.perm_; }

 private:
  std::vector<int> perm_;
};

class Dag {
 public:
  Dag() = default;
  explicit Dag(int n) : parents_(n) {}
  explicit Dag(std::vector<ParentSet> parents);
  int n() const { return static_cast<int>(parents_.size()); }
  ParentSet parents(int node) const { return parents_[node]; }
  const std::vector<ParentSet>& all_parents() const { return parents_; }
  void set_parents(int node, ParentSet pset);
  void add_edge(int parent, int child);
  bool has_edge(int parent, int child) const { return parents_[child].contains(parent); }
  std::size_t edge_count() const;
  friend bool operator==(const Dag& a, const Dag& b) { return a.parents_ == b.parents_; }
  friend bool operator<(const Dag& a, const Dag& b) { return a.parents_ < b.parents_; }

 private:
  std::vector<ParentSet> parents_;
};

class PriorMatrix {
 public:
  PriorMatrix() = default;
  static PriorMatrix neutral(int n);
  PriorMatrix(int n, std::vector<double> values);
  int n() const { return n_; }
  double r(int child, int parent) const { return v_[child * n_ + parent]; }
  void set(int child, int parent, double value);
  bool is_neutral() const;
  const std::vector<double>& values() const { return v_; }  // row-major r[child*n + parent]

 private:
  int n_ = 0;
  std::vector<double> v_;
};

enum class AlphaMode { kBdeu, kK2 };

struct RunConfig {
  int max_parents = 4;
  double gamma = 0.1;
  double ess = 1.0;
  AlphaMode alpha_mode = AlphaMode::kBdeu;
  std::uint64_t iterations = 1;
  std::uint64_t seed = 0;
  int workers = 1;
  int track_top = 10;
  bool strict_paper_tracker = false;
  bool use_pst = true;
  int tasks_per_node = 0;
  std::uint64_t memory_cap_bytes = std::uint64_t{4} << 30;
  bool debug_recheck = false;
  int device = 0;  // extension: CUDA ordinal of the table
  int n_gpus = 1;  // extension: > 1 = devices device..device+n_gpus-1 (split precompute
                   // + NCCL all-reduce, chains spread over full replicas)

  void validate() const;
};

// DAG utilities (types.cpp:123-164): acyclicity, order consistency, Kahn's
// topological order with the lowest-index tie-break (DataError on a cycle).
bool is_acyclic(const Dag& dag);
bool consistent(ParentSet pset, int node, const Order& order);
Order topological_order(const Dag& dag);

// -------------------------------------------------------------- rng.hpp
// splitmix64 streams (rng.hpp:14-45): the proposal and acceptance streams the
// device loop consumes are derived exactly like this.
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : s_(seed) {}
  Rng split(std::uint64_t tag) const { return Rng(mix(s_ + kGolden * (tag + 1))); }
  std::uint64_t next_u64() { return mix(s_ += kGolden); }
  double next_unit() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double next_unit_open() { return (static_cast<double>(next_u64() >> 11) + 0.5) * 0x1.0p-53; }
  std::uint64_t next_below(std::uint64_t bound) {
    const std::uint64_t reject_below = (0 - bound) % bound;
    for (;;) {
      const std::uint64_t x = next_u64();
      if (x >= reject_below) return x % bound;
    }
  }

 private:
  static constexpr std::uint64_t kGolden = 0x9E3779B97F4A7C15ull;
  static std::uint64_t mix(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  std::uint64_t s_;
};

template <class T>
void shuffle(std::vector<T>& v, Rng& rng) {  // Fisher-Yates, rng.hpp:86-90
  for (std::size_t i = v.size(); i > 1; --i) std::swap(v[i - 1], v[rng.next_below(i)]);
}

// ---------------------------------------------------- combinatorics.hpp
std::uint64_t binomial(int n, int k);
std::uint64_t bounded_subset_count(int n, int s);
// Cache addressing contract (combinatorics.hpp:59-64): sizes descending,
// lexicographic within a size, empty set last.
std::uint64_t global_index(ParentSet pset, int candidates, int s);
ParentSet subset_at(std::uint64_t index, int candidates, int s);
inline ParentSet apply_candidates(std::uint64_t position_mask, std::span<const int> candidates) {
  ParentSet out;
  for (std::uint64_t m = position_mask; m; m &= m - 1) out.add(candidates[std::countr_zero(m)]);
  return out;
}

// 1-based k-combinations of {1..n} (combinatorics.hpp:38-57): unrank by the
// lexicographic rank l in [1, C(n,k)] (std::out_of_range otherwise) and back.
struct Combination {
  std::vector<int> elems;
  int k() const { return static_cast<int>(elems.size()); }
  friend bool operator==(const Combination& a, const Combination& b) { return a.elems == b.elems; }
};
Combination unrank_combination(int n, int k, std::uint64_t l);
std::uint64_t rank_combination(const Combination& c, int n);

// Every subset of {0..candidates-1} with size <= s, in global_index order
// (combinatorics.hpp:81-111), as position masks / through a candidate list.
template <class F>
void enumerate_bounded_position_sets(int candidates, int s, F&& f) {
  const std::uint64_t total = bounded_subset_count(candidates, s);
  for (std::uint64_t g = 0; g < total; ++g) f(subset_at(g, candidates, s));
}
template <class F>
void enumerate_bounded_subsets(std::span<const int> candidates, int s, F&& f) {
  enumerate_bounded_position_sets(static_cast<int>(candidates.size()), s,
                                  [&](ParentSet pos) { f(apply_candidates(pos.mask, candidates)); });
}

// Parent set table (combinatorics.hpp:113-131): row i = subset_at(i).
struct ParentSetTable {
  int candidates = 0;
  int s = 0;
  std::vector<std::uint64_t> masks;
  std::uint64_t size() const { return masks.size(); }
};
ParentSetTable build_pst(int candidates, int s);
inline std::uint64_t pst_bytes_upper_bound(int candidates, int s) {
  return bounded_subset_count(candidates, s) * 16;
}

// ---------------------------------------------------------- scoring.hpp
inline double log10_gamma(double x) { return std::lgamma(x) * 0.43429448190325182765; }

struct Hyperparams {
  double gamma = 0.1;
  double ess = 1.0;
  AlphaMode alpha_mode = AlphaMode::kBdeu;
  double alpha_cell(std::uint64_t r_i, int child_card) const {
    return alpha_mode == AlphaMode::kBdeu ? ess / (static_cast<double>(r_i) * child_card) : 1.0;
  }
  friend bool operator==(const Hyperparams&, const Hyperparams&) = default;
};

// N_ijk for one (node, parent set), counted on the device. Like the
// reference's CountTable (scoring.hpp:41-77, scoring.cpp:53-80): dense
// configs() x child_card() u32 cells up to 2^22 cells
// (bnmc_gpu_count_statistics), otherwise an ordered map of the active
// configurations (bnmc_gpu_count_statistics_sparse); the config index is
// mixed-radix with the lowest parent least significant; iteration ascending.
class CountTable {
 public:
  CountTable(std::uint64_t configs, int child_card);
  std::uint64_t configs() const { return r_; }
  int child_card() const { return card_; }
  std::uint64_t samples() const;
  std::uint32_t njk(std::uint64_t config, int state) const;
  std::uint32_t nk(std::uint64_t config) const;
  template <class F>
  void for_each_active(F&& f) const {  // configs with N_ik > 0, ascending
    if (dense()) {
      for (std::uint64_t k = 0; k < r_; ++k)
        if (nk(k) > 0) f(k, cells_.data() + k * card_);
    } else {
      for (const auto& [k, c] : sparse_) f(k, c.data());
    }
  }
  bool dense() const { return !cells_.empty() || r_ == 0; }
  std::vector<std::uint32_t>& cells() { return cells_; }
  std::map<std::uint64_t, std::vector<std::uint32_t>>& sparse() { return sparse_; }

 private:
  std::uint64_t r_;
  int card_;
  std::vector<std::uint32_t> cells_;  // dense storage (r * card <= 2^22)
  std::map<std::uint64_t, std::vector<std::uint32_t>> sparse_;
};

CountTable count_statistics(const Dataset& data, int node, ParentSet pset);

// Log10 BD local score of given counts (scoring.cpp:111-135) — host formula
// over glibc lgamma in the reference's summation order (bit-identical); the
// table build itself runs on the device (ScoreCache::build).
double local_score_from_counts(const CountTable& counts, int pset_size, const Hyperparams& hyper);
// count_statistics on the device + local_score_from_counts.
double local_score(int node, ParentSet pset, const Dataset& data, const Hyperparams& hyper);

double ppf(double r_value);

class PpfTable {
 public:
  PpfTable() = default;
  explicit PpfTable(const PriorMatrix& priors);
  double weight(int child, int parent) const { return w_[child * n_ + parent]; }
  double sum(int child, ParentSet pset) const {  // ascending parents from 0.0
    double t = 0.0;
    pset.for_each([&](int p) { t += weight(child, p); });
    return t;
  }

 private:
  int n_ = 0;
  std::vector<double> w_;
};

// Device-resident score table: fp64 local scores in (node, global index)
// order plus the fp32 scan keys with the bound priors' PPF folded in.
class ScoreCache {
 public:
  ScoreCache() = default;
  static std::uint64_t estimate_bytes(int n, int s);
  static ScoreCache build(const Dataset& data, const RunConfig& cfg);
  int n() const { return n_; }
  int s() const { return s_; }
  const Hyperparams& hyper() const { return hyper_; }
  std::uint64_t entries_per_node() const { return per_node_; }
  std::uint64_t index_of(int node, ParentSet pset) const {
    const std::uint64_t below = pset.mask & ((std::uint64_t{1} << node) - 1);
    const std::uint64_t above = node + 1 < 64 ? (pset.mask >> (node + 1)) << node : 0;
    return global_index(ParentSet{below | above}, n_ - 1, s_);
  }
  double at(int node, std::uint64_t index) const;
  double lookup(int node, ParentSet pset) const { return at(node, index_of(node, pset)); }
  // BNSC persistence (scoring.hpp:148-153), byte-compatible with the reference.
  void save(const std::string& path) const;
  static ScoreCache load(const std::string& path, const RunConfig& cfg);

  // ---- B200 extensions
  // Prebuilt host table (n x S doubles, BNSC body order) -> device.
  static ScoreCache upload(std::span<const double> table, int n, const RunConfig& cfg);
  bnmc_table* device_table() const;
  const std::vector<double>& host_table() const;  // lazily downloaded mirror
  // Folds the PPF of `priors` into the scan keys when the table is bound to
  // different priors (OrderScorer / run_mcmc call this).
  void bind_priors(const PriorMatrix& priors) const;
  double build_kernel_ms() const;  // device time of the last count+score build

 private:
  struct Shared;
  std::shared_ptr<Shared> d_;
  int n_ = 0;
  int s_ = 0;
  Hyperparams hyper_;
  std::uint64_t per_node_ = 0;
};

double effective_local_score(int node, ParentSet pset, const ScoreCache& cache,
                             const PriorMatrix& priors);

struct ScoredGraph {
  Dag dag;
  double total = 0.0;
};

ScoredGraph score_graph(const Dag& dag, const ScoreCache& cache, const PriorMatrix& priors);
// The reference's serial scorer (scoring.cpp:261-289); served by the device
// scan, bit-identical.
ScoredGraph score_order(const Order& order, const ScoreCache& cache, const PriorMatrix& priors);

// ----------------------------------------------------------- engine.hpp
struct WorkSlice {
  int position = 0;
  int node = 0;
  std::uint64_t lo = 0;
  std::uint64_t hi = 0;
};

struct ArgmaxCell {
  static constexpr std::uint64_t kNoIndex = std::numeric_limits<std::uint64_t>::max();
  double score = -std::numeric_limits<double>::infinity();
  std::uint64_t idx = kNoIndex;
  bool is_identity() const { return idx == kNoIndex; }
  void consider(double s, std::uint64_t i) {  // higher score, then smaller index
    if (s > score || (s == score && i < idx)) {
      score = s;
      idx = i;
    }
  }
};

std::vector<std::pair<std::uint64_t, std::uint64_t>> partition(std::uint64_t total, int workers);
ArgmaxCell argmax_reduce(std::span<const ArgmaxCell> cells);

enum class IndexStrategy { kPst, kUnrank };

struct EngineConfig {
  int workers = 1;
  int tasks_per_node = 0;
  IndexStrategy strategy = IndexStrategy::kPst;
  static EngineConfig from(const RunConfig& cfg) {
    return {cfg.workers, cfg.tasks_per_node, cfg.use_pst ? IndexStrategy::kPst : IndexStrategy::kUnrank};
  }
};

class OrderScorer {
 public:
  OrderScorer(const ScoreCache& cache, const PriorMatrix& priors, EngineConfig cfg);
  ScoredGraph score(const Order& order) const;
  // Device argmax over PST indices [lo, hi) of the node at `position`
  // (engine.cpp:43-58 semantics: strict >, ties keep the smallest index).
  ArgmaxCell scan_slice(const WorkSlice& slice, const Order& order) const;
  const EngineConfig& config() const { return cfg_; }
  ParentSet set_at(std::uint64_t index, int predecessor_count) const;

  // ---- B200 extension: many orders in one device pass.
  std::vector<ScoredGraph> score_many(std::span<const Order> orders) const;

 private:
  const ScoreCache* cache_;
  PriorMatrix priors_;
  EngineConfig cfg_;
};

ScoredGraph parallel_score_order(const Order& order, const ScoreCache& cache,
                                 const PriorMatrix& priors, int workers);

// ---------------------------------------------------------- sampler.hpp
class BestGraphTracker {
 public:
  explicit BestGraphTracker(int capacity);
  bool update(const ScoredGraph& g);
  const std::vector<ScoredGraph>& entries() const { return entries_; }
  const ScoredGraph& best() const { return entries_.front(); }
  double best_score() const { return entries_.front().total; }
  bool empty() const { return entries_.empty(); }
  int capacity() const { return capacity_; }

 private:
  int capacity_;
  std::vector<ScoredGraph> entries_;
};

Order propose_swap(const Order& order, Rng& rng);
bool mh_accept(double old_score, double new_score, Rng& rng);

struct TraceRow {
  std::uint64_t iteration;
  double proposed_score;
  bool accepted;
  double best_score;
};

struct McmcResult {
  BestGraphTracker tracker;
  std::vector<TraceRow> trace;
  Order final_order;
  double final_score = 0.0;
  std::uint64_t accepted = 0;
  double preprocess_seconds = 0.0;
  double sampling_seconds = 0.0;
};

McmcResult run_mcmc(const Dataset& data, const RunConfig& cfg, const PriorMatrix& priors,
                    const ScoreCache* prebuilt = nullptr);

// ---- B200 extension: independent chains, chain c == run_mcmc with
// cfg.seed = seeds[c], all run by one device launch. The device writes every
// chain's trace, tracker and final state straight into page-locked host
// buffers (pooled and reused across calls); a chain's McmcResult is built only
// when it is accessed.
class ChainResults {
 public:
  std::size_t size() const { return seeds_.size(); }
  std::uint64_t iterations() const { return iters_; }
  std::uint64_t seed(std::size_t c) const { return seeds_.at(c); }
  McmcResult operator[](std::size_t c) const;  // built on access
  std::vector<McmcResult> to_vector() const;
  // raw per-chain views (valid while this object lives)
  std::span<const double> trace_proposed(std::size_t c) const;
  std::span<const std::uint8_t> trace_accepted(std::size_t c) const;
  std::span<const double> trace_best(std::size_t c) const;
  std::span<const int> final_order(std::size_t c) const;
  double final_score(std::size_t c) const;
  std::uint64_t accepted(std::size_t c) const;
  double best_score(std::size_t c) const;  // tracker best
  double device_ms() const { return device_ms_; }  // device time of the chain kernel(s)
  double sampling_seconds() const { return wall_; }  // wall time of the device call

  struct Buffers;  // page-locked blocks (dropin.cpp)

 private:
  friend ChainResults run_chains(const class ScoreCache&, const PriorMatrix&, const RunConfig&,
                                 std::span<const std::uint64_t>);
  std::shared_ptr<Buffers> buf_;
  std::vector<std::uint64_t> seeds_;
  std::uint64_t iters_ = 0;
  int n_ = 0, K_ = 0;
  double device_ms_ = 0.0, wall_ = 0.0;
};

ChainResults run_chains(const ScoreCache& cache, const PriorMatrix& priors, const RunConfig& cfg,
                        std::span<const std::uint64_t> seeds);

}  // namespace bnmc

#endif
