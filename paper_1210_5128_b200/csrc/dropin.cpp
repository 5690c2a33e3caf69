// dropin.cpp — the reference's C++ API (include/bnmc_b200/bnmc.hpp) over the
// C-ABI of include/bnmc_gpu.h. Host-side only: value types, argument checks
// with the reference's exceptions, BNSC file format, result marshalling. Every
// compute call (precompute, counts, order scan, slice scan, chain) is a
// bnmc_gpu_* call; nothing here scores anything on the CPU.
//
// Reference citations are relative to /root/reference/proj.
#include "../../include/bnmc_b200/bnmc.hpp"

#include <algorithm>
#include <array>
#include <chrono>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>

namespace bnmc {

namespace {

// Status code of the C-ABI -> the reference's exception type.
void check(int status) {
  if (status == BNMC_OK) return;
  const std::string msg = bnmc_gpu_last_error_message();
  switch (status) {
    case BNMC_USAGE: throw UsageError(msg);
    case BNMC_DATA: throw DataError(msg);
    case BNMC_CAPACITY: throw CapacityError(msg);
    default: throw Error("bnmc_gpu: " + msg);
  }
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

bnmc_score_params score_params(const RunConfig& cfg) {
  bnmc_score_params p{};
  p.max_parents = cfg.max_parents;
  p.gamma = cfg.gamma;
  p.ess = cfg.ess;
  p.alpha_mode = cfg.alpha_mode == AlphaMode::kK2 ? BNMC_ALPHA_K2 : BNMC_ALPHA_BDEU;
  p.memory_cap_bytes = cfg.memory_cap_bytes;
  p.device = cfg.device;
  p.n_gpus = cfg.n_gpus;
  return p;
}

struct PascalTable {
  std::array<std::array<std::uint64_t, kMaxNodes + 1>, kMaxNodes + 1> c{};
  PascalTable() {
    for (int n = 0; n <= kMaxNodes; ++n) {
      c[n][0] = 1;
      for (int k = 1; k <= n; ++k) c[n][k] = c[n - 1][k - 1] + c[n - 1][k];
    }
  }
};
const PascalTable kPascal;

// ---- BNSC (scoring.cpp:194-238; README.md:131-135): "BNSC", version 1, n, s,
// alpha (1 = K2), FNV-1a-64 of the LE bytes of (gamma, ess), then n*S LE f64.
constexpr char kMagic[4] = {'B', 'N', 'S', 'C'};
constexpr std::uint8_t kVersion = 1;

std::uint64_t hyper_digest(const Hyperparams& h) {
  std::uint64_t x = 0xCBF29CE484222325ull;
  for (const double d : {h.gamma, h.ess}) {
    const std::uint64_t bits = std::bit_cast<std::uint64_t>(d);
    for (int b = 0; b < 8; ++b) {
      x ^= (bits >> (8 * b)) & 0xFFu;
      x *= 0x100000001B3ull;
    }
  }
  return x;
}

void put_le64(std::ostream& o, std::uint64_t v) {
  unsigned char b[8];
  for (int i = 0; i < 8; ++i) b[i] = static_cast<unsigned char>(v >> (8 * i));
  o.write(reinterpret_cast<const char*>(b), 8);
}

std::uint64_t get_le64(std::istream& in) {
  unsigned char b[8] = {};
  in.read(reinterpret_cast<char*>(b), 8);
  std::uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= static_cast<std::uint64_t>(b[i]) << (8 * i);
  return v;
}

}  // namespace

// ================================================================ types
Dataset::Dataset(std::vector<int> cardinalities, std::vector<std::uint8_t> rows)
    : cards_(std::move(cardinalities)), cells_(std::move(rows)) {
  const std::size_t n = cards_.size();
  if (n == 0 || n > static_cast<std::size_t>(kMaxNodes))
    throw DataError("dataset must have between 1 and 64 variables");
  for (std::size_t i = 0; i < n; ++i)
    if (cards_[i] < 2 || cards_[i] > 256)
      throw DataError("cardinality of variable " + std::to_string(i) + " out of range [2,256]");
  if (cells_.size() % n) throw DataError("row data is not a multiple of the variable count");
  m_ = cells_.size() / n;
  for (std::size_t k = 0; k < cells_.size(); ++k)
    if (cells_[k] >= cards_[k % n])
      throw DataError("state out of range at row " + std::to_string(k / n) + ", column " +
                      std::to_string(k % n));
}

Order::Order(std::vector<int> perm) : perm_(std::move(perm)) {
  const int n = static_cast<int>(perm_.size());
  if (n > kMaxNodes) throw DataError("order exceeds 64 nodes");
  std::uint64_t seen = 0;
  for (const int v : perm_) {
    if (v < 0 || v >= n || ((seen >> v) & 1u)) throw DataError("order is not a permutation of 0..n-1");
    seen |= std::uint64_t{1} << v;
  }
}

Order Order::identity(int n) {
  std::vector<int> p(n);
  std::iota(p.begin(), p.end(), 0);
  return Order(std::move(p));
}

std::vector<int> Order::positions() const {
  std::vector<int> pos(perm_.size());
  for (std::size_t p = 0; p < perm_.size(); ++p) pos[perm_[p]] = static_cast<int>(p);
  return pos;
}

Dag::Dag(std::vector<ParentSet> parents) : parents_(std::move(parents)) {
  if (parents_.size() > static_cast<std::size_t>(kMaxNodes)) throw DataError("graph exceeds 64 nodes");
  for (int i = 0; i < n(); ++i) {
    const ParentSet p = parents_[i];
    parents_[i] = ParentSet{};
    set_parents(i, p);
  }
}

void Dag::set_parents(int node, ParentSet pset) {
  if (pset.contains(node)) throw DataError("self-loop at node " + std::to_string(node));
  if (n() < kMaxNodes && (pset.mask >> n()) != 0)
    throw DataError("parent index out of range for node " + std::to_string(node));
  parents_[node] = pset;
}

void Dag::add_edge(int parent, int child) {
  ParentSet p = parents_[child];
  p.add(parent);
  set_parents(child, p);
}

std::size_t Dag::edge_count() const {
  std::size_t e = 0;
  for (const ParentSet p : parents_) e += static_cast<std::size_t>(p.size());
  return e;
}

PriorMatrix PriorMatrix::neutral(int n) {
  PriorMatrix m;
  m.n_ = n;
  m.v_.assign(static_cast<std::size_t>(n) * n, 0.5);
  return m;
}

PriorMatrix::PriorMatrix(int n, std::vector<double> values) : n_(n), v_(std::move(values)) {
  if (v_.size() != static_cast<std::size_t>(n) * n) throw DataError("prior matrix must be n x n");
  for (const double x : v_)
    if (!(x >= 0.0 && x <= 1.0)) throw DataError("prior matrix entries must lie in [0,1]");
}

void PriorMatrix::set(int child, int parent, double value) {
  if (!(value >= 0.0 && value <= 1.0)) throw DataError("prior matrix entries must lie in [0,1]");
  v_[child * n_ + parent] = value;
}

bool PriorMatrix::is_neutral() const {
  for (int i = 0; i < n_; ++i)
    for (int m = 0; m < n_; ++m)
      if (i != m && r(i, m) != 0.5) return false;
  return true;
}

void RunConfig::validate() const {  // types.cpp:111-121
  if (max_parents < 0 || max_parents > 8) throw UsageError("max-parents must lie in [0,8]");
  if (!(gamma > 0.0 && gamma <= 1.0)) throw UsageError("gamma must lie in (0,1]");
  if (!(ess > 0.0)) throw UsageError("ess must be positive");
  if (iterations < 1) throw UsageError("iterations must be >= 1");
  if (workers < 1) throw UsageError("workers must be >= 1");
  if (track_top < 1) throw UsageError("track-top must be >= 1");
  if (tasks_per_node < 0) throw UsageError("tasks-per-node must be >= 0");
}

bool is_acyclic(const Dag& dag) {
  try {
    topological_order(dag);
    return true;
  } catch (const DataError&) {
    return false;
  }
}

bool consistent(ParentSet pset, int node, const Order& order) {
  const std::vector<int> pos = order.positions();
  bool ok = true;
  pset.for_each([&](int p) { ok = ok && pos[p] < pos[node]; });
  return ok;
}

Order topological_order(const Dag& dag) {
  // Kahn's procedure; the ready set is scanned for its lowest node, which is
  // the min-heap tie-break of types.cpp:140-163.
  const int n = dag.n();
  std::vector<int> indeg(n);
  for (int i = 0; i < n; ++i) indeg[i] = dag.parents(i).size();
  std::uint64_t ready = 0, done = 0;
  for (int i = 0; i < n; ++i)
    if (indeg[i] == 0) ready |= std::uint64_t{1} << i;
  std::vector<int> perm;
  perm.reserve(n);
  while (ready) {
    const int v = std::countr_zero(ready);
    ready &= ready - 1;
    done |= std::uint64_t{1} << v;
    perm.push_back(v);
    for (int child = 0; child < n; ++child)
      if (dag.parents(child).contains(v) && --indeg[child] == 0) ready |= std::uint64_t{1} << child;
  }
  if (static_cast<int>(perm.size()) != n) throw DataError("graph contains a cycle");
  return Order(std::move(perm));
}

// ======================================================== combinatorics
std::uint64_t binomial(int n, int k) {
  if (n < 0 || n > kMaxNodes || k < 0 || k > n) return 0;
  return kPascal.c[n][k];
}

std::uint64_t bounded_subset_count(int n, int s) {
  std::uint64_t t = 0;
  for (int j = 0; j <= s; ++j) t += binomial(n, j);
  return t;
}

std::uint64_t global_index(ParentSet pset, int candidates, int s) {
  // Block offset of the size class, then the combinatorial-number-system rank
  // of the sorted members (combinatorics.cpp:61-76).
  const int k = pset.size();
  std::uint64_t idx = 0;
  for (int j = k + 1; j <= s; ++j) idx += binomial(candidates, j);
  int prev = 0, i = 0;
  pset.for_each([&](int member) {
    const int a = member + 1;
    idx += binomial(candidates - prev, k - i) - binomial(candidates - a + 1, k - i);
    prev = a;
    ++i;
  });
  return idx;
}

ParentSet subset_at(std::uint64_t index, int candidates, int s) {
  int k = std::min(s, candidates);
  for (; k >= 0; --k) {
    const std::uint64_t block = binomial(candidates, k);
    if (index < block) break;
    index -= block;
  }
  if (k < 0) throw std::out_of_range("subset_at: index outside [0, S)");
  // Lexicographic unrank: walk elements, skipping C(c-x-1, k-i-1) blocks.
  ParentSet p;
  int x = 0;
  for (int i = 0; i < k; ++i, ++x) {
    for (std::uint64_t cnt; index >= (cnt = binomial(candidates - x - 1, k - i - 1)); ++x)
      index -= cnt;
    p.add(x);
  }
  return p;
}

Combination unrank_combination(int n, int k, std::uint64_t l) {  // combinatorics.cpp:8-39
  if (n < 0 || k < 0 || k > n) throw std::out_of_range("unrank_combination: need 0 <= k <= n");
  if (l < 1 || l > binomial(n, k))
    throw std::out_of_range("unrank_combination: rank " + std::to_string(l) + " outside [1, C(" +
                            std::to_string(n) + "," + std::to_string(k) + ")]");
  // with s = k the size-k class comes first in the global order, so the
  // 0-based lexicographic rank is the global index; elements reported 1-based
  const ParentSet p = subset_at(l - 1, n, k);
  Combination c;
  p.for_each([&](int x) { c.elems.push_back(x + 1); });
  return c;
}

std::uint64_t rank_combination(const Combination& c, int n) {  // combinatorics.cpp:41-59
  int prev = 0;
  ParentSet p;
  for (const int e : c.elems) {
    if (e <= prev || e > n) throw std::out_of_range("rank_combination: combination invalid over n");
    prev = e;
    p.add(e - 1);
  }
  // global_index over size c.k() only: no larger size classes before it
  return global_index(p, n, c.k()) + 1;
}

ParentSetTable build_pst(int candidates, int s) {  // combinatorics.cpp:92-101
  ParentSetTable t;
  t.candidates = candidates;
  t.s = s;
  const std::uint64_t total = bounded_subset_count(candidates, s);
  t.masks.reserve(total);
  for (std::uint64_t g = 0; g < total; ++g) t.masks.push_back(subset_at(g, candidates, s).mask);
  return t;
}

// ============================================================= scoring
namespace {
constexpr std::uint64_t kDenseCells = std::uint64_t{1} << 22;  // scoring.cpp:13
}

CountTable::CountTable(std::uint64_t configs, int child_card) : r_(configs), card_(child_card) {
  if (r_ > 0 && r_ <= kDenseCells / static_cast<std::uint64_t>(card_))
    cells_.assign(r_ * static_cast<std::uint64_t>(card_), 0u);
}

std::uint32_t CountTable::njk(std::uint64_t config, int state) const {
  if (dense()) return cells_[config * card_ + state];
  const auto it = sparse_.find(config);
  return it == sparse_.end() ? 0u : it->second[state];
}

std::uint32_t CountTable::nk(std::uint64_t config) const {
  std::uint32_t t = 0;
  for (int j = 0; j < card_; ++j) t += njk(config, j);
  return t;
}

std::uint64_t CountTable::samples() const {
  std::uint64_t t = 0;
  for (const std::uint32_t c : cells_) t += c;
  for (const auto& [k, row] : sparse_)
    for (const std::uint32_t c : row) t += c;
  return t;
}

CountTable count_statistics(const Dataset& data, int node, ParentSet pset) {
  if (node < 0 || node >= data.n() || (data.n() < kMaxNodes && (pset.mask >> data.n()) != 0))
    throw UsageError("count_statistics: bad (node, parent set)");
  if (pset.contains(node)) throw DataError("node cannot appear in its own parent set");
  std::uint64_t r = 1;
  pset.for_each([&](int p) {
    const std::uint64_t c = static_cast<std::uint64_t>(data.cardinality(p));
    if (r > std::numeric_limits<std::uint64_t>::max() / c)
      throw CapacityError("parent configuration space overflows 64 bits");
    r *= c;
  });
  CountTable t(r, data.cardinality(node));
  const int nd = node;
  const std::uint64_t mask = pset.mask;
  if (t.dense()) {
    const std::uint64_t off = 0;
    std::uint64_t configs = 0;
    check(bnmc_gpu_count_statistics(data.cells().data(), data.cardinalities().data(), data.rows(),
                                    data.n(), 1, &nd, &mask, &off, t.cells().data(), &configs,
                                    0));
    return t;
  }
  const std::uint64_t m = data.rows();
  const int card = data.cardinality(node);
  std::vector<std::uint64_t> cfg(std::max<std::uint64_t>(m, 1));
  std::vector<std::uint32_t> cnt(std::max<std::uint64_t>(m, 1) * card);
  std::uint64_t active = 0;
  check(bnmc_gpu_count_statistics_sparse(data.cells().data(), data.cardinalities().data(), m,
                                         data.n(), node, mask, cfg.data(), cnt.data(), &active, 0));
  for (std::uint64_t k = 0; k < active; ++k)
    t.sparse().emplace(cfg[k], std::vector<std::uint32_t>(cnt.begin() + k * card,
                                                          cnt.begin() + (k + 1) * card));
  return t;
}

double local_score_from_counts(const CountTable& counts, int pset_size, const Hyperparams& hyper) {
  // scoring.cpp:111-135: configs ascending with N_ik > 0, states ascending with
  // c > 0, score starts at |pi| * log10(gamma) (int x double).
  const double a_cell = hyper.alpha_cell(counts.configs(), counts.child_card());
  if (!(a_cell > 0.0)) throw UsageError("Dirichlet hyperparameter must be positive");
  const double a_row = a_cell * counts.child_card();
  const double lg_row = log10_gamma(a_row), lg_cell = log10_gamma(a_cell);
  const int card = counts.child_card();
  double score = pset_size * std::log10(hyper.gamma);
  counts.for_each_active([&](std::uint64_t, const std::uint32_t* row) {
    std::uint32_t n_ik = 0;
    double inner = 0.0;
    for (int j = 0; j < card; ++j)
      if (row[j] > 0) {
        inner += log10_gamma(row[j] + a_cell) - lg_cell;
        n_ik += row[j];
      }
    score += lg_row - log10_gamma(a_row + n_ik) + inner;
  });
  return score;
}

double local_score(int node, ParentSet pset, const Dataset& data, const Hyperparams& hyper) {
  return local_score_from_counts(count_statistics(data, node, pset), pset.size(), hyper);
}

double ppf(double r_value) {  // scoring.cpp:143-148
  const double d = r_value - 0.5;
  return 100.0 * d * d * d;
}

PpfTable::PpfTable(const PriorMatrix& priors) : n_(priors.n()) {
  w_.assign(static_cast<std::size_t>(n_) * n_, 0.0);
  for (int i = 0; i < n_; ++i)
    for (int m = 0; m < n_; ++m)
      if (i != m) w_[i * n_ + m] = ppf(priors.r(i, m));
}

struct ScoreCache::Shared {
  bnmc_table* table = nullptr;
  std::mutex mu;
  std::vector<double> mirror;
  bool mirrored = false;
  std::vector<double> bound;  // prior values the scan keys carry (empty = neutral)
  ~Shared() {
    if (table) bnmc_gpu_table_free(table);
  }
};

std::uint64_t ScoreCache::estimate_bytes(int n, int s) { return bnmc_gpu_table_estimate_bytes(n, s); }

ScoreCache ScoreCache::build(const Dataset& data, const RunConfig& cfg) {
  cfg.validate();
  const bnmc_score_params p = score_params(cfg);
  ScoreCache c;
  c.d_ = std::make_shared<Shared>();
  check(bnmc_gpu_table_build(data.cells().data(), data.cardinalities().data(), data.rows(), data.n(),
                             &p, nullptr, &c.d_->table));
  c.n_ = data.n();
  c.s_ = cfg.max_parents;
  c.hyper_ = Hyperparams{cfg.gamma, cfg.ess, cfg.alpha_mode};
  c.per_node_ = bounded_subset_count(c.n_ - 1, c.s_);
  return c;
}

ScoreCache ScoreCache::upload(std::span<const double> table, int n, const RunConfig& cfg) {
  cfg.validate();
  if (n < 1 || n > kMaxNodes) throw DataError("dataset must have between 1 and 64 variables");
  const std::uint64_t per = bounded_subset_count(n - 1, cfg.max_parents);
  if (table.size() != per * static_cast<std::uint64_t>(n))
    throw DataError("prebuilt table size does not match n * S(n-1, s)");
  const bnmc_score_params p = score_params(cfg);
  ScoreCache c;
  c.d_ = std::make_shared<Shared>();
  check(bnmc_gpu_table_upload(table.data(), n, &p, nullptr, &c.d_->table));
  c.n_ = n;
  c.s_ = cfg.max_parents;
  c.hyper_ = Hyperparams{cfg.gamma, cfg.ess, cfg.alpha_mode};
  c.per_node_ = per;
  return c;
}

bnmc_table* ScoreCache::device_table() const {
  if (!d_) throw UsageError("score cache is empty (build() or load() first)");
  return d_->table;
}

const std::vector<double>& ScoreCache::host_table() const {
  bnmc_table* t = device_table();
  std::lock_guard<std::mutex> lock(d_->mu);
  if (!d_->mirrored) {
    d_->mirror.resize(static_cast<std::size_t>(n_) * per_node_);
    check(bnmc_gpu_table_download(t, d_->mirror.data()));
    d_->mirrored = true;
  }
  return d_->mirror;
}

double ScoreCache::at(int node, std::uint64_t index) const {
  return host_table()[static_cast<std::size_t>(node) * per_node_ + index];
}

void ScoreCache::bind_priors(const PriorMatrix& priors) const {
  bnmc_table* t = device_table();
  if (priors.n() != n_) throw DataError("priors and cache disagree on node count");
  std::vector<double> want;
  if (!priors.is_neutral()) want = priors.values();
  std::lock_guard<std::mutex> lock(d_->mu);
  if (want == d_->bound) return;
  check(bnmc_gpu_table_set_priors(t, want.empty() ? nullptr : want.data()));
  d_->bound = std::move(want);
}

double ScoreCache::build_kernel_ms() const {
  float a = 0.f, b = 0.f;
  check(bnmc_gpu_table_build_ms(device_table(), &a, &b));
  return a;
}

void ScoreCache::save(const std::string& path) const {
  const std::vector<double>& body = host_table();
  std::ofstream out(path, std::ios::binary);
  if (!out) throw DataError("cannot open cache file for writing: " + path);
  out.write(kMagic, 4);
  const unsigned char meta[4] = {kVersion, static_cast<unsigned char>(n_),
                                 static_cast<unsigned char>(s_),
                                 static_cast<unsigned char>(hyper_.alpha_mode == AlphaMode::kK2)};
  out.write(reinterpret_cast<const char*>(meta), 4);
  put_le64(out, hyper_digest(hyper_));
  for (const double v : body) put_le64(out, std::bit_cast<std::uint64_t>(v));
  if (!out) throw DataError("failed writing cache file: " + path);
}

ScoreCache ScoreCache::load(const std::string& path, const RunConfig& cfg) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw DataError("cannot open cache file: " + path);
  char magic[4] = {};
  in.read(magic, 4);
  if (!in || std::memcmp(magic, kMagic, 4) != 0) throw DataError("not a score cache file: " + path);
  unsigned char meta[4] = {};
  in.read(reinterpret_cast<char*>(meta), 4);
  if (meta[0] != kVersion) throw DataError("unsupported cache version in " + path);
  const Hyperparams hyper{cfg.gamma, cfg.ess, cfg.alpha_mode};
  if (meta[2] != cfg.max_parents || meta[3] != (cfg.alpha_mode == AlphaMode::kK2 ? 1 : 0) ||
      get_le64(in) != hyper_digest(hyper))
    throw DataError("cache file " + path + " was built with different scoring parameters");
  const int n = meta[1];
  if (n < 1 || n > kMaxNodes) throw DataError("not a score cache file: " + path);
  std::vector<double> body(bounded_subset_count(n - 1, meta[2]) * static_cast<std::uint64_t>(n));
  for (double& v : body) v = std::bit_cast<double>(get_le64(in));
  if (!in) throw DataError("cache file truncated: " + path);
  RunConfig c2 = cfg;
  c2.memory_cap_bytes = std::numeric_limits<std::uint64_t>::max();  // load has no cap check
  ScoreCache c = upload(body, n, c2);
  {
    std::lock_guard<std::mutex> lock(c.d_->mu);
    c.d_->mirror = std::move(body);
    c.d_->mirrored = true;
  }
  return c;
}

double effective_local_score(int node, ParentSet pset, const ScoreCache& cache,
                             const PriorMatrix& priors) {
  // scoring.cpp:240-245: ((ls + w_a) + w_b) association.
  double e = cache.lookup(node, pset);
  pset.for_each([&](int p) { e += ppf(priors.r(node, p)); });
  return e;
}

ScoredGraph score_graph(const Dag& dag, const ScoreCache& cache, const PriorMatrix& priors) {
  if (dag.n() != cache.n()) throw DataError("graph and cache disagree on node count");
  double total = 0.0;
  for (int v = 0; v < dag.n(); ++v) {
    if (dag.parents(v).size() > cache.s())
      throw DataError("parent set of node " + std::to_string(v) + " exceeds max-parents");
    total += effective_local_score(v, dag.parents(v), cache, priors);
  }
  return {dag, total};
}

ScoredGraph score_order(const Order& order, const ScoreCache& cache, const PriorMatrix& priors) {
  return OrderScorer(cache, priors, EngineConfig{}).score(order);
}

// ============================================================== engine
std::vector<std::pair<std::uint64_t, std::uint64_t>> partition(std::uint64_t total, int workers) {
  if (workers < 1) throw UsageError("partition requires workers >= 1");
  std::vector<std::pair<std::uint64_t, std::uint64_t>> out;
  out.reserve(workers);
  const auto w = static_cast<std::uint64_t>(workers);
  for (std::uint64_t i = 0; i < w; ++i) out.emplace_back(total * i / w, total * (i + 1) / w);
  return out;
}

ArgmaxCell argmax_reduce(std::span<const ArgmaxCell> cells) {
  ArgmaxCell best;
  for (const ArgmaxCell& c : cells)
    if (!c.is_identity()) best.consider(c.score, c.idx);
  if (best.is_identity()) throw UsageError("argmax reduction over empty work");
  return best;
}

OrderScorer::OrderScorer(const ScoreCache& cache, const PriorMatrix& priors, EngineConfig cfg)
    : cache_(&cache), priors_(priors), cfg_(cfg) {
  if (priors.n() != cache.n()) throw DataError("priors and cache disagree on node count");
  if (cfg_.workers < 1) throw UsageError("workers must be >= 1");
  cache.device_table();  // empty cache -> UsageError now, not at score()
}

std::vector<ScoredGraph> OrderScorer::score_many(std::span<const Order> orders) const {
  const int n = cache_->n();
  std::vector<int> perms;
  perms.reserve(orders.size() * static_cast<std::size_t>(n));
  for (const Order& o : orders) {
    if (o.n() != n) throw DataError("order and cache disagree on node count");
    perms.insert(perms.end(), o.perm().begin(), o.perm().end());
  }
  std::vector<ScoredGraph> out;
  if (orders.empty()) return out;
  cache_->bind_priors(priors_);
  const int count = static_cast<int>(orders.size());
  std::vector<std::uint64_t> masks(perms.size());
  std::vector<double> totals(orders.size());
  check(bnmc_gpu_score_orders(cache_->device_table(), perms.data(), count, masks.data(), nullptr,
                              totals.data()));
  out.reserve(orders.size());
  for (int c = 0; c < count; ++c) {
    std::vector<ParentSet> ps(n);
    for (int v = 0; v < n; ++v) ps[v] = ParentSet{masks[static_cast<std::size_t>(c) * n + v]};
    out.push_back({Dag(std::move(ps)), totals[c]});
  }
  return out;
}

ScoredGraph OrderScorer::score(const Order& order) const {
  return std::move(score_many(std::span<const Order>(&order, 1)).front());
}

ArgmaxCell OrderScorer::scan_slice(const WorkSlice& slice, const Order& order) const {
  if (order.n() != cache_->n()) throw DataError("order and cache disagree on node count");
  if (slice.position < 0 || slice.position >= order.n() || order.node_at(slice.position) != slice.node)
    throw UsageError("work slice does not match the order");
  cache_->bind_priors(priors_);
  ArgmaxCell cell;
  check(bnmc_gpu_scan_slice(cache_->device_table(), order.perm().data(), slice.position, slice.lo,
                            slice.hi, &cell.score, &cell.idx));
  return cell;
}

ParentSet OrderScorer::set_at(std::uint64_t index, int predecessor_count) const {
  return subset_at(index, predecessor_count, cache_->s());
}

ScoredGraph parallel_score_order(const Order& order, const ScoreCache& cache,
                                 const PriorMatrix& priors, int workers) {
  EngineConfig cfg;
  cfg.workers = workers;
  return OrderScorer(cache, priors, cfg).score(order);
}

// ============================================================= sampler
BestGraphTracker::BestGraphTracker(int capacity) : capacity_(capacity) {
  if (capacity < 1) throw UsageError("tracker capacity must be >= 1");
  entries_.reserve(static_cast<std::size_t>(capacity));
}

bool BestGraphTracker::update(const ScoredGraph& g) {  // sampler.cpp:32-41
  if (std::any_of(entries_.begin(), entries_.end(), [&](const ScoredGraph& e) { return e.dag == g.dag; }))
    return false;
  const bool full = static_cast<int>(entries_.size()) == capacity_;
  if (full && g.total <= entries_.back().total) return false;
  const auto before = [](const ScoredGraph& a, const ScoredGraph& b) {
    return a.total != b.total ? a.total > b.total : a.dag < b.dag;
  };
  entries_.insert(std::lower_bound(entries_.begin(), entries_.end(), g, before), g);
  if (full) entries_.pop_back();
  return true;
}

Order propose_swap(const Order& order, Rng& rng) {  // sampler.cpp:43-52
  const int n = order.n();
  if (n < 2) throw UsageError("swap proposal needs at least two nodes");
  const int a = static_cast<int>(rng.next_below(static_cast<std::uint64_t>(n)));
  int b = static_cast<int>(rng.next_below(static_cast<std::uint64_t>(n - 1)));
  b += b >= a;
  Order next = order;
  next.swap_positions(a, b);
  return next;
}

bool mh_accept(double old_score, double new_score, Rng& rng) {  // sampler.cpp:54-56
  return std::log10(rng.next_unit_open()) < new_score - old_score;
}

// ---- run_chains: results in pooled page-locked host memory, McmcResult on access
namespace {
std::mutex g_pool_mu;
std::map<std::size_t, std::vector<void*>> g_pool;  // bytes -> free pinned blocks
std::size_t g_pool_bytes = 0;
constexpr std::size_t kPoolCap = std::size_t{8} << 30;

void* pinned_take(std::size_t bytes) {
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    auto it = g_pool.find(bytes);
    if (it != g_pool.end() && !it->second.empty()) {
      void* p = it->second.back();
      it->second.pop_back();
      g_pool_bytes -= bytes;
      return p;
    }
  }
  void* p = nullptr;
  check(bnmc_gpu_host_alloc(bytes, &p));
  return p;
}

void pinned_give(void* p, std::size_t bytes) {
  if (!p) return;
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (g_pool_bytes + bytes <= kPoolCap) {
      g_pool[bytes].push_back(p);
      g_pool_bytes += bytes;
      return;
    }
  }
  bnmc_gpu_host_free(p);
}
}  // namespace

struct ChainResults::Buffers {
  struct Block {
    void* p = nullptr;
    std::size_t bytes = 0;
  };
  Block tp, ta, tb, fo, fs, acc, tc, tm, tt;
  template <class T>
  T* take(Block& b, std::size_t count) {
    b.bytes = std::max<std::size_t>(8, count * sizeof(T));
    b.p = pinned_take(b.bytes);
    return static_cast<T*>(b.p);
  }
  ~Buffers() {
    for (Block* b : {&tp, &ta, &tb, &fo, &fs, &acc, &tc, &tm, &tt}) pinned_give(b->p, b->bytes);
  }
};

std::span<const double> ChainResults::trace_proposed(std::size_t c) const {
  return {static_cast<const double*>(buf_->tp.p) + c * iters_, iters_};
}
std::span<const std::uint8_t> ChainResults::trace_accepted(std::size_t c) const {
  return {static_cast<const std::uint8_t*>(buf_->ta.p) + c * iters_, iters_};
}
std::span<const double> ChainResults::trace_best(std::size_t c) const {
  return {static_cast<const double*>(buf_->tb.p) + c * iters_, iters_};
}
std::span<const int> ChainResults::final_order(std::size_t c) const {
  return {static_cast<const int*>(buf_->fo.p) + c * n_, static_cast<std::size_t>(n_)};
}
double ChainResults::final_score(std::size_t c) const { return static_cast<const double*>(buf_->fs.p)[c]; }
std::uint64_t ChainResults::accepted(std::size_t c) const {
  return static_cast<const std::uint64_t*>(buf_->acc.p)[c];
}
double ChainResults::best_score(std::size_t c) const {
  return static_cast<const double*>(buf_->tt.p)[c * K_];
}

McmcResult ChainResults::operator[](std::size_t c) const {
  if (c >= size()) throw UsageError("chain index out of range");
  McmcResult r{BestGraphTracker(K_), {}, Order(), 0.0, 0, 0.0, 0.0};
  const int count = static_cast<const int*>(buf_->tc.p)[c];
  const auto* tm = static_cast<const std::uint64_t*>(buf_->tm.p);
  const auto* tt = static_cast<const double*>(buf_->tt.p);
  // Device tracker entries are already in tracker order; re-offering them in
  // that order rebuilds the identical vector.
  for (int e = 0; e < count; ++e) {
    std::vector<ParentSet> ps(n_);
    for (int v = 0; v < n_; ++v) ps[v] = ParentSet{tm[(c * K_ + e) * n_ + v]};
    r.tracker.update({Dag(std::move(ps)), tt[c * K_ + e]});
  }
  const auto tp = trace_proposed(c);
  const auto ta = trace_accepted(c);
  const auto tb = trace_best(c);
  r.trace.resize(iters_);
  for (std::uint64_t t = 0; t < iters_; ++t) r.trace[t] = {t + 1, tp[t], ta[t] != 0, tb[t]};
  const auto fo = final_order(c);
  r.final_order = Order(std::vector<int>(fo.begin(), fo.end()));
  r.final_score = final_score(c);
  r.accepted = accepted(c);
  r.sampling_seconds = wall_;
  return r;
}

std::vector<McmcResult> ChainResults::to_vector() const {
  std::vector<McmcResult> out(size(), McmcResult{BestGraphTracker(std::max(K_, 1)), {}, Order(), 0.0, 0, 0.0, 0.0});
#pragma omp parallel for schedule(dynamic, 64)
  for (std::size_t c = 0; c < size(); ++c) out[c] = (*this)[c];
  return out;
}

ChainResults run_chains(const ScoreCache& cache, const PriorMatrix& priors, const RunConfig& cfg,
                        std::span<const std::uint64_t> seeds) {
  cfg.validate();
  if (priors.n() != cache.n()) throw DataError("prior matrix does not match the dataset's node count");
  if (seeds.empty()) throw UsageError("run_chains needs at least one seed");
  if (seeds.size() > 0x7fffffffu) throw UsageError("too many chains for one call");
  cache.bind_priors(priors);
  ChainResults out;
  out.seeds_.assign(seeds.begin(), seeds.end());
  out.iters_ = cfg.iterations;
  out.n_ = cache.n();
  out.K_ = cfg.track_top;
  const std::size_t C = seeds.size(), I = cfg.iterations, n = cache.n(), K = cfg.track_top;
  auto b = std::make_shared<ChainResults::Buffers>();
  double* tp = b->take<double>(b->tp, C * I);
  std::uint8_t* ta = b->take<std::uint8_t>(b->ta, C * I);
  double* tb = b->take<double>(b->tb, C * I);
  int* fo = b->take<int>(b->fo, C * n);
  double* fs = b->take<double>(b->fs, C);
  std::uint64_t* acc = b->take<std::uint64_t>(b->acc, C);
  int* tc = b->take<int>(b->tc, C);
  std::uint64_t* tm = b->take<std::uint64_t>(b->tm, C * K * n);
  double* tt = b->take<double>(b->tt, C * K);
  bnmc_chain_params params{};
  params.iterations = cfg.iterations;
  params.track_top = cfg.track_top;
  params.strict = cfg.strict_paper_tracker ? 1 : 0;
  params.debug_recheck = cfg.debug_recheck ? 1 : 0;  // device rescore every 100 iterations
  float ms = 0.f;
  const auto t0 = std::chrono::steady_clock::now();
  check(bnmc_gpu_run_chains(cache.device_table(), seeds.data(), static_cast<int>(C), &params, tp,
                            ta, tb, fo, fs, acc, tc, tm, tt, &ms));
  out.wall_ = seconds_since(t0);
  out.device_ms_ = ms;
  out.buf_ = std::move(b);
  return out;
}

McmcResult run_mcmc(const Dataset& data, const RunConfig& cfg, const PriorMatrix& priors,
                    const ScoreCache* prebuilt) {
  cfg.validate();  // sampler.cpp:58-116
  if (data.rows() == 0) throw DataError("learning requires at least one row");
  if (priors.n() != data.n()) throw DataError("prior matrix does not match the dataset's node count");
  if (prebuilt && prebuilt->n() != data.n())
    throw DataError("prebuilt cache does not match the dataset's node count");
  const auto t_pre = std::chrono::steady_clock::now();
  ScoreCache built;
  if (!prebuilt) built = ScoreCache::build(data, cfg);
  const ScoreCache& active = prebuilt ? *prebuilt : built;
  const double pre = seconds_since(t_pre);
  const std::uint64_t seed = cfg.seed;
  McmcResult r = run_chains(active, priors, cfg, std::span<const std::uint64_t>(&seed, 1))[0];
  r.preprocess_seconds = pre;
  return r;
}

}  // namespace bnmc
