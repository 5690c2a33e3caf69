// synth.cpp — synthetic BASELINE instances (input synthesis, not the hot path).
//
// Restates the reference generator so that bench.py and the GPU tests can
// build the SURVEY §8d inputs on a box without /root/reference:
//   random_dag (evalgen.cpp:38-51), random_ground_truth (evalgen.cpp:53-75),
//   forward_sample (evalgen.cpp:77-109), topological_order (types.cpp:134-164),
//   Rng::next_normal / next_gamma (rng.hpp:47-73) and the prior protocol of
//   SURVEY §8d. Compiled without -march (no FMA contraction), so with the same
//   glibc the cells are bit-identical to the reference's; tests check the
//   SHA-256 of every BASELINE dataset against tests/golden/golden.json.
#include <stdint.h>

#include <cmath>
#include <cstring>
#include <functional>
#include <queue>
#include <string>
#include <vector>

#include "../../include/bnmc_synth.h"

namespace {

thread_local std::string g_err;

struct Rng {
  uint64_t s;
  static uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  Rng split(uint64_t tag) const { return Rng{mix(s + 0x9E3779B97F4A7C15ull * (tag + 1))}; }
  uint64_t next_u64() {
    s += 0x9E3779B97F4A7C15ull;
    return mix(s);
  }
  double next_unit() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double next_unit_open() { return (static_cast<double>(next_u64() >> 11) + 0.5) * 0x1.0p-53; }
  uint64_t next_below(uint64_t bound) {
    const uint64_t threshold = (0 - bound) % bound;
    uint64_t x;
    do {
      x = next_u64();
    } while (x < threshold);
    return x % bound;
  }
  double next_normal() {
    const double u1 = next_unit_open();
    const double u2 = next_unit_open();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.141592653589793238462643 * u2);
  }
  double next_gamma(double shape) {
    if (shape < 1.0) {
      const double u = next_unit_open();
      const double g = next_gamma(shape + 1.0);
      return g * std::pow(u, 1.0 / shape);
    }
    const double d = shape - 1.0 / 3.0;
    const double c = 1.0 / (3.0 * std::sqrt(d));
    for (;;) {
      double x, v;
      do {
        x = next_normal();
        v = 1.0 + c * x;
      } while (v <= 0.0);
      v = v * v * v;
      const double u = next_unit_open();
      if (u < 1.0 - 0.0331 * x * x * x * x) return d * v;
      if (std::log(u) < 0.5 * x * x + d * (1.0 - v + std::log(v))) return d * v;
    }
  }
};

void shuffle(std::vector<int>& v, Rng& rng) {
  for (size_t i = v.size(); i > 1; --i) std::swap(v[i - 1], v[rng.next_below(i)]);
}

}  // namespace

extern "C" {

const char* bnmc_synth_last_error(void) { return g_err.c_str(); }

int bnmc_synth_instance(int n, int max_parents, double edge_prob, double concentration,
                        uint64_t m, const int* cards, uint64_t seed, uint64_t tag_dag,
                        uint64_t tag_cpt, uint64_t tag_rows, uint8_t* cells_out,
                        uint64_t* truth_out) {
  if (n < 1 || n > 64) {
    g_err = "n must lie in [1,64]";
    return 2;
  }
  if (!(concentration > 0.0)) {
    g_err = "Dirichlet concentration must be positive";
    return 2;
  }
  for (int i = 0; i < n; ++i)
    if (cards[i] < 2 || cards[i] > 256) {
      g_err = "cardinality out of range [2,256]";
      return 3;
    }
  const Rng master{seed};
  Rng dag_rng = master.split(tag_dag);
  Rng cpt_rng = master.split(tag_cpt);
  Rng row_rng = master.split(tag_rows);

  // random_dag: edges point backward along a random permutation.
  std::vector<int> perm(n);
  for (int i = 0; i < n; ++i) perm[i] = i;
  shuffle(perm, dag_rng);
  std::vector<uint64_t> parents(n, 0);
  for (int p = 1; p < n; ++p) {
    uint64_t ps = 0;
    for (int q = p - 1; q >= 0 && __builtin_popcountll(ps) < max_parents; --q)
      if (dag_rng.next_unit() < edge_prob) ps |= 1ull << perm[q];
    parents[perm[p]] = ps;
  }

  // random_ground_truth: Dirichlet(concentration) CPT rows.
  std::vector<std::vector<double>> cpts(n);
  for (int i = 0; i < n; ++i) {
    const int card = cards[i];
    uint64_t r = 1;
    for (uint64_t mm = parents[i]; mm; mm &= mm - 1) r *= cards[__builtin_ctzll(mm)];
    auto& cpt = cpts[i];
    cpt.resize(r * card);
    for (uint64_t k = 0; k < r; ++k) {
      double total = 0.0;
      for (int j = 0; j < card; ++j) {
        cpt[k * card + j] = cpt_rng.next_gamma(concentration);
        total += cpt[k * card + j];
      }
      for (int j = 0; j < card; ++j) cpt[k * card + j] /= total;
    }
  }

  // topological_order: Kahn with a min-heap on node index.
  std::vector<int> indeg(n), topo;
  for (int i = 0; i < n; ++i) indeg[i] = __builtin_popcountll(parents[i]);
  std::priority_queue<int, std::vector<int>, std::greater<int>> ready;
  for (int i = 0; i < n; ++i)
    if (indeg[i] == 0) ready.push(i);
  while (!ready.empty()) {
    const int v = ready.top();
    ready.pop();
    topo.push_back(v);
    for (int child = 0; child < n; ++child)
      if (((parents[child] >> v) & 1u) && --indeg[child] == 0) ready.push(child);
  }

  // forward_sample
  std::vector<int> state(n, 0);
  for (uint64_t t = 0; t < m; ++t) {
    for (int p = 0; p < n; ++p) {
      const int node = topo[p];
      const int card = cards[node];
      uint64_t k = 0, radix = 1;
      for (uint64_t mm = parents[node]; mm; mm &= mm - 1) {
        const int par = __builtin_ctzll(mm);
        k += radix * state[par];
        radix *= cards[par];
      }
      const double* row = cpts[node].data() + k * card;
      const double u = row_rng.next_unit();
      double cum = 0.0;
      int drawn = card - 1;
      for (int j = 0; j < card; ++j) {
        cum += row[j];
        if (u < cum) {
          drawn = j;
          break;
        }
      }
      state[node] = drawn;
      cells_out[t * n + node] = static_cast<uint8_t>(drawn);
    }
  }
  for (int i = 0; i < n; ++i) truth_out[i] = parents[i];
  return 0;
}

int bnmc_synth_priors(int n, const uint64_t* truth, uint64_t seed, uint64_t tag, double* r_out) {
  Rng pr = Rng{seed}.split(tag);
  for (int i = 0; i < n * n; ++i) r_out[i] = 0.5;
  for (int c = 0; c < n; ++c)
    for (int p = 0; p < n; ++p) {
      if (p == c) continue;
      if ((truth[c] >> p) & 1u) {
        if (pr.next_unit() < 0.3) r_out[c * n + p] = 0.75;
      } else {
        if (pr.next_unit() < 0.02) r_out[c * n + p] = 0.25;
      }
    }
  return 0;
}

}  // extern "C"
