// e2e_probe — end-to-end throughput of the reference-shaped C++ API
// (bnmc::run_chains, include/bnmc_b200/bnmc.hpp) at the bench workload:
// cfg4 (n=60, k=4, m=10,000, 3-state, SURVEY §8d priors), C chains x I
// iterations per call. Each timed call includes the H2D copy of the seeds,
// the device loop and the D2H copy of every chain's trace, tracker and final
// state into the pooled page-locked buffers; one McmcResult is materialised
// per call (the best chain's), as a caller reading the result would.
//   e2e_probe [chains] [iterations] [steps] [warmup]
// Prints one JSON object: wall it/s, device it/s and their ratio.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <vector>

#include "bnmc/sampler.hpp"
#include "bnmc_synth.h"

int main(int argc, char** argv) {
  const int chains = argc > 1 ? std::atoi(argv[1]) : 18944;
  const std::uint64_t iters = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 500;
  const int steps = argc > 3 ? std::atoi(argv[3]) : 5;
  const int warmup = argc > 4 ? std::atoi(argv[4]) : 2;
  const int n = 60, k = 4;
  const std::uint64_t m = 10000;
  std::vector<int> cards(n, 3);
  std::vector<std::uint8_t> cells(m * n);
  std::vector<std::uint64_t> truth(n);
  if (bnmc_synth_instance(n, k, 0.3, 1.0, m, cards.data(), 7, 101, 102, 103, cells.data(),
                          truth.data()) != 0) {
    std::fprintf(stderr, "synth failed: %s\n", bnmc_synth_last_error());
    return 1;
  }
  std::vector<double> r(n * n);
  bnmc_synth_priors(n, truth.data(), 7, 104, r.data());
  const bnmc::Dataset data(cards, cells);
  const bnmc::PriorMatrix pri(n, r);
  bnmc::RunConfig cfg;
  cfg.max_parents = k;
  cfg.iterations = iters;
  cfg.memory_cap_bytes = ~0ull;
  const bnmc::ScoreCache cache = bnmc::ScoreCache::build(data, cfg);
  std::vector<std::uint64_t> seeds(chains);
  double wall = 0.0, dev_ms = 0.0, best = -1e300;
  for (int s = 0; s < warmup + steps; ++s) {
    std::iota(seeds.begin(), seeds.end(), 1 + static_cast<std::uint64_t>(s) * chains);
    const auto t0 = std::chrono::steady_clock::now();
    const bnmc::ChainResults res = bnmc::run_chains(cache, pri, cfg, seeds);
    std::size_t arg = 0;
    for (std::size_t c = 1; c < res.size(); ++c)
      if (res.best_score(c) > res.best_score(arg)) arg = c;
    const bnmc::McmcResult top = res[arg];
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (s >= warmup) {
      wall += dt;
      dev_ms += res.device_ms();
      best = std::max(best, top.tracker.best_score());
    }
  }
  const double total = static_cast<double>(chains) * iters * steps;
  std::printf("{\"api\": \"bnmc::run_chains (C++ drop-in)\", \"chains\": %d, \"iterations\": %llu, "
              "\"steps\": %d, \"e2e_it_s\": %.6e, \"device_it_s\": %.6e, \"e2e_over_device\": %.4f, "
              "\"best_total\": %.17g}\n",
              chains, static_cast<unsigned long long>(iters), steps, total / wall,
              total / (dev_ms / 1e3), (total / wall) / (total / (dev_ms / 1e3)), best);
  return 0;
}
