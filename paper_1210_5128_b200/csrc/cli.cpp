// bnmc_b200 — command-line driver of the B200 backend with the reference
// CLI's subcommands and flags for the hot path (/root/reference/proj/tools/
// bnmc.cpp): `learn` (bnmc.cpp:91-138), `eval` incl. the prior-perturbation
// `--sweep` (bnmc.cpp:140-212) and `bench` (bnmc.cpp:214-339, GPU rows in the
// same CSV schema). Outputs of `learn` are byte-identical to the reference's
// (summary minus its '#' timing lines, trace CSV, best edges). Exit codes as
// the reference: 2 usage, 3 data, 4 capacity, 1 other (bnmc.cpp:454-465).
// `generate` is not provided (the generator is off the hot path).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <map>
#include <numeric>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/bnmc_b200/bnmc.hpp"
#include "../../include/bnmc_b200/io.hpp"
#include "../../include/bnmc_synth.h"

using namespace bnmc;

namespace {

double since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// --name value / --name=value / boolean --name; unknown flags are usage errors.
class Args {
 public:
  Args(int argc, char** argv, int first, const std::vector<std::string>& valued,
       const std::vector<std::string>& flags) {
    for (int i = first; i < argc; ++i) {
      std::string a = argv[i];
      if (a.rfind("--", 0) != 0) throw UsageError("unexpected argument '" + a + "'");
      std::string val;
      const auto eq = a.find('=');
      bool has_val = false;
      if (eq != std::string::npos) {
        val = a.substr(eq + 1);
        a = a.substr(0, eq);
        has_val = true;
      }
      const bool is_valued = std::find(valued.begin(), valued.end(), a) != valued.end();
      const bool is_flag = std::find(flags.begin(), flags.end(), a) != flags.end();
      if (!is_valued && !is_flag) throw UsageError("unknown option " + a);
      if (is_flag) {
        if (has_val) throw UsageError(a + " takes no value");
        vals_[a] = "1";
        continue;
      }
      if (!has_val) {
        if (i + 1 >= argc) throw UsageError(a + " requires a value");
        val = argv[++i];
      }
      vals_[a] = val;
    }
  }
  bool has(const std::string& k) const { return vals_.count(k) != 0; }
  std::string str(const std::string& k, const std::string& def = "") const {
    const auto it = vals_.find(k);
    return it == vals_.end() ? def : it->second;
  }
  std::string required(const std::string& k) const {
    if (!has(k)) throw UsageError(k + " is required");
    return str(k);
  }
  template <class T>
  T num(const std::string& k, T def) const {
    if (!has(k)) return def;
    std::istringstream ss(str(k));
    T v{};
    if (!(ss >> v) || !ss.eof()) throw UsageError(k + ": invalid value '" + str(k) + "'");
    return v;
  }

 private:
  std::map<std::string, std::string> vals_;
};

const std::vector<std::string> kRunValued = {"--iterations", "--max-parents", "--gamma", "--ess",
                                             "--seed", "--workers", "--track-top",
                                             "--tasks-per-node", "--memory-cap", "--device",
                                             "--gpus"};

RunConfig run_config(const Args& a) {
  RunConfig c;
  c.iterations = a.num<std::uint64_t>("--iterations", c.iterations);
  c.max_parents = a.num<int>("--max-parents", c.max_parents);
  c.gamma = a.num<double>("--gamma", c.gamma);
  c.ess = a.num<double>("--ess", c.ess);
  c.seed = a.num<std::uint64_t>("--seed", c.seed);
  c.workers = a.num<int>("--workers", c.workers);
  c.track_top = a.num<int>("--track-top", c.track_top);
  c.tasks_per_node = a.num<int>("--tasks-per-node", c.tasks_per_node);
  c.memory_cap_bytes = a.num<std::uint64_t>("--memory-cap", c.memory_cap_bytes);
  c.device = a.num<int>("--device", 0);
  c.n_gpus = a.num<int>("--gpus", 1);
  if (a.has("--strict-paper-tracker")) c.strict_paper_tracker = true;
  if (a.has("--k2")) c.alpha_mode = AlphaMode::kK2;
  if (a.has("--pst") && a.has("--unrank")) throw UsageError("--pst excludes --unrank");
  if (a.has("--unrank")) c.use_pst = false;
  return c;
}

int cmd_learn(int argc, char** argv) {  // bnmc.cpp:100-138
  std::vector<std::string> valued = kRunValued;
  for (const char* k : {"--data", "--priors", "--save-cache", "--load-cache", "--out-prefix"})
    valued.push_back(k);
  const Args a(argc, argv, 2, valued, {"--strict-paper-tracker", "--pst", "--unrank", "--k2"});
  const std::string data_path = a.required("--data");
  const std::string out_prefix = a.required("--out-prefix");
  RunConfig cfg = run_config(a);
  cfg.validate();
  const Dataset data = read_dataset_csv(data_path);
  if (data.rows() == 0) throw DataError(data_path + ": no data rows");
  const PriorMatrix priors =
      a.has("--priors") ? read_prior_csv(a.str("--priors"), data.n()) : PriorMatrix::neutral(data.n());
  ScoreCache loaded;
  const ScoreCache* prebuilt = nullptr;
  if (a.has("--load-cache")) {
    RunConfig lc = cfg;
    loaded = ScoreCache::load(a.str("--load-cache"), lc);
    if (loaded.n() != data.n())
      throw DataError(a.str("--load-cache") + ": cache node count " + std::to_string(loaded.n()) +
                      " != dataset " + std::to_string(data.n()));
    prebuilt = &loaded;
  }
  ScoreCache built;
  double pre = 0.0;
  if (!prebuilt) {  // built here once, so --save-cache needs no second build
    const auto t0 = std::chrono::steady_clock::now();
    built = ScoreCache::build(data, cfg);
    pre = since(t0);
  }
  McmcResult r = run_mcmc(data, cfg, priors, prebuilt ? prebuilt : &built);
  if (!prebuilt) r.preprocess_seconds = pre;
  write_summary(out_prefix + ".summary.txt", cfg, r);
  write_trace_csv(out_prefix + ".trace.csv", r.trace);
  write_edge_list(out_prefix + ".best.edges", r.tracker.best().dag);
  if (a.has("--save-cache") && !prebuilt) built.save(a.str("--save-cache"));
  std::cout << "best_score: " << format_double(r.tracker.best_score()) << "\n"
            << "best_edges: " << r.tracker.best().dag.edge_count() << "\n"
            << "acceptance_rate: " << static_cast<double>(r.accepted) / cfg.iterations << "\n"
            << "preprocess_seconds: " << r.preprocess_seconds << "\n"
            << "sampling_seconds: " << r.sampling_seconds << "\n"
            << "outputs: " << out_prefix << ".summary.txt, .trace.csv, .best.edges\n";
  return 0;
}

void metrics_row(std::ostream& out, const std::string& label, double hi, double lo,
                 double fraction, const ConfusionCounts& c, double best) {  // bnmc.cpp:150-158
  out << label << "," << format_double(hi) << "," << format_double(lo) << ","
      << format_double(fraction) << "," << c.tp << "," << c.fp << "," << c.fn << "," << c.tn
      << "," << format_double(c.tp_rate()) << "," << format_double(c.fp_rate()) << ","
      << format_double(c.f1()) << "," << format_double(best) << "\n";
}

int cmd_eval(int argc, char** argv) {  // bnmc.cpp:160-212
  std::vector<std::string> valued = {"--learned", "--truth", "--nodes", "--out", "--data",
                                     "--iterations", "--max-parents", "--gamma", "--ess",
                                     "--seed", "--workers", "--track-top", "--device"};
  const Args a(argc, argv, 2, valued, {"--sweep"});
  std::ofstream file;
  std::ostream* out = &std::cout;
  if (a.has("--out")) {
    file.open(a.str("--out"));
    if (!file) throw DataError("cannot open " + a.str("--out") + " for writing");
    out = &file;
  }
  *out << "label,prior_hi,prior_lo,fraction,tp,fp,fn,tn,tp_rate,fp_rate,f1,best_score\n";
  const Dag truth = read_edge_list(a.required("--truth"), a.num<int>("--nodes", 0));
  if (!a.has("--sweep")) {
    if (!a.has("--learned")) throw UsageError("--learned is required without --sweep");
    const Dag learned = read_edge_list(a.str("--learned"), truth.n());
    metrics_row(*out, "eval", 0.5, 0.5, 0.0, confusion(learned, truth), 0.0);
    return 0;
  }
  if (!a.has("--data")) throw UsageError("--sweep requires --data");
  const Dataset data = read_dataset_csv(a.str("--data"));
  if (truth.n() != data.n()) throw DataError("truth graph and dataset disagree on node count");
  RunConfig cfg = run_config(a);
  cfg.validate();
  // one device table serves the five runs; each prior matrix refolds the keys
  const ScoreCache cache = ScoreCache::build(data, cfg);
  const McmcResult base = run_mcmc(data, cfg, PriorMatrix::neutral(data.n()), &cache);
  const Dag& base_dag = base.tracker.best().dag;
  metrics_row(*out, "baseline", 0.5, 0.5, 0.0, confusion(base_dag, truth), base.tracker.best_score());
  const std::pair<double, double> strengths[2] = {{0.7, 0.2}, {0.8, 0.1}};
  const double fractions[2] = {0.2, 0.4};
  const Rng master(cfg.seed);
  int k = 0;
  for (const auto& st : strengths)
    for (const double f : fractions) {
      Rng proto = master.split(201 + k++);
      const PriorMatrix pr = prior_perturbation_protocol(truth, base_dag, st, f, proto);
      const McmcResult run = run_mcmc(data, cfg, pr, &cache);
      metrics_row(*out, "priors", st.first, st.second, f, confusion(run.tracker.best().dag, truth),
                  run.tracker.best_score());
    }
  return 0;
}

std::vector<int> int_list(const std::string& csv, const std::string& flag) {
  std::vector<int> out;
  std::string f;
  std::istringstream ss(csv);
  while (std::getline(ss, f, ',')) {
    try {
      out.push_back(std::stoi(f));
    } catch (const std::exception&) {
      throw UsageError(flag + ": expected a comma-separated integer list");
    }
  }
  if (out.empty()) throw UsageError(flag + ": empty list");
  return out;
}

// bench (bnmc.cpp:214-339) on the device, same CSV schema: per node count, the
// precompute, then OrderScorer::score on `reps` fixed random orders
// (Rng(seed).split(7), as the reference) one call per order ("iteration") and
// all orders in one call ("iteration_batched", per order), then `chains`
// chains x `chain_iters` iterations ("chain_iteration", seconds per chain
// iteration, speedup = chains in flight).
int cmd_bench(int argc, char** argv) {
  const Args a(argc, argv, 2,
               {"--scaling-nodes", "--workers-list", "--samples", "--reps", "--enum-candidates",
                "--seed", "--max-parents", "--out", "--chains", "--chain-iters", "--device",
                "--gpus"},
               {});
  std::ofstream file;
  std::ostream* out = &std::cout;
  if (a.has("--out")) {
    file.open(a.str("--out"));
    if (!file) throw DataError("cannot open " + a.str("--out") + " for writing");
    out = &file;
  }
  const long samples = a.num<long>("--samples", 200);
  const int reps = a.num<int>("--reps", 20);
  const std::uint64_t seed = a.num<std::uint64_t>("--seed", 1);
  const int chains = a.num<int>("--chains", 1024);
  const std::uint64_t chain_iters = a.num<std::uint64_t>("--chain-iters", 200);
  if (a.num<int>("--enum-candidates", 0) > 0)
    throw UsageError("--enum-candidates: the 2^c bit-vector baseline is CPU-only (reference)");
  RunConfig cfg;
  cfg.max_parents = a.num<int>("--max-parents", 4);
  cfg.seed = seed;
  cfg.device = a.num<int>("--device", 0);
  cfg.n_gpus = a.num<int>("--gpus", 1);
  *out << "phase,nodes,workers,candidates,reps,seconds,speedup\n";
  for (const int n : int_list(a.str("--scaling-nodes", "13,20"), "--scaling-nodes")) {
    if (n < 2 || n > kMaxNodes) throw UsageError("--scaling-nodes entries must lie in [2,64]");
    // synth_dataset (bnmc.cpp:224-233): random_dag(n, s, 0.25), binary, Dirichlet(1)
    std::vector<int> cards(n, 2);
    std::vector<std::uint8_t> cells(static_cast<std::size_t>(samples) * n);
    std::vector<std::uint64_t> truth(n);
    if (bnmc_synth_instance(n, cfg.max_parents, 0.25, 1.0, samples, cards.data(), seed, 101, 102,
                            103, cells.data(), truth.data()) != 0)
      throw DataError(bnmc_synth_last_error());
    const Dataset data(cards, cells);
    auto t0 = std::chrono::steady_clock::now();
    const ScoreCache cache = ScoreCache::build(data, cfg);
    *out << "preprocess," << n << ",1,,1," << format_double(since(t0)) << ",\n";
    Rng orng = Rng(seed).split(7);
    std::vector<Order> orders;
    for (int r = 0; r < reps; ++r) {
      std::vector<int> p(n);
      std::iota(p.begin(), p.end(), 0);
      shuffle(p, orng);
      orders.emplace_back(std::move(p));
    }
    const PriorMatrix neutral = PriorMatrix::neutral(n);
    const OrderScorer scorer(cache, neutral, EngineConfig{});
    scorer.score(orders[0]);  // warm-up (sorted rows, workspace)
    t0 = std::chrono::steady_clock::now();
    for (const Order& o : orders) scorer.score(o);
    const double per = since(t0) / reps;
    *out << "iteration," << n << ",1,," << reps << "," << format_double(per) << ",\n";
    t0 = std::chrono::steady_clock::now();
    scorer.score_many(orders);
    const double per_b = since(t0) / reps;
    *out << "iteration_batched," << n << ",1,," << reps << "," << format_double(per_b) << ","
         << format_double(per / per_b) << "\n";
    RunConfig cc = cfg;
    cc.iterations = chain_iters;
    std::vector<std::uint64_t> seeds(chains);
    std::iota(seeds.begin(), seeds.end(), seed);
    run_chains(cache, neutral, cc, std::span<const std::uint64_t>(seeds.data(), 1));  // warm-up
    t0 = std::chrono::steady_clock::now();
    run_chains(cache, neutral, cc, seeds);
    const double per_it = since(t0) / (static_cast<double>(chains) * chain_iters);
    *out << "chain_iteration," << n << ",1,," << chains << "," << format_double(per_it) << ","
         << format_double(per / per_it) << "\n";
  }
  return 0;
}

void usage() {
  std::cerr << "usage: bnmc_b200 <learn|eval|bench> [options]\n"
               "  learn --data F --out-prefix P [--priors F] [--iterations N] [--max-parents S]\n"
               "        [--gamma G] [--ess E] [--seed N] [--workers N] [--track-top K]\n"
               "        [--tasks-per-node N] [--memory-cap B] [--strict-paper-tracker]\n"
               "        [--pst|--unrank] [--k2] [--save-cache F] [--load-cache F] [--device D]\n"
               "        [--gpus G]\n"
               "  eval  --truth F (--learned F | --sweep --data F) [--nodes N] [--out F] ...\n"
               "  bench [--scaling-nodes L] [--samples N] [--reps N] [--seed N] [--max-parents S]\n"
               "        [--chains N] [--chain-iters N] [--out F] [--device D] [--gpus G]\n";
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 2) {
      usage();
      return 2;
    }
    const std::string cmd = argv[1];
    if (cmd == "learn") return cmd_learn(argc, argv);
    if (cmd == "eval") return cmd_eval(argc, argv);
    if (cmd == "bench") return cmd_bench(argc, argv);
    if (cmd == "--help" || cmd == "-h") {
      usage();
      return 0;
    }
    usage();
    return 2;
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  } catch (const CapacityError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 4;
  } catch (const DataError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
