// bnmc_b200/io.hpp — the reference's file formats around the hot path
// (/root/reference/proj/include/bnmc/io.hpp, src/io.cpp), so that `learn` on
// the B200 backend writes byte-identical outputs: dataset CSV with
// "#cards:", prior matrix CSV, edge lists, trace CSV, run summary, and the
// round-trip-exact double formatting (std::to_chars). Host code only.
#ifndef BNMC_B200_IO_HPP
#define BNMC_B200_IO_HPP

#include <iosfwd>
#include <string>
#include <vector>

#include "bnmc.hpp"

namespace bnmc {

// Dataset CSV: header row of variable names, one row of integer states per
// sample, '#' comments; "#cards: c0,c1,..." pins the cardinalities, else they
// are max state + 1 with a floor of 2 (io.cpp:69-126).
Dataset read_dataset_csv(const std::string& path);
Dataset read_dataset_csv(std::istream& in, const std::string& name);
void write_dataset_csv(const std::string& path, const Dataset& data);

// n rows of n comma-separated decimals in [0,1] (io.cpp:143-176).
PriorMatrix read_prior_csv(const std::string& path, int expected_n);
void write_prior_csv(const std::string& path, const PriorMatrix& priors);

// "child parent" per line, "# nodes: n" header (io.cpp:178-224).
Dag read_edge_list(const std::string& path, int expected_n = 0);
void write_edge_list(const std::string& path, const Dag& dag);

// iteration,proposed_score,accepted,best_score (io.cpp:243-252).
void write_trace_csv(const std::string& path, const std::vector<TraceRow>& trace);

// Deterministic "key: value" summary; timings as '#' comments (io.cpp:254-282).
void write_summary(const std::string& path, const RunConfig& cfg, const McmcResult& result);

std::string format_double(double v);  // shortest round-trip form

// ---- evaluation helpers of `eval --sweep` (evalgen.hpp:44-62)
struct ConfusionCounts {
  std::uint64_t tp = 0, fp = 0, fn = 0, tn = 0;
  double tp_rate() const { return tp + fn == 0 ? 0.0 : double(tp) / double(tp + fn); }
  double fp_rate() const { return fp + tn == 0 ? 0.0 : double(fp) / double(fp + tn); }
  double f1() const { return 2 * tp + fp + fn == 0 ? 0.0 : 2.0 * tp / (2.0 * tp + fp + fn); }
};
ConfusionCounts confusion(const Dag& learned, const Dag& truth);
PriorMatrix prior_perturbation_protocol(const Dag& truth, const Dag& baseline,
                                        std::pair<double, double> strengths, double fraction,
                                        Rng& rng);

}  // namespace bnmc

#endif
