/* bnmc_synth.h — synthetic BASELINE instances (input synthesis; NOT on the hot path).
 *
 * Bit-identical restatement of the reference generator used by `bnmc generate`
 * (proj/tools/bnmc.cpp:64-73): master = Rng(seed); random_dag(split(tag_dag))
 * (src/evalgen.cpp:38-51); random_ground_truth(split(tag_cpt)) (evalgen.cpp:53-75);
 * forward_sample(split(tag_rows)) (evalgen.cpp:77-109). Used by bench.py and the
 * tests to build the SURVEY §8d inputs on machines without the reference.
 * Status: 0 ok, 2 usage, 3 data.
 */
#ifndef BNMC_SYNTH_H
#define BNMC_SYNTH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* bnmc_synth_last_error(void);

/* cells_out: m x n row-major; truth_out: n parent masks of the generating DAG. */
int bnmc_synth_instance(int n, int max_parents, double edge_prob, double concentration,
                        uint64_t m, const int* cards, uint64_t seed, uint64_t tag_dag,
                        uint64_t tag_cpt, uint64_t tag_rows, uint8_t* cells_out,
                        uint64_t* truth_out);

/* SURVEY §8d prior matrix: R = 0.5; stream split(tag) of Rng(seed); for every
 * ordered pair (child c, parent p != c): edge in truth -> 0.75 w.p. 0.3, else
 * 0.25 w.p. 0.02. r_out is n x n row-major, r[c*n + p]. */
int bnmc_synth_priors(int n, const uint64_t* truth, uint64_t seed, uint64_t tag, double* r_out);

#ifdef __cplusplus
}
#endif
#endif
