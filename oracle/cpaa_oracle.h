/* TEST INFRASTRUCTURE — CPU oracle for the CPAA hot path (plain C restatement).
 *
 * This is the checker, never the thing measured or shipped: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.  Every
 * function restates the reference algorithm it cites (paths relative to
 * /root/reference/proj) with the same floating-point operation order, so that
 * its results are bit-identical to the reference's.  Parity pinned: the tests
 * in tests/test_oracle.py check it against the reference compiled unmodified
 * (oracle/_ref) and against the reference's own golden vectors.
 *
 * Status codes: 0 ok, 1 validation, 2 domain, 3 numeric, 4 invalid argument,
 * 5 capacity (same numbering as include/chebpr_cuda.h).
 */
#ifndef CHEBPR_ORACLE_H
#define CHEBPR_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* or_last_error(void);
void or_free(void* p);

/* src/graph.cpp:10-19 */
double or_kahan_sum(const double* x, int64_t n);

/* src/coefficients.cpp:20-23,33-71 */
int or_beta(double c, double* out);
int or_err_bound(double c, int M, double* out);
int or_plan_iterations(double c, double eps, int* M, double* predicted);
int or_coefficients(double c, int M, double* coeffs /* M+1 */, double* beta, double* c0);

/* std::mt19937_64 + src/generate.cpp:11-19,51-87 */
int or_gnp_edges(int64_t n, double p, uint64_t seed, int64_t** edges, int64_t* count);

/* Synthetic generators of BASELINE configs 2-5 (oracle/synth_gen.c): the product's
 * counter-based R-MAT / Chung-Lu definition restated; int64 (u, v) pairs, malloc'ed. */
int or_rmat_edges(int scale, int64_t edge_factor, double a, double b, double c, uint64_t seed,
                  int64_t** edges, int64_t* count);
int or_chung_lu_edges(int64_t n, double gamma, double wmin, double wmax, int64_t draws, uint64_t seed,
                      int64_t** edges, int64_t* count);

/* src/graph.cpp:23-102.  Outputs are malloc'ed (free with or_free). */
int or_build_graph(const int64_t* edges, int64_t E, int dedup, int drop_isolated,
                   int64_t n_hint, int64_t* n_out, int64_t* m_out, int64_t** offsets,
                   int64_t** neighbors, int64_t** degrees, double** inv_degree,
                   int64_t* duplicates_removed, int64_t* isolated_dropped);

/* src/graph.cpp:104-121 */
void or_transition_apply(int64_t n, const int64_t* offsets, const int64_t* neighbors,
                         const double* inv_degree, const double* x, double* y);

/* src/cpaa.cpp:40-68 */
int or_partition_vertices(int64_t n, const int64_t* degrees, int K, int64_t* cuts /* K+1 */);

/* src/cpaa.cpp:79-165 with M already resolved (cpaa.cpp:28-36) and the
 * optional personalisation start T0 = p (NULL = ones, exactly as the reference).
 * trace_out (may be NULL): M rows of 10 doubles
 *   k, c_k, S_k, residual_mass, l1_change(0), elapsed(0), mass_T, err(0), err_l1(0), 0. */
int or_run_cpaa(int64_t n, const int64_t* offsets, const int64_t* neighbors,
                const double* inv_degree, double c, int M, const double* p,
                double* ranks, double* trace_out, double* total_mass);

/* src/power.cpp:28-109.  rounds>=0 fixed, else tol>0 with max_rounds. */
int or_run_power(int64_t n, const int64_t* offsets, const int64_t* neighbors,
                 const double* inv_degree, double c, int rounds, double tol, int max_rounds,
                 double* ranks, double* trace_out, int* rounds_out, double* total_mass);

#ifdef __cplusplus
}
#endif
#endif
