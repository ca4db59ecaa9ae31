/*
 * TEST INFRASTRUCTURE ONLY — the parity oracle, never the product.
 *
 * Plain-C restatement of the reference `hsolve` algorithms on the SPD-solve
 * hot path (GP kernel assembly, blocked CG, blocked right-looking Cholesky
 * and substitutions). Each function cites the reference file:line it
 * follows (paths relative to /root/reference/proj). Arithmetic order is the
 * reference's, compiled without FMA contraction, so results are bitwise
 * identical to the reference; tests/test_oracle_vs_ref.py pins that against
 * oracle/_ref (the real reference, built here) and tests/golden/ (fixtures
 * generated from the real reference by tests/golden/make_golden.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.
 *
 * Status codes: 0 = ok, otherwise 1 + ErrorKind (errors.hpp:10-21):
 *   1 config, 2 not_spd, 3 singular_block, 4 numerical, 5 not_converged.
 */
#ifndef HS_ORACLE_H
#define HS_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* genmat.cpp:16-34 */
uint64_t hso_rng_at(uint64_t key, uint64_t counter);
double hso_uniform01(uint64_t key, uint64_t counter);
double hso_uniform_pm1(uint64_t key, uint64_t counter);

/* genmat.cpp:77-89 ; out: n*dim row-major */
int hso_generate_inputs(size_t n, size_t dim, uint64_t seed, double* out);
/* genmat.cpp:91-112 */
double hso_median_pairwise_distance(const double* pts, size_t n, size_t dim);
/* genmat.cpp:114-154 ; out: packed lower blocks, N(N+1)/2*b*b doubles */
int hso_generate_spd(size_t n, size_t b, double sigma_f2, double length_scale,
                     double sigma_n2, size_t dim, uint64_t seed, int threads,
                     double* out_packed);
/* genmat.cpp:156-162 ; out: N*b doubles */
void hso_generate_rhs(size_t n, size_t b, uint64_t seed, double* out);

/* block_kernels.cpp:59-100 over all block rows */
/* envelope measurement only: 0 = reference accumulation order (default),
 * 1 = per-tile partials added in ascending j (the GPU SYMV's class) */
void hso_set_symv_order(int order);
void hso_symv(size_t n, size_t b, const double* a, const double* x, double* y,
              int threads);
/* block_kernels.cpp:102-121 (+ dd.hpp:18-40): full-range compensated dot */
double hso_dot(size_t n, size_t b, const double* u, const double* v);

/* cg_solver.cpp:223-368, homogeneous mode (fraction 0/1; the reference's
 * heterogeneous splits are bitwise identical, test_cg_solver.cpp:93-129).
 * stats: [iterations, recomputations, converged, u0, true_residual].
 * trace (nullable): 3 doubles (u, alpha, beta) per iteration, up to cap. */
int hso_solve_cg(size_t n, size_t b, const double* a, const double* rhs,
                 double eps, size_t max_iters, size_t recompute_interval,
                 int threads, double* x, double* stats, double* trace,
                 size_t trace_cap, int64_t* err_iter);

/* block_kernels.cpp:9-57 */
int hso_potf_block(double* d, size_t b, int64_t* pivot);
int hso_trsm_block(double* x, const double* l, size_t b, int64_t* index);
void hso_gemm_update(double* c, const double* p, const double* q, size_t b);
void hso_syrk_update(double* c, const double* p, size_t b);

/* cholesky_solver.cpp:158-254 (homogeneous); err_row/err_pivot on not_spd */
int hso_factorize(size_t n, size_t b, double* a, int threads, int64_t* err_row,
                  int64_t* err_pivot);
/* cholesky_solver.cpp:23-42, 256-273 */
int hso_forward_substitute(size_t n, size_t b, const double* l,
                           const double* rhs, double* y);
int hso_back_substitute(size_t n, size_t b, const double* l, const double* y,
                        double* x);
/* cholesky_solver.cpp:275-331 ; a is destroyed (holds L). stats:
 * [true_residual] */
int hso_solve_spd(size_t n, size_t b, double* a, const double* rhs,
                  int threads, double* x, double* stats, int64_t* err_row,
                  int64_t* err_pivot);

/* partition.cpp:11-47 (return SIZE_MAX on a config error) */
size_t hso_partition_for_fraction(double fraction, size_t block_rows);
size_t hso_cholesky_border(double fraction, size_t column, size_t block_rows);

#ifdef __cplusplus
}
#endif
#endif
