/*
 * jofc_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's fJOFC hot path (arXiv 1502.03391,
 * reference tree proj/src/{solver,stress,weights,oos}.cpp and
 * proj/include/jofc/rng.hpp).  It is the CHECKER for the CUDA path: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load it.  Nothing in the product package links it.
 *
 * Parity pin: every function here is checked bit-for-bit against the real
 * reference compiled from /root/reference (oracle/_ref, see oracle/Makefile)
 * by tests/golden/make_golden.py, which writes the fixtures under
 * tests/golden/ that tests/test_oracle.py replays without the reference.
 *
 * Conventions: all matrices are dense row-major fp64.  Delta is m blocks of
 * n x n (modality-major), a configuration X is m blocks of n x d.
 * Status codes: 0 ok, 1 invalid argument, 2 numerical error (same meaning as
 * std::invalid_argument / jofc::NumericalError in the reference).
 */
#ifndef JOFC_ORACLE_H
#define JOFC_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Weight family, proj/include/jofc/weights.hpp:20-66.
 * kind 0: uniform(w)         a_l = 1,           w_ll' = w
 * kind 1: general(W, m x m)  a_l = W_ll,        w_ll' = W_ll'
 * kind 2: product(p, c)      a_l = c * p_l,     w_ll' = p_l * p_l' */
typedef struct {
  int kind;
  double w;              /* uniform */
  const double* general; /* m*m, general */
  const double* within;  /* m, product */
  double scale;          /* product fidelity scale c */
} jo_weights;

/* mt19937_64 + 53-bit uniforms + Box-Muller, proj/include/jofc/rng.hpp:17-55 */
typedef struct {
  uint64_t mt[312];
  int mti;
  double spare;
  int have_spare;
} jo_rng;

void jo_rng_seed(jo_rng* r, uint64_t seed);
uint64_t jo_rng_next_u64(jo_rng* r);
double jo_rng_uniform(jo_rng* r);
double jo_rng_normal(jo_rng* r);
void jo_rng_normals(uint64_t seed, size_t count, double scale, double* out);
/* a heap-allocated stream (ctypes callers): kind 0 uniform(), 1 normal() */
jo_rng* jo_rng_create(uint64_t seed);
void jo_rng_destroy(jo_rng* r);
void jo_rng_draw(jo_rng* r, int kind, size_t count, double* out);

/* proj/src/distance.cpp:8-29 (serial order; bitwise symmetric) */
int jo_euclidean_distance_matrix(size_t n, size_t p, const double* feats, double* out);

/* proj/src/weights.cpp:53-69 within_weight / cross_weight -> a (m), wc (m*m) */
int jo_weights_expand(const jo_weights* spec, size_t m, double* a, double* wc);
/* proj/src/weights.cpp:79-94 */
int jo_script_w(const jo_weights* spec, size_t m, size_t n, double* out);
/* proj/src/weights.cpp:96-127 (+ invert_small, proj/src/linalg.cpp:296-331) */
int jo_script_w_inverse(const jo_weights* spec, size_t m, size_t n, double* out);

/* proj/src/stress.cpp:34-37 */
double jo_stress_pair_count(size_t m, size_t n);
/* proj/src/stress.cpp:39-74 (serial order) */
int jo_raw_stress(size_t m, size_t n, size_t d, const double* delta, const jo_weights* spec,
                  const double* x, double* stress);
/* proj/src/solver.cpp:17-50 block_guttman_products -> products (m*n*d) */
int jo_block_guttman_products(size_t m, size_t n, size_t d, const double* delta,
                              const jo_weights* spec, const double* x, double* products);
/* proj/src/solver.cpp:154-161 guttman_step_fast (= products + mix :52-72) */
int jo_guttman_step_fast(size_t m, size_t n, size_t d, const double* delta,
                         const jo_weights* spec, const double* x, double* x_next);
/* proj/src/solver.cpp:106-150,223-236 fjofc_embed with InitKind::provided.
 * trace_out must hold max_it+1 doubles; returns the number of iterations
 * done in *iterations and 1 in *converged when the eps rule fired. */
int jo_fjofc_embed(size_t m, size_t n, size_t d, const double* delta, const jo_weights* spec,
                   const double* x0, double eps, size_t max_it, int normalize,
                   double* x_out, double* trace_out, size_t* iterations, int* converged);

/* proj/src/oos.cpp:43-71 ; deltas is m*n (one row per modality), y is m*d */
int jo_oos_stress(size_t m, size_t n, size_t d, const double* y, const double* x,
                  const double* deltas, double w, double* stress);
/* proj/src/oos.cpp:73-113 */
int jo_oos_step_fast(size_t m, size_t n, size_t d, const double* y, const double* x,
                     const double* deltas, double w, double* y_next);
/* proj/src/oos.cpp:180-229 ; y0 drawn from Rng(seed) exactly as the reference */
int jo_oos_start(size_t m, size_t n, size_t d, const double* x, uint64_t seed, double* y0);
int jo_oos_embed(size_t m, size_t n, size_t d, const double* x, const double* deltas,
                 double w, double eps, size_t max_it, uint64_t seed, double* y_out,
                 double* trace_out, size_t* iterations, int* converged);
/* Batch of k independent OOS embeds from caller-given starts (y0: k*m*d,
 * deltas: k*m*n), each with the per-point stop rule of proj/src/oos.cpp:221-226.
 * fixed_iterations != 0 ignores the stop rule (the reference's own timing
 * style, proj/tests/acceptance/acceptance_main.cpp:457-460). OpenMP over points. */
int jo_oos_batch(size_t k, size_t m, size_t n, size_t d, const double* x, const double* deltas,
                 double w, const double* y0, double eps, size_t max_it, int fixed_iterations,
                 double* y_out, double* traces, size_t* iterations);

const char* jo_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
