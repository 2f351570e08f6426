/*
 * jofc_workloads.h -- seeded synthetic inputs for the BASELINE.json configs
 * (exported by libjofc_gpu.so; input preparation, not part of the hot path).
 *
 * All randomness is the reference's Rng (mt19937_64, 53-bit uniforms,
 * Box-Muller with a cached spare; proj/include/jofc/rng.hpp:17-55) so any
 * caller holding the reference can regenerate the same bits.  The recipe for
 * each config is documented in DESIGN.md ("Synthetic workloads").
 *   cfg 1: m=2  n=500   d=2 p=2   general(diag 1-w, off w), w=0.5, 100 it
 *   cfg 2: m=3  n=2000  d=3 p=4   uniform(0.9), 200 it
 *   cfg 3: m=2  n=20000 d=5 p=10  uniform(0.5), 100 it
 *   cfg 4: m=10 n=10000 d=3 p=3   uniform(0.99), 100 it
 *   cfg 5: m=2  n=5000  d=3 p=3   uniform(0.5), 100 it; + k=1000 OOS points
 */
#ifndef JOFC_WORKLOADS_H
#define JOFC_WORKLOADS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  size_t m, n, d, p;   /* modalities, objects, embedding dim, feature dim */
  size_t iterations;
  double w;
  int general_weights; /* 1: general(diag 1-w, off w); 0: uniform(w) */
  size_t oos_points;   /* cfg 5 only */
} jofc_workload_shape;

int jofc_wl_shape(int cfg, jofc_workload_shape* out);
/* Per-modality features (m x n_total x p, row-major) for n_total objects.
 * For cfg 5, n_total = n + oos_points (in-sample rows first). */
int jofc_wl_features(int cfg, uint64_t seed, size_t n_total, double* out);
/* X0 ~ N(0,1), block-major (l, i, c), from Rng(seed). */
void jofc_wl_normals(uint64_t seed, size_t count, double scale, double* out);
/* euclidean_distance_matrix of n x p features (reference arithmetic; OpenMP
 * over rows, bit-identical to the serial reference). */
void jofc_wl_distance_matrix(size_t n, size_t p, const double* feats, double* out);
/* OOS dissimilarities: for each new object q < k and modality l, the distances
 * from feats[l][n + q] to feats[l][0..n).  out is k x m x n. */
void jofc_wl_oos_deltas(size_t m, size_t n, size_t k, size_t p, const double* feats,
                        double* out);
/* oos_embed's start (proj/src/oos.cpp:189-198) for one point. */
void jofc_wl_oos_start(size_t m, size_t n, size_t d, const double* x, uint64_t seed, double* y0);

#ifdef __cplusplus
}
#endif
#endif
