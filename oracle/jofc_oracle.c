/*
 * jofc_oracle.c -- TEST INFRASTRUCTURE ONLY (see jofc_oracle.h).
 *
 * A plain-C restatement of the reference fJOFC hot path.  Evaluation order
 * follows the reference line by line so that, compiled without FMA
 * contraction (-ffp-contract=off, as the reference's x86-64 build is), the
 * results are bit-identical to the reference; tests/test_oracle.py holds the
 * pins.  Serial everywhere except jo_oos_batch, whose parallelism over
 * independent points is the harness's, not the reference's.
 */
#include "jofc_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* jo_last_error(void) { return g_err; }

/* ---------------- Rng: proj/include/jofc/rng.hpp:17-55 ---------------- */
#define MT_N 312
#define MT_M 156
#define MT_A 0xB5026F5AA96619E9ULL
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL

void jo_rng_seed(jo_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->mti = MT_N;
  r->spare = 0.0;
  r->have_spare = 0;
}

static void mt_twist(jo_rng* r) {
  for (int i = 0; i < MT_N; ++i) {
    const uint64_t y = (r->mt[i] & MT_UPPER) | (r->mt[(i + 1) % MT_N] & MT_LOWER);
    r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL);
  }
  r->mti = 0;
}

uint64_t jo_rng_next_u64(jo_rng* r) {
  if (r->mti >= MT_N) mt_twist(r);
  uint64_t x = r->mt[r->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

/* rng.hpp:24-26: 53 random bits scaled by 2^-53 */
double jo_rng_uniform(jo_rng* r) { return (double)(jo_rng_next_u64(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:31-44: Box-Muller with a cached spare (cos first, sin cached) */
double jo_rng_normal(jo_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u1 = jo_rng_uniform(r);
  while (u1 <= 0.0) u1 = jo_rng_uniform(r);
  const double u2 = jo_rng_uniform(r);
  const double rad = sqrt(-2.0 * log(u1));
  const double theta = 2.0 * 3.14159265358979323846 * u2;
  r->spare = rad * sin(theta);
  r->have_spare = 1;
  return rad * cos(theta);
}

void jo_rng_normals(uint64_t seed, size_t count, double scale, double* out) {
  jo_rng r;
  jo_rng_seed(&r, seed);
  for (size_t i = 0; i < count; ++i) out[i] = scale * jo_rng_normal(&r);
}

jo_rng* jo_rng_create(uint64_t seed) {
  jo_rng* r = (jo_rng*)malloc(sizeof(jo_rng));
  if (r) jo_rng_seed(r, seed);
  return r;
}

void jo_rng_destroy(jo_rng* r) { free(r); }

void jo_rng_draw(jo_rng* r, int kind, size_t count, double* out) {
  for (size_t i = 0; i < count; ++i) out[i] = kind ? jo_rng_normal(r) : jo_rng_uniform(r);
}

/* ---------------- distance.cpp:8-29 ---------------- */
int jo_euclidean_distance_matrix(size_t n, size_t p, const double* x, double* out) {
  for (size_t i = 0; i < n * p; ++i)
    if (!isfinite(x[i])) return fail(1, "euclidean_distance_matrix: non-finite input");
  for (size_t i = 0; i < n; ++i) out[i * n + i] = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const double* xi = x + i * p;
    for (size_t j = i + 1; j < n; ++j) {
      const double* xj = x + j * p;
      double s = 0.0;
      for (size_t k = 0; k < p; ++k) {
        const double diff = xi[k] - xj[k];
        s += diff * diff;
      }
      const double dist = sqrt(s);
      out[i * n + j] = dist;
      out[j * n + i] = dist;
    }
  }
  return 0;
}

/* ---------------- weights.cpp ---------------- */
static int require_positive(double w) { return (w > 0.0) && isfinite(w); }

/* weights.cpp:21-51 (factory validation) + :71-77 (validate(m)) */
static int validate_spec(const jo_weights* s, size_t m) {
  if (m == 0) return fail(1, "WeightSpec: m must be positive");
  switch (s->kind) {
    case 0:
      if (!require_positive(s->w)) return fail(1, "WeightSpec: w must be strictly positive");
      return 0;
    case 1:
      if (!s->general) return fail(1, "WeightSpec: general weight matrix size mismatch");
      for (size_t i = 0; i < m; ++i)
        for (size_t j = i + 1; j < m; ++j)
          if (fabs(s->general[i * m + j] - s->general[j * m + i]) > 0.0)
            return fail(1, "WeightSpec: general weight matrix must be symmetric");
      for (size_t i = 0; i < m * m; ++i)
        if (!require_positive(s->general[i]))
          return fail(1, "WeightSpec: w_ij must be strictly positive");
      return 0;
    case 2:
      if (!s->within) return fail(1, "WeightSpec: product weight count mismatch");
      for (size_t i = 0; i < m; ++i)
        if (!require_positive(s->within[i]))
          return fail(1, "WeightSpec: w_ii must be strictly positive");
      if (!require_positive(s->scale)) return fail(1, "WeightSpec: c must be strictly positive");
      return 0;
  }
  return fail(1, "WeightSpec: unknown kind");
}

/* weights.cpp:53-60 */
static double within_weight(const jo_weights* s, size_t m, size_t i) {
  switch (s->kind) {
    case 0: return 1.0;
    case 1: return s->general[i * m + i];
    case 2: return s->scale * s->within[i];
  }
  return 1.0;
}

/* weights.cpp:62-69 */
static double cross_weight(const jo_weights* s, size_t m, size_t i, size_t j) {
  switch (s->kind) {
    case 0: return s->w;
    case 1: return s->general[i * m + j];
    case 2: return s->within[i] * s->within[j];
  }
  return 0.0;
}

int jo_weights_expand(const jo_weights* spec, size_t m, double* a, double* wc) {
  int rc = validate_spec(spec, m);
  if (rc) return rc;
  for (size_t i = 0; i < m; ++i) {
    a[i] = within_weight(spec, m, i);
    for (size_t j = 0; j < m; ++j) wc[i * m + j] = (i == j) ? 0.0 : cross_weight(spec, m, i, j);
  }
  return 0;
}

/* weights.cpp:79-94 */
int jo_script_w(const jo_weights* spec, size_t m, size_t n, double* w) {
  int rc = validate_spec(spec, m);
  if (rc) return rc;
  if (n < 2) return fail(1, "script_w: n must be at least 2");
  for (size_t i = 0; i < m; ++i) {
    double diag = (double)n * within_weight(spec, m, i);
    for (size_t j = 0; j < m; ++j) {
      if (j == i) continue;
      const double cross = cross_weight(spec, m, i, j);
      diag += cross;
      w[i * m + j] = -cross;
    }
    w[i * m + i] = diag;
  }
  return 0;
}

/* linalg.cpp:296-331 invert_small: partial-pivot Gauss-Jordan */
static int invert_small(size_t n, const double* a, double* inv) {
  double* work = (double*)malloc(n * n * sizeof(double));
  memcpy(work, a, n * n * sizeof(double));
  double amax = 0.0;
  for (size_t i = 0; i < n * n; ++i) amax = fmax(amax, fabs(a[i]));
  for (size_t i = 0; i < n * n; ++i) inv[i] = 0.0;
  for (size_t i = 0; i < n; ++i) inv[i * n + i] = 1.0;
  const double floor_ = 1e-13 * fmax(1.0, amax);
  for (size_t col = 0; col < n; ++col) {
    size_t pivot = col;
    for (size_t r = col + 1; r < n; ++r)
      if (fabs(work[r * n + col]) > fabs(work[pivot * n + col])) pivot = r;
    if (fabs(work[pivot * n + col]) < floor_) {
      free(work);
      return fail(2, "invert_small: singular matrix");
    }
    if (pivot != col)
      for (size_t j = 0; j < n; ++j) {
        double t = work[pivot * n + j];
        work[pivot * n + j] = work[col * n + j];
        work[col * n + j] = t;
        t = inv[pivot * n + j];
        inv[pivot * n + j] = inv[col * n + j];
        inv[col * n + j] = t;
      }
    const double dd = work[col * n + col];
    for (size_t j = 0; j < n; ++j) {
      work[col * n + j] /= dd;
      inv[col * n + j] /= dd;
    }
    for (size_t r = 0; r < n; ++r) {
      if (r == col) continue;
      const double f = work[r * n + col];
      if (f == 0.0) continue;
      for (size_t j = 0; j < n; ++j) {
        work[r * n + j] -= f * work[col * n + j];
        inv[r * n + j] -= f * inv[col * n + j];
      }
    }
  }
  free(work);
  return 0;
}

/* weights.cpp:96-127 */
int jo_script_w_inverse(const jo_weights* spec, size_t m, size_t n, double* inv) {
  int rc = validate_spec(spec, m);
  if (rc) return rc;
  if (n < 2) return fail(1, "script_w_inverse: n must be at least 2");
  const double nn = (double)n;
  if (spec->kind == 0) {
    const double w = spec->w;
    const double denom = nn * (nn + (double)m * w);
    const double diag = (nn + w) / denom;
    const double off = w / denom;
    for (size_t i = 0; i < m; ++i)
      for (size_t j = 0; j < m; ++j) inv[i * m + j] = (i == j) ? diag : off;
    return 0;
  }
  if (spec->kind == 2) {
    const double c = spec->scale;
    double sum = 0.0;
    for (size_t i = 0; i < m; ++i) sum += spec->within[i];
    const double cn = c * nn;
    const double off = 1.0 / (cn * (cn + sum));
    for (size_t i = 0; i < m; ++i)
      for (size_t j = 0; j < m; ++j)
        inv[i * m + j] = (i == j) ? 1.0 / (spec->within[i] * (cn + sum)) + off : off;
    return 0;
  }
  double* w = (double*)malloc(m * m * sizeof(double));
  jo_script_w(spec, m, n, w);
  rc = invert_small(m, w, inv);
  free(w);
  return rc;
}

/* weights.cpp:129-135 ScriptW::make: inverse + W*Winv ~ I check */
static int script_w_make(const jo_weights* spec, size_t m, size_t n, double* winv) {
  double* w = (double*)malloc(m * m * sizeof(double));
  int rc = jo_script_w(spec, m, n, w);
  if (!rc) rc = jo_script_w_inverse(spec, m, n, winv);
  if (!rc) {
    double wmax = 0.0, gap = 0.0;
    for (size_t i = 0; i < m * m; ++i) wmax = fmax(wmax, fabs(w[i]));
    for (size_t i = 0; i < m; ++i)
      for (size_t j = 0; j < m; ++j) {
        double s = 0.0;
        for (size_t k = 0; k < m; ++k) s += w[i * m + k] * winv[k * m + j];
        gap = fmax(gap, fabs(s - (i == j ? 1.0 : 0.0)));
      }
    if (gap > 1e-12 * fmax(1.0, wmax)) rc = fail(2, "ScriptW: inverse check failed");
  }
  free(w);
  return rc;
}

/* ---------------- stress.cpp ---------------- */
double jo_stress_pair_count(size_t m, size_t n) {
  const double mn = (double)m * (double)n;
  return mn * (mn - 1.0) / 2.0;
}

static double row_distance(const double* a, const double* b, size_t d) {
  double s = 0.0;
  for (size_t k = 0; k < d; ++k) {
    const double diff = a[k] - b[k];
    s += diff * diff;
  }
  return sqrt(s);
}

static int shapes_ok(size_t m, size_t n, size_t d, const jo_weights* spec) {
  int rc = validate_spec(spec, m);
  if (rc) return rc;
  if (n < 2) return fail(1, "OmnibusProblem: need at least two objects");
  if (d < 1) return fail(1, "configuration blocks have inconsistent shapes");
  return 0;
}

/* stress.cpp:39-74, serial order: per-row local sums scaled by a_l, then the
 * commensurability sum of squared (sqrt'd) matched distances. */
int jo_raw_stress(size_t m, size_t n, size_t d, const double* delta, const jo_weights* spec,
                  const double* x, double* stress) {
  int rc = shapes_ok(m, n, d, spec);
  if (rc) return rc;
  double fidelity = 0.0;
  for (size_t flat = 0; flat < m * n; ++flat) {
    const size_t l = flat / n, i = flat % n;
    const double* dl = delta + l * n * n;
    const double* xb = x + l * n * d;
    const double a = within_weight(spec, m, l);
    double local = 0.0;
    for (size_t j = i + 1; j < n; ++j) {
      const double resid = dl[i * n + j] - row_distance(xb + i * d, xb + j * d, d);
      local += resid * resid;
    }
    fidelity += a * local;
  }
  double commensurability = 0.0;
  for (size_t i = 0; i < m; ++i)
    for (size_t j = i + 1; j < m; ++j) {
      const double w = cross_weight(spec, m, i, j);
      double pairs = 0.0;
      for (size_t k = 0; k < n; ++k) {
        const double dd = row_distance(x + (i * n + k) * d, x + (j * n + k) * d, d);
        pairs += dd * dd;
      }
      commensurability += w * pairs;
    }
  *stress = fidelity + commensurability;
  return 0;
}

/* solver.cpp:17-50: P_l,i = sum_{k != i, dist != 0} (a_l delta_ik / dist)(x_i - x_k),
 * full Delta rows, k ascending. */
int jo_block_guttman_products(size_t m, size_t n, size_t d, const double* delta,
                              const jo_weights* spec, const double* x, double* products) {
  int rc = shapes_ok(m, n, d, spec);
  if (rc) return rc;
  memset(products, 0, m * n * d * sizeof(double));
  for (size_t l = 0; l < m; ++l) {
    const double* dl = delta + l * n * n;
    const double* xb = x + l * n * d;
    const double a = within_weight(spec, m, l);
    for (size_t i = 0; i < n; ++i) {
      const double* xi = xb + i * d;
      double* out = products + (l * n + i) * d;
      for (size_t k = 0; k < n; ++k) {
        if (k == i) continue;
        const double* xk = xb + k * d;
        double s = 0.0;
        for (size_t c = 0; c < d; ++c) {
          const double diff = xi[c] - xk[c];
          s += diff * diff;
        }
        const double dist = sqrt(s);
        if (dist == 0.0) continue;
        const double ratio = a * dl[i * n + k] / dist;
        for (size_t c = 0; c < d; ++c) out[c] += ratio * (xi[c] - xk[c]);
      }
    }
  }
  return 0;
}

/* solver.cpp:52-72: X'^(j)_i = sum_l Winv(j,l) P_l,i from 0.0, l ascending */
static void mix_products(size_t m, size_t n, size_t d, const double* products,
                         const double* winv, double* next) {
  memset(next, 0, m * n * d * sizeof(double));
  for (size_t j = 0; j < m; ++j)
    for (size_t i = 0; i < n; ++i) {
      double* out = next + (j * n + i) * d;
      for (size_t l = 0; l < m; ++l) {
        const double coeff = winv[j * m + l];
        const double* p = products + (l * n + i) * d;
        for (size_t c = 0; c < d; ++c) out[c] += coeff * p[c];
      }
    }
}

/* solver.cpp:154-161 */
int jo_guttman_step_fast(size_t m, size_t n, size_t d, const double* delta,
                         const jo_weights* spec, const double* x, double* x_next) {
  double* winv = (double*)malloc(m * m * sizeof(double));
  int rc = shapes_ok(m, n, d, spec);
  if (!rc) rc = script_w_make(spec, m, n, winv);
  if (!rc) {
    double* prod = (double*)malloc(m * n * d * sizeof(double));
    rc = jo_block_guttman_products(m, n, d, delta, spec, x, prod);
    if (!rc) mix_products(m, n, d, prod, winv, x_next);
    free(prod);
  }
  free(winv);
  return rc;
}

/* problem.cpp:34-42 OmnibusProblem::normalized (into a fresh copy) */
static void normalize_copy(size_t m, size_t n, const double* delta, double* out) {
  for (size_t l = 0; l < m; ++l) {
    const double* src = delta + l * n * n;
    double* dst = out + l * n * n;
    double s = 0.0;
    for (size_t i = 0; i < n * n; ++i) s += src[i] * src[i];
    const double norm = sqrt(s);
    for (size_t i = 0; i < n * n; ++i) dst[i] = (norm == 0.0) ? src[i] : src[i] / norm;
  }
}

/* solver.cpp:106-150 run_majorization + :223-236 fjofc_embed (provided init) */
int jo_fjofc_embed(size_t m, size_t n, size_t d, const double* delta, const jo_weights* spec,
                   const double* x0, double eps, size_t max_it, int normalize,
                   double* x_out, double* trace_out, size_t* iterations, int* converged) {
  if (normalize) {
    double* scaled = (double*)malloc(m * n * n * sizeof(double));
    normalize_copy(m, n, delta, scaled);
    int rc = jo_fjofc_embed(m, n, d, scaled, spec, x0, eps, max_it, 0, x_out, trace_out,
                            iterations, converged);
    free(scaled);
    return rc;
  }
  int rc = shapes_ok(m, n, d, spec);
  if (rc) return rc;
  if (!(eps > 0.0)) return fail(1, "SolveOptions: eps must be positive");
  double* winv = (double*)malloc(m * m * sizeof(double));
  rc = script_w_make(spec, m, n, winv);
  if (rc) {
    free(winv);
    return rc;
  }
  const double pairs = jo_stress_pair_count(m, n);
  const size_t sz = m * n * d;
  double* cur = (double*)malloc(sz * sizeof(double));
  double* nxt = (double*)malloc(sz * sizeof(double));
  double* prod = (double*)malloc(sz * sizeof(double));
  memcpy(cur, x0, sz * sizeof(double));
  double stress;
  jo_raw_stress(m, n, d, delta, spec, cur, &stress);
  *iterations = 0;
  *converged = 0;
  if (!isfinite(stress)) {
    rc = fail(2, "embed: non-finite stress at the initial configuration");
    goto done;
  }
  trace_out[0] = stress;
  for (size_t it = 0; it < max_it; ++it) {
    jo_block_guttman_products(m, n, d, delta, spec, cur, prod);
    mix_products(m, n, d, prod, winv, nxt);
    double next_stress;
    jo_raw_stress(m, n, d, delta, spec, nxt, &next_stress);
    if (!isfinite(next_stress)) {
      snprintf(g_err, sizeof g_err, "embed: non-finite stress at iteration %zu", it + 1);
      rc = 2;
      goto done;
    }
    double* t = cur;
    cur = nxt;
    nxt = t;
    trace_out[it + 1] = next_stress;
    ++*iterations;
    const double decrease = (stress - next_stress) / pairs;
    stress = next_stress;
    if (decrease < eps) {
      *converged = 1;
      break;
    }
  }
  memcpy(x_out, cur, sz * sizeof(double));
done:
  free(cur);
  free(nxt);
  free(prod);
  free(winv);
  return rc;
}

/* ---------------- oos.cpp ---------------- */
/* oos.cpp:13-29 */
static int oos_consistent(size_t m, size_t n, size_t d, const double* deltas, double w) {
  if (!(w > 0.0)) return fail(1, "oos: w must be strictly positive");
  if (m == 0 || n == 0 || d == 0) return fail(1, "oos: y must be m x d");
  for (size_t i = 0; i < m * n; ++i)
    if (!(deltas[i] >= 0.0) || !isfinite(deltas[i]))
      return fail(1, "oos: deltas must be finite and nonnegative");
  return 0;
}

/* oos.cpp:43-71 */
int jo_oos_stress(size_t m, size_t n, size_t d, const double* y, const double* x,
                  const double* deltas, double w, double* stress) {
  int rc = oos_consistent(m, n, d, deltas, w);
  if (rc) return rc;
  double fidelity = 0.0;
  for (size_t i = 0; i < m; ++i) {
    const double* yi = y + i * d;
    for (size_t j = 0; j < n; ++j) {
      const double resid = deltas[i * n + j] - row_distance(x + (i * n + j) * d, yi, d);
      fidelity += resid * resid;
    }
  }
  double commensurability = 0.0;
  for (size_t i = 0; i < m; ++i)
    for (size_t j = i + 1; j < m; ++j) {
      double s = 0.0;
      for (size_t c = 0; c < d; ++c) {
        const double diff = y[i * d + c] - y[j * d + c];
        s += diff * diff;
      }
      commensurability += s;
    }
  *stress = fidelity + w * commensurability;
  return 0;
}

/* oos.cpp:73-113: xi_j = sum_k (1 - r_k) X^(j)_k, psi_j = sum_k r_k, then the
 * closed-form corner update y'_j = (xi_j + psi_j y_j)/(n+mw) + w/(n(n+mw)) sum_l (...) */
static void oos_step_core(size_t m, size_t n, size_t d, const double* y, const double* x,
                          const double* deltas, double w, double* next, double* scratch) {
  const double nn = (double)n;
  const double mw = (double)m * w;
  double* xi = scratch;          /* m*d */
  double* psi = scratch + m * d; /* m */
  double* xi_sum = psi + m;      /* d */
  double* psi_y_sum = xi_sum + d;
  memset(scratch, 0, (m * d + m + 2 * d) * sizeof(double));
  for (size_t j = 0; j < m; ++j) {
    const double* yj = y + j * d;
    double* xij = xi + j * d;
    for (size_t k = 0; k < n; ++k) {
      const double* xk = x + (j * n + k) * d;
      const double dist = row_distance(xk, yj, d);
      const double ratio = (dist != 0.0) ? deltas[j * n + k] / dist : 0.0;
      psi[j] += ratio;
      const double coeff = 1.0 - ratio;
      for (size_t c = 0; c < d; ++c) xij[c] += coeff * xk[c];
    }
  }
  for (size_t j = 0; j < m; ++j)
    for (size_t c = 0; c < d; ++c) {
      xi_sum[c] += xi[j * d + c];
      psi_y_sum[c] += psi[j] * y[j * d + c];
    }
  const double direct = 1.0 / (nn + mw);
  const double spread = w / (nn * (nn + mw));
  for (size_t j = 0; j < m; ++j)
    for (size_t c = 0; c < d; ++c)
      next[j * d + c] =
          direct * (xi[j * d + c] + psi[j] * y[j * d + c]) + spread * (xi_sum[c] + psi_y_sum[c]);
}

int jo_oos_step_fast(size_t m, size_t n, size_t d, const double* y, const double* x,
                     const double* deltas, double w, double* y_next) {
  int rc = oos_consistent(m, n, d, deltas, w);
  if (rc) return rc;
  double* scratch = (double*)malloc((m * d + m + 2 * d) * sizeof(double));
  oos_step_core(m, n, d, y, x, deltas, w, y_next, scratch);
  free(scratch);
  return 0;
}

/* oos.cpp:189-198: rms row scale of the frozen configuration, Rng(seed) normals */
int jo_oos_start(size_t m, size_t n, size_t d, const double* x, uint64_t seed, double* y0) {
  double rms = 0.0;
  for (size_t l = 0; l < m; ++l) {
    double s = 0.0;
    for (size_t i = 0; i < n * d; ++i) s += x[l * n * d + i] * x[l * n * d + i];
    const double f = sqrt(s);
    rms += f * f;
  }
  rms = sqrt(rms / (double)(m * n));
  jo_rng r;
  jo_rng_seed(&r, seed);
  const double row_scale = rms / sqrt((double)d);
  for (size_t i = 0; i < m * d; ++i) y0[i] = row_scale * jo_rng_normal(&r);
  return 0;
}

static int oos_loop(size_t m, size_t n, size_t d, const double* x, const double* deltas,
                    double w, const double* y0, double eps, size_t max_it, int fixed,
                    double* y_out, double* trace_out, size_t* iterations, int* converged) {
  const double term_count = (double)(m * n) + 0.5 * (double)(m * (m - 1));
  double* cur = (double*)malloc(m * d * sizeof(double));
  double* nxt = (double*)malloc(m * d * sizeof(double));
  double* scratch = (double*)malloc((m * d + m + 2 * d) * sizeof(double));
  int rc = 0;
  memcpy(cur, y0, m * d * sizeof(double));
  double stress;
  jo_oos_stress(m, n, d, cur, x, deltas, w, &stress);
  *iterations = 0;
  *converged = 0;
  if (!isfinite(stress)) {
    rc = fail(2, "oos_embed: non-finite stress at the initial point");
    goto done;
  }
  trace_out[0] = stress;
  for (size_t it = 0; it < max_it; ++it) {
    oos_step_core(m, n, d, cur, x, deltas, w, nxt, scratch);
    double next_stress;
    jo_oos_stress(m, n, d, nxt, x, deltas, w, &next_stress);
    if (!isfinite(next_stress)) {
      snprintf(g_err, sizeof g_err, "oos_embed: non-finite stress at iteration %zu", it + 1);
      rc = 2;
      goto done;
    }
    double* t = cur;
    cur = nxt;
    nxt = t;
    trace_out[it + 1] = next_stress;
    ++*iterations;
    const double decrease = (stress - next_stress) / term_count;
    stress = next_stress;
    if (!fixed && decrease < eps) {
      *converged = 1;
      break;
    }
  }
done:
  memcpy(y_out, cur, m * d * sizeof(double));
  free(cur);
  free(nxt);
  free(scratch);
  return rc;
}

/* oos.cpp:180-229 */
int jo_oos_embed(size_t m, size_t n, size_t d, const double* x, const double* deltas,
                 double w, double eps, size_t max_it, uint64_t seed, double* y_out,
                 double* trace_out, size_t* iterations, int* converged) {
  if (!(eps > 0.0)) return fail(1, "OosOptions: eps must be positive");
  int rc = oos_consistent(m, n, d, deltas, w);
  if (rc) return rc;
  double* y0 = (double*)malloc(m * d * sizeof(double));
  jo_oos_start(m, n, d, x, seed, y0);
  rc = oos_loop(m, n, d, x, deltas, w, y0, eps, max_it, 0, y_out, trace_out, iterations,
                converged);
  free(y0);
  return rc;
}

int jo_oos_batch(size_t k, size_t m, size_t n, size_t d, const double* x, const double* deltas,
                 double w, const double* y0, double eps, size_t max_it, int fixed_iterations,
                 double* y_out, double* traces, size_t* iterations) {
  if (!(eps > 0.0)) return fail(1, "OosOptions: eps must be positive");
  if (!(w > 0.0)) return fail(1, "oos: w must be strictly positive");
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(| : bad)
  for (size_t p = 0; p < k; ++p) {
    int conv = 0;
    bad |= oos_loop(m, n, d, x, deltas + p * m * n, w, y0 + p * m * d, eps, max_it,
                    fixed_iterations, y_out + p * m * d, traces + p * (max_it + 1),
                    iterations + p, &conv);
  }
  return bad ? 2 : 0;
}
