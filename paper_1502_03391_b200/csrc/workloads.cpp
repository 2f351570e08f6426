// workloads.cpp -- seeded synthetic inputs for the BASELINE.json configs.
// See include/jofc_workloads.h and DESIGN.md "Synthetic workloads".
#include "jofc_workloads.h"

#include "jofc_rng.h"

#include <cmath>
#include <cstring>
#include <random>
#include <vector>

namespace {

using Rng = jofc_gpu::RefRng;

// Gram-Schmidt on a Gaussian draw, column by column.
std::vector<double> random_orthogonal(Rng& rng, size_t q) {
  std::vector<double> a(q * q);
  for (double& v : a) v = rng.normal();
  for (size_t j = 0; j < q; ++j) {
    for (size_t i = 0; i < j; ++i) {
      double dot = 0.0;
      for (size_t r = 0; r < q; ++r) dot += a[r * q + i] * a[r * q + j];
      for (size_t r = 0; r < q; ++r) a[r * q + j] -= dot * a[r * q + i];
    }
    double nrm = 0.0;
    for (size_t r = 0; r < q; ++r) nrm += a[r * q + j] * a[r * q + j];
    nrm = std::sqrt(nrm);
    for (size_t r = 0; r < q; ++r) a[r * q + j] /= nrm;
  }
  return a;
}

}  // namespace

extern "C" {

int jofc_wl_shape(int cfg, jofc_workload_shape* o) {
  std::memset(o, 0, sizeof(*o));
  switch (cfg) {
    case 1: *o = {2, 500, 2, 2, 100, 0.5, 1, 0}; return 0;
    case 2: *o = {3, 2000, 3, 4, 200, 0.9, 0, 0}; return 0;
    case 3: *o = {2, 20000, 5, 10, 100, 0.5, 0, 0}; return 0;
    case 4: *o = {10, 10000, 3, 3, 100, 0.99, 0, 0}; return 0;
    case 5: *o = {2, 5000, 3, 3, 100, 0.5, 0, 1000}; return 0;
  }
  return 1;
}

int jofc_wl_features(int cfg, uint64_t seed, size_t N, double* out) {
  jofc_workload_shape s;
  if (jofc_wl_shape(cfg, &s)) return 1;
  const size_t m = s.m, p = s.p;
  Rng rng(seed);
  std::vector<double> z;
  switch (cfg) {
    case 1: {  // Z ~ N(0, I2); X_l = Z + 0.1 N
      z.resize(N * p);
      for (double& v : z) v = rng.normal();
      for (size_t l = 0; l < m; ++l)
        for (size_t i = 0; i < N * p; ++i) out[l * N * p + i] = z[i] + 0.1 * rng.normal();
      return 0;
    }
    case 2: {  // Dirichlet(1,1,1,1) latent; X_l = Z Q_l + 0.05 N
      z.resize(N * p);
      for (size_t i = 0; i < N; ++i) {
        double sum = 0.0;
        for (size_t k = 0; k < p; ++k) {
          const double e = -std::log(1.0 - rng.uniform());
          z[i * p + k] = e;
          sum += e;
        }
        for (size_t k = 0; k < p; ++k) z[i * p + k] /= sum;
      }
      for (size_t l = 0; l < m; ++l) {
        const std::vector<double> q = random_orthogonal(rng, p);
        double* X = out + l * N * p;
        for (size_t i = 0; i < N; ++i)
          for (size_t c = 0; c < p; ++c) {
            double acc = 0.0;
            for (size_t k = 0; k < p; ++k) acc += z[i * p + k] * q[k * p + c];
            X[i * p + c] = acc;
          }
        for (size_t i = 0; i < N * p; ++i) X[i] += 0.05 * rng.normal();
      }
      return 0;
    }
    case 3: {  // Z ~ N(0, I10); X_1 = Z; X_2 = Z A + 0.2 N, A_ij ~ N(0, 1/10)
      z.resize(N * p);
      for (double& v : z) v = rng.normal();
      std::memcpy(out, z.data(), N * p * sizeof(double));
      std::vector<double> A(p * p);
      const double sa = 1.0 / std::sqrt(static_cast<double>(p));
      for (double& v : A) v = sa * rng.normal();
      double* X = out + N * p;
      for (size_t i = 0; i < N; ++i)
        for (size_t c = 0; c < p; ++c) {
          double acc = 0.0;
          for (size_t k = 0; k < p; ++k) acc += z[i * p + k] * A[k * p + c];
          X[i * p + c] = acc;
        }
      for (size_t i = 0; i < N * p; ++i) X[i] += 0.2 * rng.normal();
      return 0;
    }
    case 4: {  // Z ~ U[0,1)^3; X_l = s_l Z + 0.05 N, s_l ~ U[0.5, 2]
      z.resize(N * p);
      for (double& v : z) v = rng.uniform();
      for (size_t l = 0; l < m; ++l) {
        const double sl = rng.uniform(0.5, 2.0);
        double* X = out + l * N * p;
        for (size_t i = 0; i < N * p; ++i) X[i] = sl * z[i] + 0.05 * rng.normal();
      }
      return 0;
    }
    case 5: {  // Z ~ N(0, I3) for n + k objects; X_l = Z + 0.1 N
      z.resize(N * p);
      for (double& v : z) v = rng.normal();
      for (size_t l = 0; l < m; ++l)
        for (size_t i = 0; i < N * p; ++i) out[l * N * p + i] = z[i] + 0.1 * rng.normal();
      return 0;
    }
  }
  return 1;
}

void jofc_wl_normals(uint64_t seed, size_t count, double scale, double* out) {
  Rng rng(seed);
  for (size_t i = 0; i < count; ++i) out[i] = scale * rng.normal();
}

void jofc_wl_distance_matrix(size_t n, size_t p, const double* x, double* out) {
#pragma omp parallel for schedule(dynamic, 16)
  for (long long ii = 0; ii < static_cast<long long>(n); ++ii) {
    const size_t i = static_cast<size_t>(ii);
    out[i * n + i] = 0.0;
    const double* xi = x + i * p;
    for (size_t j = i + 1; j < n; ++j) {
      const double* xj = x + j * p;
      double s = 0.0;
      for (size_t k = 0; k < p; ++k) {
        const double diff = xi[k] - xj[k];
        s += diff * diff;
      }
      const double dist = std::sqrt(s);
      out[i * n + j] = dist;
      out[j * n + i] = dist;
    }
  }
}

void jofc_wl_oos_deltas(size_t m, size_t n, size_t k, size_t p, const double* feats,
                        double* out) {
  const size_t N = n + k;
#pragma omp parallel for schedule(static)
  for (long long qq = 0; qq < static_cast<long long>(k); ++qq) {
    const size_t q = static_cast<size_t>(qq);
    for (size_t l = 0; l < m; ++l) {
      const double* F = feats + l * N * p;
      const double* y = F + (n + q) * p;
      double* o = out + (q * m + l) * n;
      for (size_t j = 0; j < n; ++j) {
        double s = 0.0;
        for (size_t c = 0; c < p; ++c) {
          const double diff = F[j * p + c] - y[c];
          s += diff * diff;
        }
        o[j] = std::sqrt(s);
      }
    }
  }
}

void jofc_wl_oos_start(size_t m, size_t n, size_t d, const double* x, uint64_t seed,
                       double* y0) {
  double rms = 0.0;
  for (size_t l = 0; l < m; ++l) {
    double s = 0.0;
    for (size_t i = 0; i < n * d; ++i) s += x[l * n * d + i] * x[l * n * d + i];
    const double f = std::sqrt(s);
    rms += f * f;
  }
  rms = std::sqrt(rms / static_cast<double>(m * n));
  Rng rng(seed);
  const double scale = rms / std::sqrt(static_cast<double>(d));
  for (size_t i = 0; i < m * d; ++i) y0[i] = scale * rng.normal();
}

}  // extern "C"
