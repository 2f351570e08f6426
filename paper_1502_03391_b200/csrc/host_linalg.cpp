// host_linalg.cpp -- see host_linalg.h.
#include "host_linalg.h"

#include <algorithm>
#include <cmath>
#include <numeric>

namespace jofc_gpu {
namespace hostla {

namespace {

// A plane rotation J(p, q) with cos c, sin s and tau = s / (1 + c): applied
// to a pair (g, h) of entries it yields (g - s (h + tau g), h + s (g - tau h)),
// i.e. (c g - s h, s g + c h) with one rounding less in the c * g products.
struct Givens {
  double c, s, tau;
  static Givens from_tangent(double t) {
    Givens r;
    r.c = 1.0 / std::sqrt(t * t + 1.0);
    r.s = t * r.c;
    r.tau = r.s / (1.0 + r.c);
    return r;
  }
  void apply(double& g, double& h) const {
    const double g0 = g, h0 = h;
    g = g0 - s * (h0 + tau * g0);
    h = h0 + s * (g0 - tau * h0);
  }
};

// The smaller-magnitude root of t^2 + 2 theta t - 1 = 0 (rotation angle
// <= pi / 4); theta = 0 picks t = 1.
double small_tangent(double theta) {
  const double sgn = theta < 0.0 ? -1.0 : 1.0;
  return sgn / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
}

double dot_columns(const double* g, std::size_t rows, std::size_t ld, std::size_t p,
                   std::size_t q) {
  double acc = 0.0;
  for (std::size_t r = 0; r < rows; ++r) acc += g[r * ld + p] * g[r * ld + q];
  return acc;
}

// Project column j of q (rows x ld) against columns 0..j-1, twice.
void project_against_earlier(double* q, std::size_t rows, std::size_t ld, std::size_t j) {
  for (int round = 0; round < 2; ++round)
    for (std::size_t i = 0; i < j; ++i) {
      const double h = dot_columns(q, rows, ld, i, j);
      for (std::size_t r = 0; r < rows; ++r) q[r * ld + j] -= h * q[r * ld + i];
    }
}

}  // namespace

bool jacobi_eigh(const double* a_in, std::size_t n, double* w, double* v, int max_sweeps,
                 double rel_tol) {
  std::vector<double> a(a_in, a_in + n * n);
  std::fill(v, v + n * n, 0.0);
  for (std::size_t i = 0; i < n; ++i) v[i * n + i] = 1.0;
  double fro2 = 0.0;
  for (double x : a) fro2 += x * x;
  const double target = rel_tol * std::sqrt(fro2);
  auto off_diagonal = [&] {
    double upper = 0.0;
    for (std::size_t i = 0; i < n; ++i)
      for (std::size_t j = i + 1; j < n; ++j) upper += a[i * n + j] * a[i * n + j];
    return std::sqrt(2.0 * upper);
  };
  bool converged = false;
  for (int sweep = 0;; ++sweep) {
    if (off_diagonal() <= target) {
      converged = true;
      break;
    }
    if (sweep == max_sweeps) break;
    for (std::size_t p = 0; p + 1 < n; ++p)
      for (std::size_t q = p + 1; q < n; ++q) {
        double& apq = a[p * n + q];
        if (apq == 0.0) continue;
        const double t = small_tangent((a[q * n + q] - a[p * n + p]) / (2.0 * apq));
        const Givens rot = Givens::from_tangent(t);
        a[p * n + p] -= t * apq;
        a[q * n + q] += t * apq;
        apq = 0.0;
        a[q * n + p] = 0.0;
        for (std::size_t r = 0; r < n; ++r) {
          if (r != p && r != q) {
            rot.apply(a[r * n + p], a[r * n + q]);
            a[p * n + r] = a[r * n + p];
            a[q * n + r] = a[r * n + q];
          }
          rot.apply(v[r * n + p], v[r * n + q]);
        }
      }
  }
  for (std::size_t i = 0; i < n; ++i) w[i] = a[i * n + i];
  return converged;
}

std::vector<std::size_t> descending_order(const double* w, std::size_t n) {
  std::vector<std::size_t> idx(n);
  std::iota(idx.begin(), idx.end(), std::size_t{0});
  std::stable_sort(idx.begin(), idx.end(), [w](std::size_t x, std::size_t y) { return w[x] > w[y]; });
  return idx;
}

void orient(double* x, std::size_t n, std::size_t stride) {
  std::size_t lead = 0;
  for (std::size_t i = 1; i < n; ++i)
    if (std::fabs(x[i * stride]) > std::fabs(x[lead * stride])) lead = i;
  if (n && x[lead * stride] < 0.0)
    for (std::size_t i = 0; i < n; ++i) x[i * stride] = -x[i * stride];
}

void svd_jacobi(const double* a, std::size_t n, double* u, double* s, double* v) {
  std::vector<double> g(a, a + n * n);  // columns converge to u_j s_j
  std::vector<double> rv(n * n, 0.0);
  for (std::size_t i = 0; i < n; ++i) rv[i * n + i] = 1.0;
  for (int sweep = 0; sweep < 64; ++sweep) {
    bool any = false;
    for (std::size_t p = 0; p + 1 < n; ++p)
      for (std::size_t q = p + 1; q < n; ++q) {
        const double alpha = dot_columns(g.data(), n, n, p, p);
        const double beta = dot_columns(g.data(), n, n, q, q);
        const double gamma = dot_columns(g.data(), n, n, p, q);
        if (gamma == 0.0 || std::fabs(gamma) <= 1e-14 * std::sqrt(alpha * beta)) continue;
        any = true;
        const Givens rot = Givens::from_tangent(small_tangent((beta - alpha) / (2.0 * gamma)));
        for (std::size_t r = 0; r < n; ++r) {
          rot.apply(g[r * n + p], g[r * n + q]);
          rot.apply(rv[r * n + p], rv[r * n + q]);
        }
      }
    if (!any) break;
  }
  std::vector<double> norm(n);
  for (std::size_t j = 0; j < n; ++j) norm[j] = std::sqrt(dot_columns(g.data(), n, n, j, j));
  const std::vector<std::size_t> order = descending_order(norm.data(), n);
  const double keep = 1e-13 * std::max(1.0, n ? norm[order[0]] : 0.0);
  std::fill(u, u + n * n, 0.0);
  std::size_t have = 0;  // leading columns of u taken from g
  for (std::size_t j = 0; j < n; ++j) {
    const std::size_t src = order[j];
    s[j] = norm[src];
    for (std::size_t r = 0; r < n; ++r) v[r * n + j] = rv[r * n + src];
    if (norm[src] > keep) {
      for (std::size_t r = 0; r < n; ++r) u[r * n + j] = g[r * n + src] / norm[src];
      have = j + 1;
    }
  }
  // complete u: e_0, e_1, ... orthogonalised (once) against the columns so far
  std::vector<double> cand(n);
  for (std::size_t j = have; j < n; ++j)
    for (std::size_t e = 0; e < n; ++e) {
      std::fill(cand.begin(), cand.end(), 0.0);
      cand[e] = 1.0;
      for (std::size_t i = 0; i < j; ++i) {
        double h = 0.0;
        for (std::size_t r = 0; r < n; ++r) h += u[r * n + i] * cand[r];
        for (std::size_t r = 0; r < n; ++r) cand[r] -= h * u[r * n + i];
      }
      double len = 0.0;
      for (double x : cand) len += x * x;
      len = std::sqrt(len);
      if (len > 1e-6) {
        for (std::size_t r = 0; r < n; ++r) u[r * n + j] = cand[r] / len;
        break;
      }
    }
}

void orthonormalize_columns(double* q, std::size_t rows, std::size_t cols) {
  for (std::size_t j = 0; j < cols; ++j) {
    project_against_earlier(q, rows, cols, j);
    double len = std::sqrt(dot_columns(q, rows, cols, j, j));
    for (std::size_t e = 0; len < 1e-150 && e < rows; ++e) {
      for (std::size_t r = 0; r < rows; ++r) q[r * cols + j] = (r == e) ? 1.0 : 0.0;
      project_against_earlier(q, rows, cols, j);
      const double l2 = std::sqrt(dot_columns(q, rows, cols, j, j));
      if (l2 > 1e-8) len = l2;
    }
    for (std::size_t r = 0; r < rows; ++r) q[r * cols + j] /= len;
  }
}

bool gauss_jordan_inverse(const double* a, std::size_t n, double* inv, double pivot_rel) {
  // augmented rows [a_i | e_i]: every row operation acts on both halves
  const std::size_t w = 2 * n;
  std::vector<double> aug(n * w, 0.0);
  double amax = 0.0;
  for (std::size_t i = 0; i < n; ++i) {
    for (std::size_t j = 0; j < n; ++j) {
      aug[i * w + j] = a[i * n + j];
      amax = std::max(amax, std::fabs(a[i * n + j]));
    }
    aug[i * w + n + i] = 1.0;
  }
  const double floor_v = pivot_rel * std::max(1.0, amax);
  for (std::size_t k = 0; k < n; ++k) {
    std::size_t best = k;  // first row with the largest |entry| in column k
    for (std::size_t r = k + 1; r < n; ++r)
      if (std::fabs(aug[r * w + k]) > std::fabs(aug[best * w + k])) best = r;
    if (std::fabs(aug[best * w + k]) < floor_v) return false;
    if (best != k) std::swap_ranges(aug.begin() + best * w, aug.begin() + (best + 1) * w,
                                    aug.begin() + k * w);
    double* pivot_row = aug.data() + k * w;
    const double pv = pivot_row[k];
    for (std::size_t j = 0; j < w; ++j) pivot_row[j] /= pv;
    for (std::size_t r = 0; r < n; ++r) {
      const double f = aug[r * w + k];
      if (r == k || f == 0.0) continue;
      double* row = aug.data() + r * w;
      for (std::size_t j = 0; j < w; ++j) row[j] -= f * pivot_row[j];
    }
  }
  for (std::size_t i = 0; i < n; ++i)
    std::copy(aug.begin() + i * w + n, aug.begin() + (i + 1) * w, inv + i * n);
  return true;
}

}  // namespace hostla
}  // namespace jofc_gpu
