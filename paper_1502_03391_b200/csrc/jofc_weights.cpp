// jofc_weights.cpp -- see jofc_weights.h.
#include "jofc_weights.h"

#include "host_linalg.h"

#include <algorithm>
#include <cmath>

namespace jofc_gpu {

namespace {

bool positive(double v) { return v > 0.0 && std::isfinite(v); }

double within_of(const jofc_weights* s, std::size_t m, std::size_t i) {
  switch (s->kind) {
    case 1: return s->general[i * m + i];
    case 2: return s->scale * s->within[i];
    default: return 1.0;
  }
}

double cross_of(const jofc_weights* s, std::size_t m, std::size_t i, std::size_t j) {
  switch (s->kind) {
    case 1: return s->general[i * m + j];
    case 2: return s->within[i] * s->within[j];
    default: return s->w;
  }
}

}  // namespace

int validate_weights(const jofc_weights* s, std::size_t m, std::string* msg) {
  if (!s) {
    *msg = "WeightSpec: null";
    return JOFC_EINVAL;
  }
  if (m == 0) {
    *msg = "WeightSpec: m must be positive";
    return JOFC_EINVAL;
  }
  switch (s->kind) {
    case 0:
      if (!positive(s->w)) {
        *msg = "WeightSpec: w must be strictly positive";
        return JOFC_EINVAL;
      }
      return JOFC_OK;
    case 1:
      if (!s->general) {
        *msg = "WeightSpec: general weight matrix size mismatch";
        return JOFC_EINVAL;
      }
      for (std::size_t i = 0; i < m; ++i)
        for (std::size_t j = i + 1; j < m; ++j)
          if (s->general[i * m + j] != s->general[j * m + i]) {
            *msg = "WeightSpec: general weight matrix must be symmetric";
            return JOFC_EINVAL;
          }
      for (std::size_t i = 0; i < m * m; ++i)
        if (!positive(s->general[i])) {
          *msg = "WeightSpec: w_ij must be strictly positive";
          return JOFC_EINVAL;
        }
      return JOFC_OK;
    case 2:
      if (!s->within) {
        *msg = "WeightSpec: product weight count mismatch";
        return JOFC_EINVAL;
      }
      for (std::size_t i = 0; i < m; ++i)
        if (!positive(s->within[i])) {
          *msg = "WeightSpec: w_ii must be strictly positive";
          return JOFC_EINVAL;
        }
      if (!positive(s->scale)) {
        *msg = "WeightSpec: c must be strictly positive";
        return JOFC_EINVAL;
      }
      return JOFC_OK;
  }
  *msg = "WeightSpec: unknown kind";
  return JOFC_EINVAL;
}

int build_weights(const jofc_weights* s, std::size_t m, std::size_t n, HostWeights* out,
                  std::string* msg) {
  int rc = validate_weights(s, m, msg);
  if (rc) return rc;
  if (n < 2) {
    *msg = "script_w: n must be at least 2";
    return JOFC_EINVAL;
  }
  const double nn = static_cast<double>(n);
  out->within.assign(m, 0.0);
  out->cross.assign(m * m, 0.0);
  std::vector<double> W(m * m, 0.0);
  for (std::size_t i = 0; i < m; ++i) {
    out->within[i] = within_of(s, m, i);
    double diag = nn * out->within[i];
    for (std::size_t j = 0; j < m; ++j) {
      if (j == i) continue;
      const double cw = cross_of(s, m, i, j);
      out->cross[i * m + j] = cw;
      diag += cw;
      W[i * m + j] = -cw;
    }
    W[i * m + i] = diag;
  }
  auto& inv = out->winv;
  inv.assign(m * m, 0.0);
  if (s->kind == 0) {
    const double w = s->w;
    const double denom = nn * (nn + static_cast<double>(m) * w);
    const double diag = (nn + w) / denom, off = w / denom;
    for (std::size_t i = 0; i < m; ++i)
      for (std::size_t j = 0; j < m; ++j) inv[i * m + j] = (i == j) ? diag : off;
  } else if (s->kind == 2) {
    double sum = 0.0;
    for (std::size_t i = 0; i < m; ++i) sum += s->within[i];
    const double cn = s->scale * nn;
    const double off = 1.0 / (cn * (cn + sum));
    for (std::size_t i = 0; i < m; ++i)
      for (std::size_t j = 0; j < m; ++j)
        inv[i * m + j] = (i == j) ? 1.0 / (s->within[i] * (cn + sum)) + off : off;
  } else if (!hostla::gauss_jordan_inverse(W.data(), m, inv.data())) {
    *msg = "invert_small: singular matrix";
    return JOFC_ENUMERIC;
  }
  double wmax = 0.0, gap = 0.0;
  for (double v : W) wmax = std::max(wmax, std::fabs(v));
  for (std::size_t i = 0; i < m; ++i)
    for (std::size_t j = 0; j < m; ++j) {
      double acc = 0.0;
      for (std::size_t k = 0; k < m; ++k) acc += W[i * m + k] * inv[k * m + j];
      gap = std::max(gap, std::fabs(acc - (i == j ? 1.0 : 0.0)));
    }
  if (gap > 1e-12 * std::max(1.0, wmax)) {
    *msg = "ScriptW: inverse check failed";
    return JOFC_ENUMERIC;
  }
  out->coef.assign(m * m, 0.0);
  for (std::size_t j = 0; j < m; ++j)
    for (std::size_t l = 0; l < m; ++l) out->coef[j * m + l] = inv[j * m + l] * out->within[l];
  return JOFC_OK;
}

}  // namespace jofc_gpu
