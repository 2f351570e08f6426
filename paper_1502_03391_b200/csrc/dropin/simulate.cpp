// Synthetic settings of the drop-in API (include/jofc/simulate.hpp), the
// paper's section 4.1 generator as proj/src/simulate.cpp:37-66 draws it:
// one Rng stream -- latent N(5,1) entries row-major, then per modality the
// U(-a, a) jitter entries (a = range / 50), the anomalous modality last with
// its shifted rows drawn before its jitter.
#include "jofc/simulate.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>

#include "jofc/distance.hpp"
#include "jofc/rng.hpp"

namespace jofc {

std::vector<DenseMatrix> simulate_features(std::size_t n, std::size_t m, std::size_t n_anom,
                                           std::size_t dim, std::uint64_t seed) {
  if (n < 2 || m < 1 || dim < 1)
    throw std::invalid_argument("generate: n >= 2, m >= 1, dim >= 1 required");
  if (n_anom > n) throw std::invalid_argument("generate: n_anom exceeds n");
  Rng rng(seed);
  DenseMatrix latent(n, dim);
  for (std::size_t i = 0; i < latent.size(); ++i) latent.data()[i] = 5.0 + 1.0 * rng.normal();
  const auto [lo, hi] = std::minmax_element(latent.data(), latent.data() + latent.size());
  const double amp = (*hi - *lo) / 50.0;
  auto jitter = [&](DenseMatrix y) {
    for (std::size_t i = 0; i < y.size(); ++i) y.data()[i] += rng.uniform(-amp, amp);
    return y;
  };
  std::vector<DenseMatrix> out;
  const std::size_t plain = n_anom > 0 ? m - 1 : m;
  for (std::size_t l = 0; l < plain; ++l) out.push_back(jitter(latent));
  if (n_anom > 0) {
    DenseMatrix shifted = latent;
    for (std::size_t r = 0; r < n_anom; ++r)
      for (std::size_t c = 0; c < dim; ++c) shifted(r, c) = 8.0 + std::sqrt(2.0) * rng.normal();
    out.push_back(jitter(shifted));
  }
  return out;
}

namespace {

SimulatedProblem from_features(const std::vector<DenseMatrix>& feats, std::size_t n,
                               std::size_t n_anom) {
  SimulatedProblem sim;
  for (const DenseMatrix& f : feats) sim.modalities.push_back(euclidean_distance_matrix(f));
  sim.labels.resize(n);
  for (std::size_t i = 0; i < n; ++i) sim.labels[i] = static_cast<int>(i);
  for (std::size_t r = 0; r < n_anom; ++r) sim.anomalies.push_back(r);
  return sim;
}

}  // namespace

SimulatedProblem generate_matched(std::size_t n, std::size_t m, std::size_t dim,
                                  std::uint64_t seed) {
  return from_features(simulate_features(n, m, 0, dim, seed), n, 0);
}

SimulatedProblem generate_anomaly(std::size_t n, std::size_t m, std::size_t n_anom,
                                  std::size_t dim, std::uint64_t seed) {
  if (m < 1) throw std::invalid_argument("generate_anomaly: m >= 1 required");
  return from_features(simulate_features(n, m, n_anom, dim, seed), n, n_anom);
}

}  // namespace jofc
