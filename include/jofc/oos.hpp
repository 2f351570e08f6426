// Drop-in for the fast entry points of proj/include/jofc/oos.hpp (GPU-backed).
#pragma once

#include <cstdint>
#include <vector>

#include "jofc/problem.hpp"

namespace jofc {

struct OosDissimilarity {
  std::vector<std::vector<double>> deltas;  // m vectors of length n

  std::size_t modality_count() const { return deltas.size(); }
  std::size_t object_count() const { return deltas.empty() ? 0 : deltas.front().size(); }
};

struct OosResult {
  DenseMatrix y;
  std::vector<double> stress_trace;
  std::size_t iterations = 0;
  Termination terminated = Termination::converged;
};

struct OosOptions {
  double eps = 1e-6;
  std::size_t max_iterations = 1000;
};

double oos_stress(const DenseMatrix& y, const Configuration& x, const OosDissimilarity& deltas,
                  double w);
DenseMatrix oos_step_fast(const DenseMatrix& y, const Configuration& x,
                          const OosDissimilarity& deltas, double w);
OosResult oos_embed(const Configuration& x, const OosDissimilarity& deltas, double w,
                    const OosOptions& options, std::uint64_t seed);

// Batched form (new): k points, one GPU solve; results in input order.
std::vector<OosResult> oos_embed_batch(const Configuration& x,
                                       const std::vector<OosDissimilarity>& points, double w,
                                       const OosOptions& options,
                                       const std::vector<std::uint64_t>& seeds);

}  // namespace jofc
