// Drop-in for proj/include/jofc/stress.hpp (GPU-backed).
#pragma once

#include <vector>

#include "jofc/problem.hpp"
#include "jofc/weights.hpp"

namespace jofc {

// Fidelity + commensurability raw stress; `parallel` is accepted for source
// compatibility (the GPU path is always parallel).
double raw_stress(const Configuration& config, const OmnibusProblem& problem,
                  const WeightSpec& spec, bool parallel = false);

// C(nm, 2), the normalizer of the stress trace.
double stress_pair_count(std::size_t m, std::size_t n);

void require_consistent_shapes(const Configuration& config, const OmnibusProblem& problem,
                               const WeightSpec& spec);

}  // namespace jofc
