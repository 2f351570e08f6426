// Drop-in for the fast entry points of proj/include/jofc/solver.hpp
// (GPU-backed; the dense Algorithm-1 oracle is not part of this build).
#pragma once

#include "jofc/problem.hpp"
#include "jofc/stress.hpp"
#include "jofc/weights.hpp"

namespace jofc {

Configuration guttman_step_fast(const Configuration& config, const OmnibusProblem& problem,
                                const WeightSpec& spec, bool parallel = false);

// Every InitKind: provided, averaged_procrustes (the default) and imputed_cmds,
// the latter two computed on the GPU from the resident Delta.
EmbeddingResult fjofc_embed(const OmnibusProblem& problem, const WeightSpec& spec,
                            const SolveOptions& options);

// Selects the CUDA device used by the calls above in this thread (default 0).
void set_device(int device);

}  // namespace jofc
