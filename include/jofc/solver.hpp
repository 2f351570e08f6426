// Drop-in for the fast entry points of proj/include/jofc/solver.hpp
// (GPU-backed; the dense Algorithm-1 oracle is not part of this build).
#pragma once

#include <vector>

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

// Multi-GPU, one process (or thread) per GPU: makes this thread's context
// rank `rank` of a `world`-rank group.  The packed Delta of the next problem
// is sharded (each rank streams 1/world of it) and every Guttman iteration
// exchanges through NCCL inside the solve's CUDA graph: reduce-scatter of the
// products, own-row W^-1 mix, all-gather of the configuration rows.  Rank 0
// makes the id with nccl_unique_id(); the caller hands the same bytes to every
// rank (its own transport), then every rank calls set_shard and makes the same
// fjofc_embed / raw_stress / guttman_step_fast calls (InitKind::provided).
// set_shard(0, 1, {}) returns to the unsharded context.  Replaces the
// reference's OpenMP loop over (modality, object), proj/src/solver.cpp:27-49.
std::vector<unsigned char> nccl_unique_id();
void set_shard(int rank, int world, const std::vector<unsigned char>& nccl_id);

}  // namespace jofc
