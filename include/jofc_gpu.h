/*
 * jofc_gpu.h -- C ABI of the B200 fJOFC hot path (libjofc_gpu.so).
 *
 * This is the drop-in boundary under the reference's C++ entry points
 * (proj/include/jofc/{solver,stress,oos}.hpp).  Plain pointers and sizes
 * only.  Every array is dense row-major fp64 unless noted; a configuration
 * is m blocks of n x d (modality-major), exactly Configuration::blocks of
 * the reference (proj/include/jofc/problem.hpp:37-46).  Any pointer argument
 * may point to host memory (pageable or pinned) or to device memory of the
 * context's GPU: copies are resolved through unified addressing.
 *
 * Status codes (mirroring the reference's exceptions):
 *   0 JOFC_OK
 *   1 JOFC_EINVAL    std::invalid_argument (shape / weight / option checks)
 *   2 JOFC_ENUMERIC  jofc::NumericalError  (non-finite stress, bad inverse)
 *   3 JOFC_ECUDA     CUDA runtime failure
 *   4 JOFC_ECOMM     the registered all-reduce hook failed
 * jofc_last_error() returns the message of the calling thread's last failure
 * (the reference's what() text where one exists).
 *
 * Threading: a context is driven by one host thread at a time.  Functions are
 * synchronous on return (results are in the caller's buffers) except where
 * noted.
 */
#ifndef JOFC_GPU_H
#define JOFC_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  JOFC_OK = 0,
  JOFC_EINVAL = 1,
  JOFC_ENUMERIC = 2,
  JOFC_ECUDA = 3,
  JOFC_ECOMM = 4
};

/* WeightSpec (proj/include/jofc/weights.hpp:20-66):
 *   kind 0 uniform(w)              a_l = 1,     w_ll' = w
 *   kind 1 general(W: m x m)       a_l = W_ll,  w_ll' = W_ll'
 *   kind 2 product(within: m, c)   a_l = c p_l, w_ll' = p_l p_l'          */
typedef struct {
  int kind;
  double w;
  const double* general;
  const double* within;
  double scale;
} jofc_weights;

typedef struct jofc_ctx jofc_ctx;

/* Sum-all-reduce hook for multi-GPU sharding: must replace buf[0..count) on
 * every rank by the elementwise sum over ranks, enqueued on `stream` (a
 * cudaStream_t).  Return 0 on success. */
typedef int (*jofc_allreduce_fn)(double* device_buf, size_t count, void* stream, void* user);

const char* jofc_last_error(void);
int jofc_version(void);

/* Context on one CUDA device; owns a non-blocking stream and all buffers. */
int jofc_ctx_create(int device, jofc_ctx** out);
int jofc_ctx_destroy(jofc_ctx* ctx);
/* The cudaStream_t every kernel of this context is launched on. */
void* jofc_ctx_stream(jofc_ctx* ctx);

/* Multi-GPU: this context owns shard `rank` of `world` balanced contiguous
 * ranges of the packed tile stream (call before jofc_set_problem*), and
 * reduces partial products through `fn` each iteration. */
int jofc_set_shard(jofc_ctx* ctx, int rank, int world);
int jofc_set_allreduce(jofc_ctx* ctx, jofc_allreduce_fn fn, void* user);

/* OmnibusProblem upload (proj/include/jofc/problem.hpp:16-34): m dense n x n
 * dissimilarities, delta[l] -> n*n row-major.  Only the upper triangle is
 * read; it is packed into HBM-resident 128x64 blocks and checked finite and
 * nonnegative.  normalize != 0 divides each modality by its Frobenius norm
 * first (OmnibusProblem::normalized, proj/src/problem.cpp:34-42). */
int jofc_set_problem(jofc_ctx* ctx, size_t m, size_t n, const double* const* delta,
                     int normalize);
/* Input preparation on the device: delta_l = euclidean_distance_matrix(F_l)
 * for features F (m x n x p), with the reference's exact per-pair arithmetic
 * (proj/src/distance.cpp:8-29), written straight into the packed layout. */
int jofc_set_problem_features(jofc_ctx* ctx, size_t m, size_t n, size_t p,
                              const double* features);
/* load_dissimilarities (proj/include/jofc/io.hpp:19-23, proj/src/io.cpp:152-215)
 * streamed from files straight into the packed layout, no host n x n copy:
 * one headerless CSV per modality, or a single ".jofc" problem file
 * (proj/src/io.cpp:84-125).  Same validation, order and messages as the
 * reference (symmetry averaged within 1e-9 relative, nonzero diagonals warned
 * on stderr and dropped, negative / non-finite entries rejected naming file
 * and index), then OmnibusProblem's checks.  normalize != 0 divides each
 * modality by its Frobenius norm (device reduction; unsharded contexts). */
int jofc_load_problem_files(jofc_ctx* ctx, size_t count, const char* const* paths,
                            int normalize);
/* Shape (m, n) of the resident problem. */
int jofc_problem_shape(jofc_ctx* ctx, size_t* m, size_t* n);
/* Bytes of packed Delta resident on this context (its shard only). */
size_t jofc_problem_bytes(jofc_ctx* ctx);
/* Number of packed pairs m*n(n-1)/2 (all shards). */
double jofc_problem_pairs(jofc_ctx* ctx);

/* raw_stress (proj/src/stress.cpp:39-74). */
int jofc_raw_stress(jofc_ctx* ctx, const jofc_weights* spec, size_t d, const double* x,
                    double* stress);

/* guttman_step_fast (proj/src/solver.cpp:154-161): one fast transform. */
int jofc_guttman_step(jofc_ctx* ctx, const jofc_weights* spec, size_t d, const double* x,
                      double* x_next);

/* fjofc_embed with InitKind::provided (proj/src/solver.cpp:106-150,223-236).
 * trace_out: max_it+1 doubles, sigma(X_0..X_iterations); iterations /
 * converged as EmbeddingResult.  step_seconds: max_it doubles or NULL; the
 * first `iterations` entries get the solve's mean device time per iteration
 * (a fused pass + epilogue: the transform and the stress of its input, which
 * the fused kernel does not time apart; the reference times fast_step alone,
 * proj/src/solver.cpp:123-127). */
int jofc_fjofc_embed(jofc_ctx* ctx, const jofc_weights* spec, size_t d, const double* x0,
                     double eps, size_t max_it, double* x_out, double* trace_out,
                     size_t* iterations, int* converged, double* step_seconds);

/* Asynchronous form for device-resident use: enqueue the whole solve on the
 * context stream; results are read with jofc_fetch_result after a sync. */
int jofc_fjofc_enqueue(jofc_ctx* ctx, const jofc_weights* spec, size_t d, const double* x0,
                       double eps, size_t max_it);
int jofc_fetch_result(jofc_ctx* ctx, double* x_out, double* trace_out, size_t* iterations,
                      int* converged);
/* Kernel launches issued by this context since creation (evidence counter). */
uint64_t jofc_launch_count(jofc_ctx* ctx);
/* Stress evaluations (= iterations t = 0..T of every solve, counted on the
 * device by the step that writes trace[t]) since the context was created;
 * synchronises the context stream.  bench.py divides these by its timed
 * region instead of assuming every enqueued solve ran max_it iterations. */
int jofc_stress_evaluations(jofc_ctx* ctx, uint64_t* evaluations);
/* Instrumentation: when enabled, CUDA events bracket every pass-kernel launch
 * on the context stream; jofc_profile_read synchronises and returns the summed
 * pass time (ms) and launch count since the last read. */
int jofc_profile(jofc_ctx* ctx, int enable);
int jofc_profile_read(jofc_ctx* ctx, double* pass_ms, uint64_t* pass_launches);
/* How a solve evaluates the fidelity part of sigma(X_t).  AUTO (default):
 * on the one-GPU route with a separate epilogue kernel (n > 1024 and more than
 * 4096 packed blocks, or stream launches), iterations t >= 1 use the SMACOF
 * identity F = sum delta^2 + sum d^2 - 2 tr(X'B(X)X) from the products the
 * transform computes anyway (no per-pair fidelity work in the pass); once a
 * modality's F falls below 1e-5 of A + S + 2|R| the rest of the solve sums
 * (delta - d)^2 pair by pair (trace error < ~5e-11 relative either way).
 * DIRECT: always pair by pair (every route other than the one above is).
 * The environment JOFC_FIDELITY=direct forces DIRECT process-wide. */
#define JOFC_FIDELITY_AUTO 0
#define JOFC_FIDELITY_DIRECT 1
int jofc_set_fidelity_form(jofc_ctx* ctx, int form);

/* Which kernels run an out-of-sample batch (jofc_oos_batch / _step / _stress;
 * same results to rounding).  AUTO (default): the whole batch as ONE
 * persistent launch (each CTA owns whole points for every update) when the
 * batch fills its point slots -- at least Q points per SM and >= 80% of the
 * slots used (Q = 4 at d <= 4, 2 at d <= 8, 1 above): C5's 1000 points on 148
 * SMs; smaller batches (a single point of oos_embed, a few hundred points) use
 * one fused launch per update, which spreads each point over several CTAs.
 * PERSISTENT / PER_UPDATE force one route (the persistent one still falls
 * back when its shared-memory plan does not fit). */
#define JOFC_OOS_AUTO 0
#define JOFC_OOS_PERSISTENT 1
#define JOFC_OOS_PER_UPDATE 2
int jofc_set_oos_route(jofc_ctx* ctx, int route);

/* Multi-GPU: let the caller own the product/exchange buffer (device memory of
 * this context's GPU, >= m*n_pad*d + 1 doubles with n_pad = 64*ceil(n/64)) so
 * that its collective library can reduce it in place.  NULL reverts. */
int jofc_set_exchange_buffer(jofc_ctx* ctx, double* device_buf, size_t capacity);
size_t jofc_exchange_count(jofc_ctx* ctx, size_t d);

/* C-native NCCL exchange (csrc/capi_nccl.cu), the default of a sharded
 * context: per iteration an m-way ncclReduceScatter of the partial products'
 * row chunks (+ a 1-double all-reduce of the fidelity), the W^-1 mix of this
 * rank's chunk only, and an m-way ncclAllGather of the new configuration rows
 * -- all on the context stream, inside the solve's CUDA graph.  SPMD after
 * jofc_set_shard(ctx, rank, world) and the problem: rank 0 makes an id with
 * jofc_nccl_unique_id, the caller broadcasts its JOFC_NCCL_ID_BYTES bytes,
 * every rank calls jofc_nccl_init.  The world must divide the padded object
 * count (any power of two up to 128).  NCCL is the process's libnccl.so.2
 * (dlopen; the system NCCL when none is loaded yet).  Replaces the same
 * data-parallel site as the reference's OpenMP loop over (modality, object),
 * proj/src/solver.cpp:27-49. */
#define JOFC_NCCL_ID_BYTES 128
int jofc_nccl_version(int* version);
int jofc_nccl_unique_id(void* id_out);
int jofc_nccl_init(jofc_ctx* ctx, const void* id, int rank, int world);
int jofc_nccl_release(jofc_ctx* ctx);

/* Peer-memory exchange (NVLink / NVSwitch), the alternative to the all-reduce
 * hook: the exchange of the products (the hook's all-reduce + epilogue) becomes
 * two kernels that read the world's partial products and write the mixed
 * configuration straight through peer pointers
 * (paper_1502_03391_b200/csrc/jofc_peer.cuh).
 * Same SPMD call sequence on every rank, after jofc_set_shard and the problem:
 *   jofc_peer_export(ctx, handle, NULL)     64-byte CUDA IPC handle of this
 *                                           rank's exchange slab
 *   (the caller all-gathers the handles, rank order)
 *   jofc_peer_attach(ctx, rank, world, handles)   handles: world x 64 bytes
 * then the usual solve / stress / step calls; every rank must make the same
 * calls in the same order.  world <= 16.  jofc_peer_attach_pointers takes
 * device pointers of slabs instead of IPC handles (contexts of one process);
 * jofc_peer_detach reverts to the hook.  Re-export after a new problem. */
int jofc_peer_export(jofc_ctx* ctx, void* ipc_handle_out, void** slab_out);
int jofc_peer_attach(jofc_ctx* ctx, int rank, int world, const void* handles);
int jofc_peer_attach_pointers(jofc_ctx* ctx, int rank, int world, void* const* slabs);
int jofc_peer_detach(jofc_ctx* ctx);
/* Device address through which this context reaches rank q's slab (its own
 * for q == rank; the CUDA IPC mapping otherwise; NULL when not attached or
 * attached by pointers).  Diagnostics. */
void* jofc_peer_address(jofc_ctx* ctx, int q);
/* Test driver: one solve over `world` peer-attached contexts of ONE process,
 * launched stage by stage with stream-event ordering so that no kernel ever
 * waits for a flag another context has not raised yet (a single GPU can host
 * all ranks).  Results via jofc_fetch_result on each context. */
int jofc_peer_lockstep_solve(jofc_ctx* const* ctxs, int world, const jofc_weights* spec, size_t d,
                             const double* x0, double eps, size_t max_iterations);

/* Out-of-sample (proj/src/oos.cpp), uniform w only as in the reference.
 * x: frozen configuration m x n x d; deltas: m x n for one point. */
int jofc_oos_stress(jofc_ctx* ctx, size_t m, size_t n, size_t d, const double* y,
                    const double* x, const double* deltas, double w, double* stress);
int jofc_oos_step(jofc_ctx* ctx, size_t m, size_t n, size_t d, const double* y,
                  const double* x, const double* deltas, double w, double* y_next);
/* k independent points in one batched solve: deltas k x m x n, y0 k x m x d.
 * Each point follows oos_embed's loop and stop rule (proj/src/oos.cpp:200-227)
 * unless fixed_iterations != 0 (then exactly max_it steps).  traces:
 * k x (max_it+1) or NULL; iterations: k or NULL. */
int jofc_oos_batch(jofc_ctx* ctx, size_t k, size_t m, size_t n, size_t d, const double* x,
                   const double* deltas, double w, const double* y0, double eps,
                   size_t max_it, int fixed_iterations, double* y_out, double* traces,
                   size_t* iterations);

/* Initialisation on the resident problem (unsharded
 * context): cmds of one modality, or of the modality average when
 * modality < 0 (proj/src/init.cpp:21-42), x_out n x d; and
 * averaged_procrustes_init (proj/src/init.cpp:57-88), x_out m x n x d -- the
 * reference's default InitKind. */
int jofc_cmds(jofc_ctx* ctx, int modality, size_t d, double* x_out);
int jofc_init_averaged_procrustes(jofc_ctx* ctx, size_t d, double* x_out);
/* imputed_omnibus_init (proj/src/init.cpp:90-116): cmds of the m n x m n
 * omnibus matrix (off-diagonal blocks (Delta_i + Delta_j) / 2), split into
 * modality blocks, each re-centred.  Rejects m n > dense_cap like the
 * reference. */
int jofc_init_imputed_cmds(jofc_ctx* ctx, size_t d, size_t dense_cap, double* x_out);
/* symmetric_top_eigenpairs_subspace (proj/include/jofc/linalg.hpp:29-35,
 * proj/src/linalg.cpp:198-271): top-k eigenpairs by algebraic value of the
 * symmetric n x n matrix s (row-major, host or device memory; symmetry is the
 * caller's contract), descending.  n <= 64 or k + 4 >= n: the reference's
 * cyclic Jacobi; else its shifted orthogonal iteration with the S Q products on
 * the device.  values: k; vectors: k x n (eigenvector c at vectors + c n, unit
 * norm, largest-magnitude component positive).  k + 4 <= 14 on the subspace
 * route. */
int jofc_symmetric_top_eigenpairs_subspace(jofc_ctx* ctx, size_t n, const double* s, size_t k,
                                           double* values, double* vectors);

#ifdef __cplusplus
}
#endif
#endif
