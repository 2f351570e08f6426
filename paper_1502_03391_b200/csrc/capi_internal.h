// capi_internal.h -- what the translation units of libjofc_gpu.so share:
// the context struct, error plumbing, device buffers and the small helpers
// (jofc_capi.cu: context, solve, stress, step, out-of-sample; capi_init.cu:
// the initialisers and the eigen-solver; capi_ingest.cu: file ingest).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "jofc_gpu.h"
#include "jofc_kernels.cuh"
#include "jofc_oos.cuh"
#include "jofc_peer.cuh"

namespace jofc_gpu {
namespace capi {

// Largest n whose epilogue the pass kernel's last CTA runs itself (one GPU).
constexpr long long kFuseEpilogueMaxN = 1024;
// Synchronous solves stop enqueuing iterations once the device says done,
// checked every kStopChunk iterations (at most ~2 chunks of no-op launches).
constexpr size_t kStopChunk = 32;
// Largest packed block stream (all modalities) solved by the single-launch
// persistent kernel on one GPU.
constexpr long long kPersistentMaxBlocks = 4096;

inline thread_local std::string g_error;

// NVTX range over one C-ABI call (header-only NVTX v3: no link dependency;
// free when no tool is attached).  The per-iteration device work is visible
// to a profiler as kernels; these mark the API calls around them.
struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
  NvtxScope(const NvtxScope&) = delete;
  NvtxScope& operator=(const NvtxScope&) = delete;
};

inline int set_error(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_error = buf;
  return code;
}

#define JOFC_CUDA(call)                                                                 \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return set_error(JOFC_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                       __FILE__, __LINE__);                                             \
  } while (0)

#define JOFC_TRY(call)     \
  do {                     \
    const int rc_ = (call); \
    if (rc_) return rc_;   \
  } while (0)

constexpr int kMaxD = 10;

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device setting: set it
// once per (kernel, device) of the process.
template <class K>
cudaError_t ensure_smem_attr(K kernel, int bytes, int device) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  const auto key = std::make_pair(reinterpret_cast<const void*>(kernel), device);
  std::lock_guard<std::mutex> lock(mu);
  if (done.count(key)) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             bytes);
  if (e == cudaSuccess) done.insert(key);
  return e;
}

// FN<D>(args) for the runtime dimension d (1..kMaxD)
#define JOFC_DISPATCH_D(d, FN, ...)         \
  switch (d) {                              \
    case 1: return FN<1>(__VA_ARGS__);      \
    case 2: return FN<2>(__VA_ARGS__);      \
    case 3: return FN<3>(__VA_ARGS__);      \
    case 4: return FN<4>(__VA_ARGS__);      \
    case 5: return FN<5>(__VA_ARGS__);      \
    case 6: return FN<6>(__VA_ARGS__);      \
    case 7: return FN<7>(__VA_ARGS__);      \
    case 8: return FN<8>(__VA_ARGS__);      \
    case 9: return FN<9>(__VA_ARGS__);      \
    case 10: return FN<10>(__VA_ARGS__);    \
    default:                                \
      return set_error(JOFC_EINVAL, "dim %zu unsupported (1..10)", static_cast<size_t>(d)); \
  }

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  cudaError_t ensure(size_t count) {
    if (count <= n && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T));
    if (e == cudaSuccess) n = count;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

// Double-buffered staging of streaming ingest (kept across loads): pinned
// host panels, their copy-done events, and the device panels.
struct IngestPanels {
  double* host[2] = {nullptr, nullptr};
  size_t cap = 0;  // doubles per panel
  cudaEvent_t copied[2] = {nullptr, nullptr};
  DevBuf<double> stage[2];
  void release() {
    for (int k = 0; k < 2; ++k) {
      if (host[k]) cudaFreeHost(host[k]);
      if (copied[k]) cudaEventDestroy(copied[k]);
      host[k] = nullptr;
      copied[k] = nullptr;
      stage[k].release();
    }
    cap = 0;
  }
  cudaError_t ensure(size_t doubles) {
    if (doubles <= cap) return cudaSuccess;
    release();
    for (int k = 0; k < 2; ++k) {
      cudaError_t e = cudaMallocHost(&host[k], doubles * sizeof(double));
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&copied[k], cudaEventDisableTiming);
      if (e == cudaSuccess) e = stage[k].ensure(doubles);
      if (e != cudaSuccess) {
        release();
        return e;
      }
    }
    cap = doubles;
    return cudaSuccess;
  }
};

// Peer-memory exchange state of a sharded context (capi_peer.cu).
struct PeerState {
  bool active = false;
  int rank = 0, world = 1;
  double* slab = nullptr;  // own slab (cudaMalloc: IPC-exportable)
  size_t slab_doubles = 0;
  long long p_off[2] = {0, 0}, x_off[2] = {0, 0};
  long long p_len = 0, com_off = 0, flag1_off = 0, flag2_off = 0;
  std::vector<long long> key;   // (m, n_pad) the slab is laid out for
  std::vector<void*> opened;    // IPC-mapped peer slabs
  DevBuf<double*> ptrs;         // device array of the world's slab bases
  DevBuf<double> com_part;      // per mix CTA
  unsigned epoch = 0;           // solves started (flags carry it)
  int phase = 0;                // P region of the next solve's iteration 0
  bool pending = false;         // a solve was enqueued and not yet finished
  long long row_lo = 0, row_hi = 0;
  int rows_cta = 32, mix_grid = 1;
};

}  // namespace capi
}  // namespace jofc_gpu

// The opaque handle of include/jofc_gpu.h.
struct jofc_ctx {
  template <class T>
  using DevBuf = jofc_gpu::capi::DevBuf<T>;
  using IngestPanels = jofc_gpu::capi::IngestPanels;
  using Layout = jofc_gpu::Layout;
  using Control = jofc_gpu::Control;
  using OosPoint = jofc_gpu::OosPoint;
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  uint64_t launches = 0;
  // sharding / exchange
  int rank = 0, world = 1;
  jofc_allreduce_fn allreduce = nullptr;
  void* allreduce_user = nullptr;
  // problem
  bool has_problem = false;
  Layout lay;
  DevBuf<double> delta;
  // A_l (sum of squared stored entries per modality, this shard) of the
  // identity-form fidelity; computed by delta_sumsq() whenever Delta changes
  DevBuf<double> sumsq, sumsq_part;
  DevBuf<double> rho_part;  // epilogue partials of the identity form
  int fidelity_form = JOFC_FIDELITY_AUTO;
  int oos_route = JOFC_OOS_AUTO;
  int rho_grid = 0;  // epilogue grid of the identity-form solve (its partial rows)
  // solve state (sized for the current d)
  size_t d = 0;
  DevBuf<double> x0, x1, P, fid_part, com_part, trace, consts;
  DevBuf<Control> ctrl;
  Control* ctrl_host = nullptr;  // pinned
  int pass_grid = 0, epi_grid = 0;
  // per-CTA stream ranges of the pass kernel (pass_bounds) and what they were
  // computed for
  DevBuf<long long> bounds;
  std::vector<long long> bounds_key;
  size_t max_it_enqueued = 0;
  // caller-owned exchange buffer (multi-GPU) and pass-kernel instrumentation
  double* ext_P = nullptr;
  size_t ext_cap = 0;
  bool profiling = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_events;
  size_t prof_used = 0;
  // CUDA graph of the whole launch sequence (single-GPU, no events)
  std::map<std::vector<uintptr_t>, cudaGraphExec_t> graphs;
  bool use_graphs = true;
  // oos state
  DevBuf<double> oos_x, oos_delta, oos_y0, oos_y1, oos_part, oos_trace;
  DevBuf<double> oos_delta_t;  // [j][point group][n][32] (v2 pass)
  DevBuf<double> oos_delta_p;  // ring order of the persistent solve (jofc_oos_permute_kernel)
  DevBuf<OosPoint> oos_st;
  DevBuf<unsigned> oos_done;
  // streaming ingest staging
  IngestPanels ingest;
  DevBuf<unsigned long long> ingest_keys;
  // host -> device upload: copies on their own stream, overlapped with packing
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t up_copied[2] = {nullptr, nullptr}, up_packed[2] = {nullptr, nullptr};
  DevBuf<int> up_bad;  // set by the pack kernel on a non-finite / negative entry
  // early stop of synchronous solves: the done flag every kStopChunk
  // iterations (pinned) and the events that say it has landed
  int* stop_flag = nullptr;
  cudaEvent_t stop_ev[2] = {nullptr, nullptr};
  // peer-memory exchange (multi-GPU without NCCL)
  jofc_gpu::capi::PeerState peer;
  // C-native NCCL exchange (capi_nccl.cu): reduce-scatter of P, own-row mix,
  // all-gather of X; ncclComm_t, kept opaque here
  void* nccl_comm = nullptr;
  int nccl_world = 0;
};

namespace jofc_gpu {
namespace capi {

int copy_sync(jofc_ctx* c, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind);
int prof_begin(jofc_ctx* c, cudaEvent_t* end);
int require_problem(jofc_ctx* c);
// A_l of the resident Delta into c->sumsq (enqueued on the context stream);
// every path that (re)writes c->delta calls it before setting has_problem
int delta_sumsq(jofc_ctx* c);
// identity-form fidelity allowed (JOFC_FIDELITY=direct turns it off)
bool rho_enabled();
int diag_mode();
size_t stop_chunk();
long long fuse_epilogue_max_n();
double band_cost();
double block_cost(const Layout& L, int B, int J, bool enters_band);
void make_layout(jofc_ctx* c, size_t m, size_t n);
int finish_solve(jofc_ctx* c, Control* out);
// configuration buffer k (0/1): the context's own, or its peer slab's
double* xbuf(jofc_ctx* c, int k);
// launches of the D-templated kernels (c->d)
int pass_for_d(jofc_ctx* c, const PassParams& pp);
// everything before the first launch of a solve (validation, weights,
// buffers, X0, control block); fills the kernel parameters
int prepare_solve(jofc_ctx* c, const jofc_weights* spec, size_t d, const double* x0, double eps,
                  size_t max_it, PassParams* pp, EpiParams* ep);
// peer exchange: stage 0 pass, 1 mix, 2 decide of iteration t
int peer_stage(jofc_ctx* c, const PassParams& pp, size_t t, int stage);
int peer_check(jofc_ctx* c);
void peer_release(jofc_ctx* c);
// NCCL exchange: the world divides n_pad; collectives of iteration t
int nccl_check(jofc_ctx* c);
long long nccl_chunk_rows(const jofc_ctx* c);
int nccl_reduce(jofc_ctx* c, double* P, size_t fid_slot);
int nccl_gather(jofc_ctx* c, double* xn, double* sums = nullptr, size_t count = 0);
int nccl_wait(jofc_ctx* c);
void nccl_release(jofc_ctx* c);

}  // namespace capi
}  // namespace jofc_gpu
