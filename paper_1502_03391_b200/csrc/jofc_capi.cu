// jofc_capi.cu -- host side of libjofc_gpu.so: the C ABI in include/jofc_gpu.h.
//
// Owns the device state of one solve context: the packed Delta shard, the
// ping-pong configuration buffers, the product/fidelity exchange buffer, the
// control block, and the launch sequence
//
//     for t = 0 .. max_it:   pass(t) -> [all-reduce hook] -> epilogue(t)
//
// enqueued without host synchronisation: termination (the reference's
// decrease < eps rule, proj/src/solver.cpp:138-143) is decided on the device
// and later launches exit at entry once the control block says done.
#include <cuda_runtime.h>
#include <omp.h>
#include <unistd.h>

#include <chrono>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <map>
#include <memory>
#include <vector>

#include "jofc_gpu.h"
#include "jofc_kernels.cuh"
#include "jofc_oos.cuh"
#include "jofc_init.cuh"
#include "jofc_weights.h"
#include "ingest_io.h"

using namespace jofc_gpu;

namespace {

thread_local std::string g_error;

int set_error(int code, const char* fmt, ...) {
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

}  // namespace

struct jofc_ctx {
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
  DevBuf<OosPoint> oos_st;
  // streaming ingest staging
  IngestPanels ingest;
  // host -> device upload: copies on their own stream, overlapped with packing
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t up_copied[2] = {nullptr, nullptr}, up_packed[2] = {nullptr, nullptr};
};

namespace {

double* exchange(jofc_ctx* c) {
  const size_t need = static_cast<size_t>(c->lay.m) * c->lay.n_pad * c->d + 1;
  return (c->ext_P && c->ext_cap >= need) ? c->ext_P : c->P.p;
}

size_t fid_slot(const jofc_ctx* c) { return static_cast<size_t>(c->lay.m) * c->lay.n_pad * c->d; }

template <int D>
int setup_pass() {
  static bool attr_done = false;
  if (!attr_done) {
    JOFC_CUDA(cudaFuncSetAttribute(jofc_pass_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(sizeof(PassSmem<D>))));
    attr_done = true;
  }
  return JOFC_OK;
}

template <int D>
int launch_pass(jofc_ctx* c, const PassParams& pp) {
  int rc = setup_pass<D>();
  if (rc) return rc;
  jofc_pass_kernel<D><<<c->pass_grid, kPassThreads, sizeof(PassSmem<D>), c->stream>>>(pp);
  JOFC_CUDA(cudaGetLastError());
  return JOFC_OK;
}

template <int D>
int setup_for(jofc_ctx*) {
  return setup_pass<D>();
}

template <int D>
int launch_epi(jofc_ctx* c, const EpiParams& ep) {
  jofc_epilogue_kernel<D><<<c->epi_grid, 256, 0, c->stream>>>(ep);
  JOFC_CUDA(cudaGetLastError());
  return JOFC_OK;
}

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

// Synchronous copy ordered on the context stream (the context stream is a
// non-blocking stream: a plain cudaMemcpy on the legacy stream would not wait
// for its kernels, and a pageable H2D cudaMemcpy may return before the DMA).
int copy_sync(jofc_ctx* c, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
  JOFC_CUDA(cudaMemcpyAsync(dst, src, bytes, kind, c->stream));
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  return JOFC_OK;
}

// When profiling, records the start event of the next profiled launch on the
// context stream and hands back its end event (else leaves *end null).
int prof_begin(jofc_ctx* c, cudaEvent_t* end) {
  *end = nullptr;
  if (!c->profiling) return JOFC_OK;
  if (c->prof_used == c->prof_events.size()) {
    cudaEvent_t a, b;
    JOFC_CUDA(cudaEventCreate(&a));
    JOFC_CUDA(cudaEventCreate(&b));
    c->prof_events.emplace_back(a, b);
  }
  JOFC_CUDA(cudaEventRecord(c->prof_events[c->prof_used].first, c->stream));
  *end = c->prof_events[c->prof_used].second;
  ++c->prof_used;
  return JOFC_OK;
}

int pass_for_d(jofc_ctx* c, const PassParams& pp) { JOFC_DISPATCH_D(c->d, launch_pass, c, pp); }
int setup_for_d(jofc_ctx* c) { JOFC_DISPATCH_D(c->d, setup_for, c); }
int epi_for_d(jofc_ctx* c, const EpiParams& ep) { JOFC_DISPATCH_D(c->d, launch_epi, c, ep); }

int require_problem(jofc_ctx* c) {
  if (!c) return set_error(JOFC_EINVAL, "null context");
  if (!c->has_problem) return set_error(JOFC_EINVAL, "no problem uploaded (jofc_set_problem)");
  return JOFC_OK;
}

// Estimated pass-kernel cost of one block, in units of an interior block: masked
// blocks (diagonal-crossing or padded) +0.1, the first block a CTA processes
// of a row band +band_cost() (flush of the row sums, X row-block staging, two
// CTA barriers; 1.0 measured best at C3/C4/C5 among 0, 0.5, 1, 1.5, 2, 4, 8).
double band_cost() {
  static const double v = [] {
    const char* e = std::getenv("JOFC_BAND_COST");  // experiments
    return e ? std::atof(e) : 1.0;
  }();
  return v;
}

double block_cost(const Layout& L, int B, int J, bool enters_band) {
  const bool masked = J <= 2 * B + 1 || static_cast<long long>(kCols) * (J + 1) > L.n ||
                      static_cast<long long>(kRows) * (B + 1) > L.n;
  return 1.0 + (masked ? 0.1 : 0.0) + (enters_band ? band_cost() : 0.0);
}

// Layout for m modalities of n objects; this shard's contiguous stream range.
void make_layout(jofc_ctx* c, size_t m, size_t n) {
  Layout& L = c->lay;
  L.m = static_cast<int>(m);
  L.n = static_cast<long long>(n);
  L.nT = static_cast<int>((n + kCols - 1) / kCols);
  L.nB = (L.nT + 1) / 2;
  L.n_pad = static_cast<long long>(L.nB) * kRows;
  L.bpm = blocks_per_modality(L.nT);
  const long long total = L.total();
  if (c->world == 1) {
    L.begin = 0;
    L.end = total;
    return;
  }
  // shards: contiguous slices of equal estimated cost (block_cost; the same
  // model the CTA ranges use), identical on every rank
  std::vector<double> cost;
  cost.reserve(static_cast<size_t>(total));
  for (int l = 0; l < L.m; ++l)
    for (int B = 0; B < L.nB; ++B)
      for (int J = 2 * B; J < L.nT; ++J) cost.push_back(block_cost(L, B, J, J == 2 * B));
  double sum = 0.0;
  for (double v : cost) sum += v;
  long long cut_lo = 0, cut_hi = total;
  double acc = 0.0;
  for (long long g = 0; g < total; ++g) {
    acc += cost[g];
    if (c->rank > 0 && cut_lo == 0 && acc >= sum * c->rank / c->world) cut_lo = g + 1;
    if (acc >= sum * (c->rank + 1) / c->world && c->rank + 1 < c->world) {
      cut_hi = g + 1;
      break;
    }
  }
  L.begin = cut_lo;
  L.end = cut_hi;
}

// CTA ranges of the pass kernel: contiguous slices of this shard's block
// stream with equal estimated cost (block_cost).  With equal block counts the
// CTAs holding the short bands at the end of the stream ran ~6% longer than
// the average (ncu: SM active 93.8% of elapsed); balanced, the C3 pass is 5.7%
// faster, C4 4.6%, C5 13%.
int pass_bounds(jofc_ctx* c) {
  const Layout& L = c->lay;
  const std::vector<long long> key = {L.begin, L.end, L.nT, L.n, c->pass_grid,
                                      static_cast<long long>(band_cost() * 1000)};
  if (key == c->bounds_key && c->bounds.p) return JOFC_OK;
  const int NG = c->pass_grid;
  std::vector<double> cost;
  cost.reserve(static_cast<size_t>(L.local()));
  long long g = 0;
  for (int l = 0; l < L.m; ++l)
    for (int B = 0; B < L.nB; ++B)
      for (int J = 2 * B; J < L.nT; ++J, ++g) {
        if (g < L.begin || g >= L.end) continue;
        cost.push_back(block_cost(L, B, J, J == 2 * B || g == L.begin));
      }
  double total = 0.0;
  for (double v : cost) total += v;
  std::vector<long long> b(NG + 1, L.end);
  b[0] = L.begin;
  double acc = 0.0;
  int cut = 1;
  for (size_t i = 0; i < cost.size() && cut < NG; ++i) {
    acc += cost[i];
    if (acc >= total * cut / NG) b[cut++] = L.begin + static_cast<long long>(i) + 1;
  }
  for (; cut < NG; ++cut) b[cut] = L.end;
  JOFC_CUDA(c->bounds.ensure(NG + 1));
  JOFC_TRY(copy_sync(c, c->bounds.p, b.data(), (NG + 1) * sizeof(long long),
                     cudaMemcpyHostToDevice));
  c->bounds_key = key;
  return JOFC_OK;
}

int alloc_solve_state(jofc_ctx* c, size_t d, size_t max_it) {
  const Layout& L = c->lay;
  const size_t cfg = static_cast<size_t>(L.m) * L.n_pad * d;
  const bool resize = (d != c->d) || !c->x0.p || c->x0.n < cfg;
  c->d = d;
  JOFC_CUDA(c->x0.ensure(cfg));
  JOFC_CUDA(c->x1.ensure(cfg));
  if (c->ext_P && c->ext_cap >= cfg + 1) {
    c->P.release();
  } else {
    JOFC_CUDA(c->P.ensure(cfg + 1));
  }
  c->pass_grid = static_cast<int>(std::max<long long>(1, std::min<long long>(c->num_sms, L.local())));
  c->epi_grid = static_cast<int>((L.n + 255) / 256);
  JOFC_CUDA(c->fid_part.ensure(c->pass_grid));
  JOFC_TRY(pass_bounds(c));
  JOFC_CUDA(c->com_part.ensure(c->epi_grid));
  JOFC_CUDA(c->trace.ensure(max_it + 1));
  JOFC_CUDA(c->ctrl.ensure(1));
  JOFC_CUDA(c->consts.ensure(3 * static_cast<size_t>(L.m) * L.m + L.m));
  if (resize) {
    JOFC_CUDA(cudaMemsetAsync(c->x0.p, 0, cfg * sizeof(double), c->stream));
    JOFC_CUDA(cudaMemsetAsync(c->x1.p, 0, cfg * sizeof(double), c->stream));
  }
  JOFC_CUDA(cudaMemsetAsync(exchange(c), 0, (cfg + 1) * sizeof(double), c->stream));
  return JOFC_OK;
}

// Caller configuration (m blocks of n x d) -> padded device layout.
int upload_config(jofc_ctx* c, const double* x, double* dst) {
  const Layout& L = c->lay;
  const size_t block = static_cast<size_t>(L.n) * c->d;
  for (int l = 0; l < L.m; ++l)
    JOFC_CUDA(cudaMemcpyAsync(dst + static_cast<size_t>(l) * L.n_pad * c->d, x + l * block,
                              block * sizeof(double), cudaMemcpyDefault, c->stream));
  return JOFC_OK;
}

int download_config(jofc_ctx* c, const double* src, double* x) {
  const Layout& L = c->lay;
  const size_t block = static_cast<size_t>(L.n) * c->d;
  for (int l = 0; l < L.m; ++l)
    JOFC_CUDA(cudaMemcpyAsync(x + l * block, src + static_cast<size_t>(l) * L.n_pad * c->d,
                              block * sizeof(double), cudaMemcpyDefault, c->stream));
  return JOFC_OK;
}

// Enqueue the whole majorization (max_it transforms, max_it + 1 stress
// evaluations) on the context stream.  events (optional) get max_it + 2
// records: before pass t and after the final epilogue.
int enqueue_solve(jofc_ctx* c, const jofc_weights* spec, size_t d, const double* x0, double eps,
                  size_t max_it, std::vector<cudaEvent_t>* events) {
  int rc = require_problem(c);
  if (rc) return rc;
  if (d < 1 || d > static_cast<size_t>(kMaxD))
    return set_error(JOFC_EINVAL, "dim %zu unsupported (1..%d)", d, kMaxD);
  if (!(eps > 0.0)) return set_error(JOFC_EINVAL, "SolveOptions: eps must be positive");
  if (!x0) return set_error(JOFC_EINVAL, "null configuration");
  const Layout& L = c->lay;
  HostWeights hw;
  std::string msg;
  rc = build_weights(spec, static_cast<size_t>(L.m), static_cast<size_t>(L.n), &hw, &msg);
  if (rc) return set_error(rc, "%s", msg.c_str());
  rc = alloc_solve_state(c, d, max_it);
  if (rc) return rc;

  const size_t mm = static_cast<size_t>(L.m) * L.m;
  std::vector<double> consts(3 * mm + L.m);
  std::copy(hw.coef.begin(), hw.coef.end(), consts.begin());
  std::copy(hw.cross.begin(), hw.cross.end(), consts.begin() + mm);
  std::copy(hw.winv.begin(), hw.winv.end(), consts.begin() + 2 * mm);
  std::copy(hw.within.begin(), hw.within.end(), consts.begin() + 3 * mm);
  JOFC_CUDA(cudaMemcpyAsync(c->consts.p, consts.data(), consts.size() * sizeof(double),
                            cudaMemcpyHostToDevice, c->stream));
  rc = upload_config(c, x0, c->x0.p);
  if (rc) return rc;

  Control& h = *c->ctrl_host;
  std::memset(&h, 0, sizeof(Control));
  h.max_it = static_cast<int>(max_it);
  h.eps = eps;
  const double mn = static_cast<double>(L.m) * static_cast<double>(L.n);
  h.pairs = mn * (mn - 1.0) / 2.0;
  JOFC_CUDA(cudaMemcpyAsync(c->ctrl.p, &h, sizeof(Control), cudaMemcpyHostToDevice, c->stream));

  PassParams pp{};
  pp.delta = c->delta.p;
  pp.x0 = c->x0.p;
  pp.x1 = c->x1.p;
  pp.P = exchange(c);
  pp.fid_partials = c->fid_part.p;
  pp.ctrl = c->ctrl.p;
  pp.within = c->consts.p + 3 * mm;
  pp.n = L.n;
  pp.n_pad = L.n_pad;
  pp.nT = L.nT;
  pp.bpm = L.bpm;
  pp.begin = L.begin;
  pp.end = L.end;
  pp.fid_slot = fid_slot(c);
  pp.bounds = c->bounds.p;
  {
    const char* dg = getenv("JOFC_DIAG");  // experiments only; results are wrong when set
    pp.diag = dg ? atoi(dg) : 0;
  }

  EpiParams ep{};
  ep.x0 = c->x0.p;
  ep.x1 = c->x1.p;
  ep.P = exchange(c);
  ep.com_partials = c->com_part.p;
  ep.trace = c->trace.p;
  ep.ctrl = c->ctrl.p;
  ep.coef = c->consts.p;
  ep.cross = c->consts.p + mm;
  ep.m = L.m;
  ep.n = L.n;
  ep.n_pad = L.n_pad;
  ep.fid_slot = fid_slot(c);

  // Single GPU, no per-launch events: replay a captured CUDA graph of the
  // whole 2(max_it + 1)-kernel sequence (kernel parameters only hold buffer
  // pointers; everything iteration-dependent lives in the control block).
  const bool graphable = c->use_graphs && c->world == 1 && !events && !c->profiling;
  if (graphable) {
    std::vector<uintptr_t> key = {c->d, max_it, static_cast<uintptr_t>(c->pass_grid),
                                  static_cast<uintptr_t>(c->epi_grid),
                                  reinterpret_cast<uintptr_t>(pp.delta),
                                  reinterpret_cast<uintptr_t>(pp.x0),
                                  reinterpret_cast<uintptr_t>(pp.x1),
                                  reinterpret_cast<uintptr_t>(pp.P),
                                  reinterpret_cast<uintptr_t>(pp.ctrl),
                                  reinterpret_cast<uintptr_t>(ep.trace),
                                  reinterpret_cast<uintptr_t>(ep.com_partials),
                                  reinterpret_cast<uintptr_t>(pp.fid_partials),
                                  reinterpret_cast<uintptr_t>(ep.coef),
                                  static_cast<uintptr_t>(L.n), static_cast<uintptr_t>(L.m),
                                  static_cast<uintptr_t>(L.begin), static_cast<uintptr_t>(L.end),
                                  static_cast<uintptr_t>(pp.diag)};
    auto it = c->graphs.find(key);
    if (it == c->graphs.end()) {
      if (c->graphs.size() >= 8) {
        for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
        c->graphs.clear();
      }
      rc = setup_for_d(c);
      if (rc) return rc;
      JOFC_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
      int lrc = JOFC_OK;
      for (size_t t = 0; t <= max_it && !lrc; ++t) {
        lrc = pass_for_d(c, pp);
        if (!lrc) lrc = epi_for_d(c, ep);
      }
      cudaGraph_t g = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(c->stream, &g);
      if (lrc) {
        if (g) cudaGraphDestroy(g);
        return lrc;
      }
      if (ce != cudaSuccess)
        return set_error(JOFC_ECUDA, "graph capture failed: %s", cudaGetErrorString(ce));
      cudaGraphExec_t exec = nullptr;
      const cudaError_t ie = cudaGraphInstantiate(&exec, g, 0);
      cudaGraphDestroy(g);
      if (ie != cudaSuccess)
        return set_error(JOFC_ECUDA, "graph instantiate failed: %s", cudaGetErrorString(ie));
      it = c->graphs.emplace(key, exec).first;
    }
    JOFC_CUDA(cudaGraphLaunch(it->second, c->stream));
    c->launches += 2 * (max_it + 1);
    c->max_it_enqueued = max_it;
    return JOFC_OK;
  }

  for (size_t t = 0; t <= max_it; ++t) {
    if (events) JOFC_CUDA(cudaEventRecord((*events)[t], c->stream));
    cudaEvent_t pe1 = nullptr;
    rc = prof_begin(c, &pe1);
    if (rc) return rc;
    rc = pass_for_d(c, pp);
    if (rc) return rc;
    if (pe1) JOFC_CUDA(cudaEventRecord(pe1, c->stream));
    ++c->launches;
    if (c->world > 1) {
      if (!c->allreduce)
        return set_error(JOFC_ECOMM, "sharded context (world %d) without an all-reduce hook",
                         c->world);
      if (c->allreduce(exchange(c), fid_slot(c) + 1, c->stream, c->allreduce_user) != 0)
        return set_error(JOFC_ECOMM, "all-reduce hook failed at iteration %zu", t);
    }
    rc = epi_for_d(c, ep);
    if (rc) return rc;
    ++c->launches;
  }
  if (events) JOFC_CUDA(cudaEventRecord((*events)[max_it + 1], c->stream));
  c->max_it_enqueued = max_it;
  return JOFC_OK;
}

// Synchronise, then fetch the control block; maps device status to errors.
int finish_solve(jofc_ctx* c, Control* out) {
  JOFC_CUDA(cudaMemcpyAsync(c->ctrl_host, c->ctrl.p, sizeof(Control), cudaMemcpyDeviceToHost,
                            c->stream));
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  *out = *c->ctrl_host;
  if (out->status == 2) {
    if (out->err_iter == 0)
      return set_error(JOFC_ENUMERIC, "embed: non-finite stress at the initial configuration");
    return set_error(JOFC_ENUMERIC, "embed: non-finite stress at iteration %d", out->err_iter);
  }
  if (!out->done) return set_error(JOFC_ECUDA, "solve did not terminate (internal)");
  return JOFC_OK;
}

}  // namespace

// ======================================================================= C ABI
extern "C" {

const char* jofc_last_error(void) { return g_error.c_str(); }

int jofc_version(void) { return 1; }

int jofc_ctx_create(int device, jofc_ctx** out) {
  if (!out) return set_error(JOFC_EINVAL, "null output");
  *out = nullptr;
  int ndev = 0;
  JOFC_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev)
    return set_error(JOFC_EINVAL, "device %d out of range (%d devices)", device, ndev);
  JOFC_CUDA(cudaSetDevice(device));
  jofc_ctx* c = new jofc_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMallocHost(&c->ctrl_host, sizeof(Control));
  if (e != cudaSuccess) {
    delete c;
    return set_error(JOFC_ECUDA, "context setup: %s", cudaGetErrorString(e));
  }
  *out = c;
  return JOFC_OK;
}

int jofc_ctx_destroy(jofc_ctx* c) {
  if (!c) return JOFC_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (DevBuf<double>* b : {&c->delta, &c->x0, &c->x1, &c->P, &c->fid_part, &c->com_part,
                            &c->trace, &c->consts, &c->oos_x, &c->oos_delta, &c->oos_y0,
                            &c->oos_y1, &c->oos_part, &c->oos_trace})
    b->release();
  c->ctrl.release();
  c->oos_st.release();
  for (auto& e : c->prof_events) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
  if (c->ctrl_host) cudaFreeHost(c->ctrl_host);
  c->ingest.release();
  for (int k = 0; k < 2; ++k) {
    if (c->up_copied[k]) cudaEventDestroy(c->up_copied[k]);
    if (c->up_packed[k]) cudaEventDestroy(c->up_packed[k]);
  }
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return JOFC_OK;
}

void* jofc_ctx_stream(jofc_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

uint64_t jofc_launch_count(jofc_ctx* c) { return c ? c->launches : 0; }

int jofc_profile(jofc_ctx* c, int enable) {
  if (!c) return set_error(JOFC_EINVAL, "null context");
  c->profiling = enable != 0;
  c->prof_used = 0;
  return JOFC_OK;
}

int jofc_profile_read(jofc_ctx* c, double* pass_ms, uint64_t* pass_launches) {
  if (!c) return set_error(JOFC_EINVAL, "null context");
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  double total = 0.0;
  for (size_t i = 0; i < c->prof_used; ++i) {
    float ms = 0.f;
    JOFC_CUDA(cudaEventElapsedTime(&ms, c->prof_events[i].first, c->prof_events[i].second));
    total += ms;
  }
  if (pass_ms) *pass_ms = total;
  if (pass_launches) *pass_launches = c->prof_used;
  c->prof_used = 0;
  return JOFC_OK;
}

int jofc_set_exchange_buffer(jofc_ctx* c, double* buf, size_t capacity) {
  if (!c) return set_error(JOFC_EINVAL, "null context");
  c->ext_P = buf;
  c->ext_cap = buf ? capacity : 0;
  return JOFC_OK;
}

size_t jofc_exchange_count(jofc_ctx* c, size_t d) {
  if (!c || !c->has_problem) return 0;
  return static_cast<size_t>(c->lay.m) * c->lay.n_pad * d + 1;
}

int jofc_set_shard(jofc_ctx* c, int rank, int world) {
  if (!c) return set_error(JOFC_EINVAL, "null context");
  if (world < 1 || rank < 0 || rank >= world)
    return set_error(JOFC_EINVAL, "shard %d of %d invalid", rank, world);
  c->rank = rank;
  c->world = world;
  c->has_problem = false;
  return JOFC_OK;
}

int jofc_set_allreduce(jofc_ctx* c, jofc_allreduce_fn fn, void* user) {
  if (!c) return set_error(JOFC_EINVAL, "null context");
  c->allreduce = fn;
  c->allreduce_user = user;
  return JOFC_OK;
}

size_t jofc_problem_bytes(jofc_ctx* c) {
  return (c && c->has_problem) ? static_cast<size_t>(c->lay.local()) * kBlockBytes : 0;
}

double jofc_problem_pairs(jofc_ctx* c) {
  if (!c || !c->has_problem) return 0.0;
  const double n = static_cast<double>(c->lay.n);
  return static_cast<double>(c->lay.m) * n * (n - 1.0) / 2.0;
}

int jofc_set_problem(jofc_ctx* c, size_t m, size_t n, const double* const* delta, int normalize) {
  if (!c) return set_error(JOFC_EINVAL, "null context");
  if (m == 0) return set_error(JOFC_EINVAL, "OmnibusProblem: at least one modality required");
  if (n < 2) return set_error(JOFC_EINVAL, "OmnibusProblem: need at least two objects");
  if (!delta) return set_error(JOFC_EINVAL, "null delta");
  for (size_t l = 0; l < m; ++l)
    if (!delta[l]) return set_error(JOFC_EINVAL, "OmnibusProblem: modality %zu is null", l);
  JOFC_CUDA(cudaSetDevice(c->device));
  c->has_problem = false;
  make_layout(c, m, n);
  const Layout& L = c->lay;
  JOFC_CUDA(c->delta.ensure(static_cast<size_t>(std::max<long long>(L.local(), 1)) * kBlockElems));

  // Frobenius norms over the full dense matrix in the reference's order.
  std::vector<double> norms(m, 0.0);
  if (normalize)
    for (size_t l = 0; l < m; ++l) {
      double s = 0.0;
      const double* dl = delta[l];
      for (size_t i = 0; i < n * n; ++i) s += dl[i] * dl[i];
      norms[l] = std::sqrt(s);
    }

  // Staging: up to kChunk row blocks (128 rows each) of the dense matrix,
  // columns from the chunk's first row onwards (the upper part only).  Two
  // stage buffers: the copy of chunk k+1 (copy stream) runs under the packing
  // of chunk k (context stream).
  const int kChunk = 4;
  if (!c->copy_stream) {
    JOFC_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
      JOFC_CUDA(cudaEventCreateWithFlags(&c->up_copied[k], cudaEventDisableTiming));
      JOFC_CUDA(cudaEventCreateWithFlags(&c->up_packed[k], cudaEventDisableTiming));
    }
  }
  DevBuf<double> stage[2];
  DevBuf<int> bad;
  for (int k = 0; k < 2; ++k) JOFC_CUDA(stage[k].ensure(static_cast<size_t>(kChunk) * kRows * L.n_pad));
  JOFC_CUDA(bad.ensure(1));
  JOFC_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), c->stream));
  // the copy stream starts after everything already queued on the context stream
  JOFC_CUDA(cudaEventRecord(c->up_packed[0], c->stream));
  JOFC_CUDA(cudaStreamWaitEvent(c->copy_stream, c->up_packed[0], 0));
  long long chunk = 0;
  for (int l = 0; l < L.m; ++l) {
    for (int B0 = 0; B0 < L.nB; B0 += kChunk) {
      const int B1 = std::min(L.nB, B0 + kChunk);
      const long long g_lo = static_cast<long long>(l) * L.bpm + row_first(L.nT, B0);
      const long long g_hi = static_cast<long long>(l) * L.bpm + row_first(L.nT, B1);
      if (g_hi <= L.begin || g_lo >= L.end) continue;  // not in this shard
      const int k = static_cast<int>(chunk & 1);
      const long long r0 = static_cast<long long>(B0) * kRows;
      const long long r1 = std::min<long long>(L.n, static_cast<long long>(B1) * kRows);
      const long long c0 = r0;
      if (chunk >= 2) JOFC_CUDA(cudaStreamWaitEvent(c->copy_stream, c->up_packed[k], 0));
      if (r1 > r0 && c0 < L.n) {
        const size_t width = static_cast<size_t>(L.n - c0) * sizeof(double);
        JOFC_CUDA(cudaMemcpy2DAsync(stage[k].p, L.n_pad * sizeof(double), delta[l] + r0 * L.n + c0,
                                    L.n * sizeof(double), width, static_cast<size_t>(r1 - r0),
                                    cudaMemcpyDefault, c->copy_stream));
      }
      JOFC_CUDA(cudaEventRecord(c->up_copied[k], c->copy_stream));
      JOFC_CUDA(cudaStreamWaitEvent(c->stream, c->up_copied[k], 0));
      PackParams pk{};
      pk.stage = stage[k].p;
      pk.pitch = L.n_pad;
      pk.r0 = r0;
      pk.c0 = c0;
      pk.n = L.n;
      pk.nT = L.nT;
      pk.bpm = L.bpm;
      pk.g_first = g_lo;
      pk.begin = L.begin;
      pk.end = L.end;
      pk.dst = c->delta.p;
      pk.norm = (normalize && norms[l] != 0.0) ? norms[l] : 0.0;
      pk.bad = bad.p;
      jofc_pack_kernel<<<static_cast<unsigned>(g_hi - g_lo), 256, 0, c->stream>>>(pk);
      JOFC_CUDA(cudaGetLastError());
      JOFC_CUDA(cudaEventRecord(c->up_packed[k], c->stream));
      ++c->launches;
      ++chunk;
    }
  }
  int hbad = 0;
  JOFC_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  if (hbad) return set_error(JOFC_EINVAL, "OmnibusProblem: delta has a non-finite or negative entry");
  c->has_problem = true;
  return JOFC_OK;
}

int jofc_set_problem_features(jofc_ctx* c, size_t m, size_t n, size_t p, const double* feats) {
  if (!c) return set_error(JOFC_EINVAL, "null context");
  if (m == 0 || n < 2 || p == 0 || !feats)
    return set_error(JOFC_EINVAL, "features: need m >= 1, n >= 2, p >= 1");
  JOFC_CUDA(cudaSetDevice(c->device));
  c->has_problem = false;
  make_layout(c, m, n);
  const Layout& L = c->lay;
  JOFC_CUDA(c->delta.ensure(static_cast<size_t>(std::max<long long>(L.local(), 1)) * kBlockElems));
  DevBuf<double> f;
  JOFC_CUDA(f.ensure(m * n * p));
  JOFC_CUDA(cudaMemcpyAsync(f.p, feats, m * n * p * sizeof(double), cudaMemcpyDefault, c->stream));
  const size_t smem = (kRows + kCols) * p * sizeof(double);
  if (smem > 48 * 1024)
    JOFC_CUDA(cudaFuncSetAttribute(jofc_edm_block_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
  const long long blocks = L.local();
  for (long long off = 0; off < blocks; off += (1LL << 30)) {
    const long long cnt = std::min<long long>(blocks - off, 1LL << 30);
    jofc_edm_block_kernel<<<static_cast<unsigned>(cnt), 256, smem, c->stream>>>(
        f.p, L.n, static_cast<int>(p), L.nT, L.bpm, L.begin + off, L.end, c->delta.p);
    JOFC_CUDA(cudaGetLastError());
    ++c->launches;
  }
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  f.release();
  c->has_problem = true;
  return JOFC_OK;
}

int jofc_fjofc_enqueue(jofc_ctx* c, const jofc_weights* spec, size_t d, const double* x0,
                       double eps, size_t max_it) {
  if (!c) return set_error(JOFC_EINVAL, "null context");
  JOFC_CUDA(cudaSetDevice(c->device));
  return enqueue_solve(c, spec, d, x0, eps, max_it, nullptr);
}

int jofc_fetch_result(jofc_ctx* c, double* x_out, double* trace_out, size_t* iterations,
                      int* converged) {
  int rc = require_problem(c);
  if (rc) return rc;
  Control h;
  rc = finish_solve(c, &h);
  if (rc) return rc;
  if (x_out) {
    rc = download_config(c, (h.iterations & 1) ? c->x1.p : c->x0.p, x_out);
    if (rc) return rc;
  }
  if (trace_out)
    JOFC_CUDA(cudaMemcpyAsync(trace_out, c->trace.p, (h.iterations + 1) * sizeof(double),
                              cudaMemcpyDefault, c->stream));
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  if (iterations) *iterations = static_cast<size_t>(h.iterations);
  if (converged) *converged = h.converged;
  return JOFC_OK;
}

int jofc_fjofc_embed(jofc_ctx* c, const jofc_weights* spec, size_t d, const double* x0, double eps,
                     size_t max_it, double* x_out, double* trace_out, size_t* iterations,
                     int* converged, double* step_seconds) {
  if (!c) return set_error(JOFC_EINVAL, "null context");
  JOFC_CUDA(cudaSetDevice(c->device));
  std::vector<cudaEvent_t> ev;
  if (step_seconds) {
    ev.resize(max_it + 2);
    for (auto& e : ev) JOFC_CUDA(cudaEventCreate(&e));
  }
  int rc = enqueue_solve(c, spec, d, x0, eps, max_it, step_seconds ? &ev : nullptr);
  size_t its = 0;
  if (!rc) rc = jofc_fetch_result(c, x_out, trace_out, &its, converged);
  if (!rc && iterations) *iterations = its;
  if (!rc && step_seconds) {
    for (size_t t = 0; t < its; ++t) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[t], ev[t + 1]);
      step_seconds[t] = ms * 1e-3;
    }
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return rc;
}

int jofc_raw_stress(jofc_ctx* c, const jofc_weights* spec, size_t d, const double* x,
                    double* stress) {
  if (!c) return set_error(JOFC_EINVAL, "null context");
  JOFC_CUDA(cudaSetDevice(c->device));
  int rc = enqueue_solve(c, spec, d, x, 1.0, 0, nullptr);
  if (rc) return rc;
  double s = 0.0;
  JOFC_CUDA(cudaMemcpyAsync(&s, c->trace.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  *stress = s;  // non-finite stress is returned as is (raw_stress does not throw)
  return JOFC_OK;
}

int jofc_guttman_step(jofc_ctx* c, const jofc_weights* spec, size_t d, const double* x,
                      double* x_next) {
  if (!c) return set_error(JOFC_EINVAL, "null context");
  JOFC_CUDA(cudaSetDevice(c->device));
  // One pass + epilogue with max_it = 1 (eps tiny so the rule cannot fire at
  // t = 0): X_1 lands in buffer 1 whatever the stress is.
  const Layout& L = c->lay;
  int rc = require_problem(c);
  if (rc) return rc;
  if (d < 1 || d > static_cast<size_t>(kMaxD))
    return set_error(JOFC_EINVAL, "dim %zu unsupported (1..%d)", d, kMaxD);
  rc = enqueue_solve(c, spec, d, x, 1e-300, 0, nullptr);
  (void)L;
  if (rc) return rc;
  // enqueue_solve(max_it = 0) marks the solve done at t = 0 after the mix, so
  // buffer 1 holds the transform of x.
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  rc = download_config(c, c->x1.p, x_next);
  if (rc) return rc;
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  return JOFC_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- out-of-sample
namespace {

template <int D>
int oos_launch(jofc_ctx* c, const OosParams& op, int steps) {
  // 4 slices of the in-sample range (measured best at C5 among 2..16)
  const dim3 pg((op.k + kOosWarps - 1) / kOosWarps, op.m,
                static_cast<unsigned>(std::min<long long>(kOosSplits, std::max<long long>(1, op.n / 256))));
  const unsigned ug = (op.k + 127) / 128;
  // The 2(steps + 1) launches are replayed from a captured CUDA graph (all
  // per-step state is in the device-side point records).
  std::vector<uintptr_t> key = {0x0005u, static_cast<uintptr_t>(D), static_cast<uintptr_t>(op.k),
                                static_cast<uintptr_t>(op.m), static_cast<uintptr_t>(op.n),
                                static_cast<uintptr_t>(steps), static_cast<uintptr_t>(op.fixed),
                                static_cast<uintptr_t>(op.max_it),
                                reinterpret_cast<uintptr_t>(op.x),
                                reinterpret_cast<uintptr_t>(op.deltas),
                                reinterpret_cast<uintptr_t>(op.y0),
                                reinterpret_cast<uintptr_t>(op.y1),
                                reinterpret_cast<uintptr_t>(op.part),
                                reinterpret_cast<uintptr_t>(op.st),
                                reinterpret_cast<uintptr_t>(op.traces)};
  uint64_t wbits, ebits;
  std::memcpy(&wbits, &op.w, 8);
  std::memcpy(&ebits, &op.eps, 8);
  key.push_back(static_cast<uintptr_t>(wbits));
  key.push_back(static_cast<uintptr_t>(ebits));
  auto it = c->graphs.find(key);
  if (it == c->graphs.end()) {
    if (c->graphs.size() >= 8) {
      for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
      c->graphs.clear();
    }
    JOFC_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    constexpr int smem = oos_smem_bytes<D>();
    if (smem > 48 * 1024)
      JOFC_CUDA(cudaFuncSetAttribute(jofc_oos_pass_kernel<D>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    for (int t = 0; t <= steps; ++t) {
      jofc_oos_pass_kernel<D><<<pg, kOosWarps * 32, smem, c->stream>>>(op);
      jofc_oos_update_kernel<D><<<ug, 128, 0, c->stream>>>(op);
    }
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(c->stream, &g);
    if (ce != cudaSuccess)
      return set_error(JOFC_ECUDA, "oos graph capture failed: %s", cudaGetErrorString(ce));
    cudaGraphExec_t exec = nullptr;
    const cudaError_t ie = cudaGraphInstantiate(&exec, g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess)
      return set_error(JOFC_ECUDA, "oos graph instantiate failed: %s", cudaGetErrorString(ie));
    it = c->graphs.emplace(key, exec).first;
  }
  JOFC_CUDA(cudaGraphLaunch(it->second, c->stream));
  c->launches += 2 * (steps + 1);
  return JOFC_OK;
}

int oos_run(jofc_ctx* c, size_t k, size_t m, size_t n, size_t d, const double* x,
            const double* deltas, double w, const double* y0, double eps, size_t max_it,
            int fixed, double* y_out, double* traces, size_t* iterations, double* stress0) {
  if (!c) return set_error(JOFC_EINVAL, "null context");
  if (!(w > 0.0)) return set_error(JOFC_EINVAL, "oos: w must be strictly positive");
  if (!(eps > 0.0)) return set_error(JOFC_EINVAL, "OosOptions: eps must be positive");
  if (m == 0 || n == 0 || k == 0) return set_error(JOFC_EINVAL, "oos: empty input");
  if (d < 1 || d > static_cast<size_t>(kMaxD))
    return set_error(JOFC_EINVAL, "dim %zu unsupported (1..%d)", d, kMaxD);
  JOFC_CUDA(cudaSetDevice(c->device));
  JOFC_CUDA(c->oos_x.ensure(m * n * d + 4));  // + slack: chunk copies round up to 16 bytes
  JOFC_CUDA(c->oos_delta.ensure(k * m * n));
  JOFC_CUDA(c->oos_y0.ensure(k * m * d));
  JOFC_CUDA(c->oos_y1.ensure(k * m * d));
  JOFC_CUDA(c->oos_part.ensure(k * m * (d + 2) + k));
  JOFC_CUDA(c->oos_trace.ensure(k * (max_it + 1)));
  JOFC_CUDA(c->oos_st.ensure(k));
  JOFC_CUDA(cudaMemcpyAsync(c->oos_x.p, x, m * n * d * sizeof(double), cudaMemcpyDefault, c->stream));
  JOFC_CUDA(cudaMemcpyAsync(c->oos_delta.p, deltas, k * m * n * sizeof(double), cudaMemcpyDefault,
                            c->stream));
  JOFC_CUDA(cudaMemcpyAsync(c->oos_y0.p, y0, k * m * d * sizeof(double), cudaMemcpyDefault,
                            c->stream));
  JOFC_CUDA(cudaMemsetAsync(c->oos_st.p, 0, k * sizeof(OosPoint), c->stream));
  JOFC_CUDA(cudaMemsetAsync(c->oos_part.p, 0, (k * m * (d + 2) + k) * sizeof(double), c->stream));
  OosParams op{};
  op.x = c->oos_x.p;
  op.deltas = c->oos_delta.p;
  op.y0 = c->oos_y0.p;
  op.y1 = c->oos_y1.p;
  op.part = c->oos_part.p;
  op.st = c->oos_st.p;
  op.traces = c->oos_trace.p;
  op.k = static_cast<int>(k);
  op.m = static_cast<int>(m);
  op.n = static_cast<long long>(n);
  op.w = w;
  op.eps = eps;
  op.term_count = static_cast<double>(m * n) + 0.5 * static_cast<double>(m * (m - 1));
  op.max_it = static_cast<int>(max_it);
  op.fixed = fixed;
  int rc;
  switch (d) {
    case 1: rc = oos_launch<1>(c, op, static_cast<int>(max_it)); break;
    case 2: rc = oos_launch<2>(c, op, static_cast<int>(max_it)); break;
    case 3: rc = oos_launch<3>(c, op, static_cast<int>(max_it)); break;
    case 4: rc = oos_launch<4>(c, op, static_cast<int>(max_it)); break;
    case 5: rc = oos_launch<5>(c, op, static_cast<int>(max_it)); break;
    case 6: rc = oos_launch<6>(c, op, static_cast<int>(max_it)); break;
    case 7: rc = oos_launch<7>(c, op, static_cast<int>(max_it)); break;
    case 8: rc = oos_launch<8>(c, op, static_cast<int>(max_it)); break;
    case 9: rc = oos_launch<9>(c, op, static_cast<int>(max_it)); break;
    default: rc = oos_launch<10>(c, op, static_cast<int>(max_it)); break;
  }
  if (rc) return rc;
  std::vector<OosPoint> st(k);
  JOFC_CUDA(cudaMemcpyAsync(st.data(), c->oos_st.p, k * sizeof(OosPoint), cudaMemcpyDeviceToHost,
                            c->stream));
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  for (size_t p = 0; p < k; ++p)
    if (st[p].status == 2) {
      if (st[p].iterations == 0)
        return set_error(JOFC_ENUMERIC, "oos_embed: non-finite stress at the initial point");
      return set_error(JOFC_ENUMERIC, "oos_embed: non-finite stress at iteration %d",
                       st[p].iterations);
    }
  // Final y of point p is in buffer (iterations_p & 1).
  std::vector<double> ya(k * m * d), yb(k * m * d);
  if (y_out) {
    JOFC_CUDA(cudaMemcpyAsync(ya.data(), c->oos_y0.p, k * m * d * sizeof(double),
                              cudaMemcpyDeviceToHost, c->stream));
    JOFC_CUDA(cudaMemcpyAsync(yb.data(), c->oos_y1.p, k * m * d * sizeof(double),
                              cudaMemcpyDeviceToHost, c->stream));
  }
  if (traces)
    JOFC_CUDA(cudaMemcpyAsync(traces, c->oos_trace.p, k * (max_it + 1) * sizeof(double),
                              cudaMemcpyDefault, c->stream));
  if (stress0)
    JOFC_CUDA(cudaMemcpyAsync(stress0, c->oos_trace.p, sizeof(double), cudaMemcpyDeviceToHost,
                              c->stream));
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  std::vector<double> y_all(y_out ? k * m * d : 0);
  for (size_t p = 0; p < k; ++p) {
    if (iterations) iterations[p] = static_cast<size_t>(st[p].iterations);
    if (y_out) {
      const double* src = (st[p].iterations & 1) ? yb.data() : ya.data();
      std::memcpy(y_all.data() + p * m * d, src + p * m * d, m * d * sizeof(double));
    }
  }
  if (y_out)  // y_out may be host or device memory
    JOFC_TRY(copy_sync(c, y_out, y_all.data(), y_all.size() * sizeof(double), cudaMemcpyDefault));
  return JOFC_OK;
}

}  // namespace

extern "C" {

int jofc_oos_batch(jofc_ctx* c, size_t k, size_t m, size_t n, size_t d, const double* x,
                   const double* deltas, double w, const double* y0, double eps, size_t max_it,
                   int fixed_iterations, double* y_out, double* traces, size_t* iterations) {
  return oos_run(c, k, m, n, d, x, deltas, w, y0, eps, max_it, fixed_iterations, y_out, traces,
                 iterations, nullptr);
}

int jofc_oos_stress(jofc_ctx* c, size_t m, size_t n, size_t d, const double* y, const double* x,
                    const double* deltas, double w, double* stress) {
  return oos_run(c, 1, m, n, d, x, deltas, w, y, 1.0, 0, 1, nullptr, nullptr, nullptr, stress);
}

int jofc_oos_step(jofc_ctx* c, size_t m, size_t n, size_t d, const double* y, const double* x,
                  const double* deltas, double w, double* y_next) {
  return oos_run(c, 1, m, n, d, x, deltas, w, y, 1.0, 1, 1, y_next, nullptr, nullptr, nullptr);
}

}  // extern "C"

// ---------------------------------------------------------------- initialisation
namespace {

// The panel kernels, instantiated per subspace width p = d + 4.
struct PanelOps {
  void (*matvec)(const double*, long long, const double*, double*, int, cudaStream_t);
  void (*gram_shift)(const double*, const double*, double*, double*, long long, int, double,
                     double*, int, cudaStream_t);
  void (*ritz_orth)(double*, const double*, const double*, long long, int,
                    const init::RitzParams&, double*, double*, int, cudaStream_t);
  void (*apply_rinv)(double*, long long, const init::RitzParams&, cudaStream_t);
};

template <int P>
PanelOps panel_ops() {
  PanelOps o;
  o.matvec = [](const double* S, long long n, const double* q, double* z, int splits,
                 cudaStream_t st) {
    const dim3 grid(static_cast<unsigned>((n + init::kMvRows - 1) / init::kMvRows),
                    static_cast<unsigned>(splits));
    init::matvec_sym_kernel<P><<<grid, 256, 0, st>>>(S, n, q, z);
  };
  o.gram_shift = [](const double* q, const double* zp, double* z, double* w, long long n,
                    int splits, double shift, double* part, int grid, cudaStream_t st) {
    init::gram_shift_kernel<P><<<grid, 256, 0, st>>>(q, zp, z, w, n, splits, shift, part);
  };
  o.ritz_orth = [](double* q, const double* z, const double* w, long long n, int k,
                   const init::RitzParams& prm, double* ritz, double* part, int grid,
                   cudaStream_t st) {
    init::ritz_orth_kernel<P><<<grid, 256, 0, st>>>(q, z, w, n, k, prm, ritz, part);
  };
  o.apply_rinv = [](double* q, long long n, const init::RitzParams& prm, cudaStream_t st) {
    init::apply_rinv_kernel<P><<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(q, n, prm);
  };
  return o;
}

bool panel_ops_for(int p, PanelOps& o) {
  switch (p) {
    case 5: o = panel_ops<5>(); return true;
    case 6: o = panel_ops<6>(); return true;
    case 7: o = panel_ops<7>(); return true;
    case 8: o = panel_ops<8>(); return true;
    case 9: o = panel_ops<9>(); return true;
    case 10: o = panel_ops<10>(); return true;
    case 11: o = panel_ops<11>(); return true;
    case 12: o = panel_ops<12>(); return true;
    case 13: o = panel_ops<13>(); return true;
    case 14: o = panel_ops<14>(); return true;
    default: return false;
  }
}

// Top-k eigenpairs of the symmetric n x n matrix S (device, row-major) with
// ||S||_F = snorm: the reference's dense cyclic Jacobi (host) when
// n <= jacobi_limit or k + 4 >= n, else its shifted orthogonal iteration with
// Rayleigh-Ritz (proj/src/linalg.cpp:167-271) with the n x p panels on the
// device.  values (k, descending) and vecs (n x k, unit columns, largest
// component positive).
int eigen_top_device(jofc_ctx* c, const double* S_dev, long long n, size_t k, double snorm,
                     long long jacobi_limit, std::vector<double>& values, init::Mat& vecs,
                     int& sweeps, double& t_sync) {
  using clk = std::chrono::steady_clock;
  struct {
    const double* p;
  } S{S_dev};
  values.assign(k, 0.0);
  vecs = init::Mat(n, k);
  if (n <= jacobi_limit || k + 4 >= static_cast<size_t>(n)) {
    // the reference's dense route (cyclic Jacobi on the whole S)
    init::Mat h(n, n);
    JOFC_TRY(copy_sync(c, h.a.data(), S.p, h.a.size() * sizeof(double), cudaMemcpyDeviceToHost));
    std::vector<double> ev;
    init::Mat v;
    if (!init::jacobi_eigen(h, ev, v))
      return set_error(JOFC_ENUMERIC, "jacobi eigensolver did not converge within the sweep cap");
    std::vector<size_t> order(n);
    std::iota(order.begin(), order.end(), size_t{0});
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return ev[a] > ev[b]; });
    for (size_t cc = 0; cc < k; ++cc) {
      std::vector<double> col(n);
      for (long long r = 0; r < n; ++r) col[r] = v(r, order[cc]);
      init::fix_sign(col);
      values[cc] = ev[order[cc]];
      for (long long r = 0; r < n; ++r) vecs(r, cc) = col[r];
    }
  } else if (snorm == 0.0) {
    for (size_t cc = 0; cc < k; ++cc) {
      values[cc] = 0.0;
      vecs(cc, cc) = 1.0;
    }
  } else {
    // shifted orthogonal iteration with Rayleigh-Ritz (proj/src/linalg.cpp:167-271)
    const size_t p = k + 4;
    const double shift = snorm, tol = 1e-9 * snorm;
    PanelOps ops;
    if (!panel_ops_for(static_cast<int>(p), ops))
      return set_error(JOFC_EINVAL, "cmds: subspace width %zu unsupported", p);
    init::Mat q(n, p);
    init::Normals rng(0x9e3779b97f4a7c15ull);
    for (double& v : q.a) v = rng.next();
    init::orthonormalize(q);
    const int grid1 = std::min<int>(c->num_sms * 8, static_cast<int>((n + 63) / 64));
    const int grid2 = std::min<int>(c->num_sms * 2, static_cast<int>((n + 255) / 256));
    const int grid = std::max(grid1, grid2);
    const size_t part1 = 2 * p * p, part2 = p + p * p;
    // column splits: enough CTAs for ~16 per SM, each split one n x p partial
    const long long row_blocks = (n + init::kMvRows - 1) / init::kMvRows;
    const int splits = static_cast<int>(std::min<long long>(
        init::kMvMaxSplits, std::max<long long>(1, (16LL * c->num_sms + row_blocks - 1) / row_blocks)));
    DevBuf<double> dq, dzp, dz, dw, dritz, dpart;
    JOFC_CUDA(dzp.ensure(splits * n * p));
    JOFC_CUDA(dq.ensure(n * p));
    JOFC_CUDA(dz.ensure(n * p));
    JOFC_CUDA(dw.ensure(n * p));
    JOFC_CUDA(dritz.ensure(n * k));
    JOFC_CUDA(dpart.ensure(grid * std::max(part1, part2)));
    // pinned staging for the per-CTA partials (two small D2H reads per sweep)
    struct Pinned {
      double* p = nullptr;
      ~Pinned() {
        if (p) cudaFreeHost(p);
      }
    } hpart;
    JOFC_CUDA(cudaMallocHost(&hpart.p, grid * std::max(part1, part2) * sizeof(double)));
    JOFC_CUDA(cudaMemcpyAsync(dq.p, q.a.data(), q.a.size() * sizeof(double),
                              cudaMemcpyHostToDevice, c->stream));
    auto fetch = [&](int blocks, size_t per) -> int {
      JOFC_CUDA(cudaGetLastError());
      const auto t0 = clk::now();
      JOFC_CUDA(cudaMemcpyAsync(hpart.p, dpart.p, blocks * per * sizeof(double),
                                cudaMemcpyDeviceToHost, c->stream));
      JOFC_CUDA(cudaStreamSynchronize(c->stream));
      t_sync += std::chrono::duration<double>(clk::now() - t0).count();
      return JOFC_OK;
    };
    auto sum_part = [&](int blocks, size_t per, size_t off, size_t cnt, std::vector<double>& out) {
      out.assign(cnt, 0.0);
      for (int b = 0; b < blocks; ++b)
        for (size_t e = 0; e < cnt; ++e) out[e] += hpart.p[b * per + off + e];
    };
    bool done = false;
    std::vector<double> acc;
    for (int iter = 0; iter < 5000 && !done; ++iter) {
      ++sweeps;
      cudaEvent_t pe1 = nullptr;
      int rc = prof_begin(c, &pe1);
      if (rc) return rc;
      ops.matvec(S.p, n, dq.p, dzp.p, splits, c->stream);
      if (pe1) JOFC_CUDA(cudaEventRecord(pe1, c->stream));
      ops.gram_shift(dq.p, dzp.p, dz.p, dw.p, n, splits, shift, dpart.p, grid1, c->stream);
      c->launches += 2;
      rc = fetch(grid1, part1);
      if (rc) return rc;
      init::Mat t(p, p), g(p, p);
      sum_part(grid1, part1, 0, p * p, acc);
      std::copy(acc.begin(), acc.end(), t.a.begin());
      sum_part(grid1, part1, p * p, p * p, acc);
      std::copy(acc.begin(), acc.end(), g.a.begin());
      for (size_t i = 0; i < p; ++i)
        for (size_t j = i + 1; j < p; ++j) t(i, j) = t(j, i) = 0.5 * (t(i, j) + t(j, i));
      std::vector<double> theta;
      init::Mat u;
      if (!init::jacobi_eigen(t, theta, u))
        return set_error(JOFC_ENUMERIC, "jacobi eigensolver did not converge within the sweep cap");
      std::vector<size_t> order(p);
      std::iota(order.begin(), order.end(), size_t{0});
      std::stable_sort(order.begin(), order.end(),
                       [&](size_t a, size_t b) { return theta[a] > theta[b]; });
      init::RitzParams prm{};
      for (size_t cc = 0; cc < k; ++cc) {
        for (size_t j = 0; j < p; ++j) prm.u[j * init::kMaxP + cc] = u(j, order[cc]);
        prm.theta[cc] = theta[order[cc]];
        values[cc] = theta[order[cc]];
      }
      init::Mat rinv;
      const bool chol = init::cholesky_rinv(g, rinv);
      for (size_t i = 0; i < p; ++i)
        for (size_t j = 0; j < p; ++j)
          prm.rinv[i * init::kMaxP + j] = chol ? rinv(i, j) : (i == j ? 1.0 : 0.0);
      ops.ritz_orth(dq.p, dz.p, dw.p, n, static_cast<int>(k), prm, dritz.p, dpart.p, grid2,
                    c->stream);
      ++c->launches;
      rc = fetch(grid2, part2);
      if (rc) return rc;
      sum_part(grid2, part2, 0, k, acc);
      bool conv = true;
      for (size_t cc = 0; cc < k; ++cc)
        if (std::sqrt(acc[cc]) > tol) conv = false;
      if (conv) {
        init::Mat ritz(n, k);
        JOFC_TRY(copy_sync(c, ritz.a.data(), dritz.p, ritz.a.size() * sizeof(double),
                             cudaMemcpyDeviceToHost));
        for (size_t cc = 0; cc < k; ++cc) {
          std::vector<double> col(n);
          double nr = 0.0;
          for (long long r = 0; r < n; ++r) {
            col[r] = ritz(r, cc);
            nr += col[r] * col[r];
          }
          nr = std::sqrt(nr);
          for (double& v : col) v /= nr;
          init::fix_sign(col);
          for (long long r = 0; r < n; ++r) vecs(r, cc) = col[r];
        }
        done = true;
        break;
      }
      if (!chol) {  // ill-conditioned panel: the reference's Gram-Schmidt on the host
        JOFC_TRY(copy_sync(c, q.a.data(), dw.p, q.a.size() * sizeof(double),
                             cudaMemcpyDeviceToHost));
        init::orthonormalize(q);
        JOFC_TRY(copy_sync(c, dq.p, q.a.data(), q.a.size() * sizeof(double),
                             cudaMemcpyHostToDevice));
        continue;
      }
      sum_part(grid2, part2, p, p * p, acc);
      std::copy(acc.begin(), acc.end(), g.a.begin());
      if (init::cholesky_rinv(g, rinv)) {
        for (size_t i = 0; i < p; ++i)
          for (size_t j = 0; j < p; ++j) prm.rinv[i * init::kMaxP + j] = rinv(i, j);
        ops.apply_rinv(dq.p, n, prm, c->stream);
        ++c->launches;
        JOFC_CUDA(cudaGetLastError());
      } else {
        JOFC_TRY(copy_sync(c, q.a.data(), dq.p, q.a.size() * sizeof(double),
                             cudaMemcpyDeviceToHost));
        init::orthonormalize(q);
        JOFC_TRY(copy_sync(c, dq.p, q.a.data(), q.a.size() * sizeof(double),
                             cudaMemcpyHostToDevice));
      }
    }
    if (!done)
      return set_error(JOFC_ENUMERIC,
                       "subspace eigensolver did not converge within the iteration cap");
  }
  return JOFC_OK;
}

constexpr int kOmnibus = -2;

// cmds (proj/src/init.cpp:21-42) of modality `which` (-1: the modality
// average, kOmnibus: the imputed omnibus matrix) of the resident problem; x is
// n x d (m n x d for the omnibus) row-major.
int cmds_gpu(jofc_ctx* c, int which, size_t d, init::Mat& x) {
  using clk = std::chrono::steady_clock;
  const bool trace = std::getenv("JOFC_INIT_TRACE") != nullptr;
  const auto t_start = clk::now();
  double t_sync = 0.0;  // seconds spent waiting on the device inside the sweep loop
  int sweeps = 0;
  const Layout& L = c->lay;
  // which >= 0: modality, -1: modality average, kOmnibus: the m n x m n
  // imputed omnibus matrix
  const long long n = (which == kOmnibus) ? static_cast<long long>(L.m) * L.n : L.n;
  if (d < 1 || static_cast<long long>(d) > n)
    return set_error(JOFC_EINVAL, "cmds: dimension out of range");
  DevBuf<double> S, aux;
  JOFC_CUDA(S.ensure(static_cast<size_t>(n) * n));
  JOFC_CUDA(aux.ensure(static_cast<size_t>(n) + 1));
  JOFC_CUDA(cudaMemsetAsync(S.p, 0, static_cast<size_t>(n) * n * sizeof(double), c->stream));
  if (which == kOmnibus)
    init::omnibus_d2_kernel<<<static_cast<unsigned>(L.bpm), 256, 0, c->stream>>>(
        c->delta.p, L.n, L.nT, L.bpm, L.m, S.p);
  else
    init::dense_d2_kernel<<<static_cast<unsigned>(L.bpm), 256, 0, c->stream>>>(
        c->delta.p, n, L.nT, L.bpm, L.m, which, S.p);
  JOFC_CUDA(cudaGetLastError());
  init::row_sums_kernel<<<static_cast<unsigned>((n * 32 + 255) / 256), 256, 0, c->stream>>>(S.p, n,
                                                                                          aux.p);
  JOFC_CUDA(cudaGetLastError());
  std::vector<double> rs(n);
  JOFC_CUDA(cudaMemcpyAsync(rs.data(), aux.p, n * sizeof(double), cudaMemcpyDeviceToHost,
                            c->stream));
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  const double inv_n = 1.0 / static_cast<double>(n);
  double total = 0.0;
  for (long long i = 0; i < n; ++i) {
    total += rs[i];
    rs[i] *= inv_n;
  }
  total *= inv_n * inv_n;
  JOFC_CUDA(cudaMemcpyAsync(aux.p, rs.data(), n * sizeof(double), cudaMemcpyHostToDevice,
                            c->stream));
  DevBuf<double> fro2;
  JOFC_CUDA(fro2.ensure(1));
  JOFC_CUDA(cudaMemsetAsync(fro2.p, 0, sizeof(double), c->stream));
  init::double_center_kernel<<<static_cast<unsigned>(c->num_sms * 8), 256, 0, c->stream>>>(
      S.p, n, aux.p, total, fro2.p);
  JOFC_CUDA(cudaGetLastError());
  c->launches += 3;
  double f2 = 0.0;
  JOFC_CUDA(cudaMemcpyAsync(&f2, fro2.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  const double snorm = std::sqrt(f2);

  const size_t k = d;
  std::vector<double> values;
  init::Mat vecs;
  {
    const int rc = eigen_top_device(c, S.p, n, k, snorm, 320, values, vecs, sweeps, t_sync);
    if (rc) return rc;
  }
  if (trace)
    std::fprintf(stderr, "[init] cmds(%d) total %.3f s, %d sweeps, device wait %.3f s\n", which,
                 std::chrono::duration<double>(clk::now() - t_start).count(), sweeps, t_sync);
  x = init::Mat(n, d);
  for (size_t cc = 0; cc < d; ++cc) {
    const double sc = std::sqrt(std::max(values[cc], 0.0));  // Torgerson clamp
    for (long long r = 0; r < n; ++r) x(r, cc) = sc * vecs(r, cc);
  }
  init::center_columns(x);
  return JOFC_OK;
}

int require_full_problem(jofc_ctx* c) {
  int rc = require_problem(c);
  if (rc) return rc;
  if (c->world != 1)
    return set_error(JOFC_EINVAL, "initialisation needs an unsharded context (whole Delta)");
  return JOFC_OK;
}

}  // namespace

extern "C" {

int jofc_cmds(jofc_ctx* c, int modality, size_t d, double* x_out) {
  int rc = require_full_problem(c);
  if (rc) return rc;
  if (modality >= c->lay.m) return set_error(JOFC_EINVAL, "cmds: modality out of range");
  JOFC_CUDA(cudaSetDevice(c->device));
  init::Mat x;
  rc = cmds_gpu(c, modality, d, x);
  if (rc) return rc;
  JOFC_TRY(copy_sync(c, x_out, x.a.data(), x.a.size() * sizeof(double), cudaMemcpyDefault));
  return JOFC_OK;
}

int jofc_symmetric_top_eigenpairs_subspace(jofc_ctx* c, size_t n, const double* s, size_t k,
                                           double* values, double* vectors) {
  if (!c) return set_error(JOFC_EINVAL, "null context");
  if (!s || !values || !vectors) return set_error(JOFC_EINVAL, "null argument");
  if (k < 1 || k > n)
    return set_error(JOFC_EINVAL, "symmetric_top_eigenpairs_subspace: k out of range");
  if (k + 4 > static_cast<size_t>(init::kMaxP) && n > 64 && k + 4 < n)
    return set_error(JOFC_EINVAL, "symmetric_top_eigenpairs_subspace: k %zu above %d", k,
                     init::kMaxP - 4);
  JOFC_CUDA(cudaSetDevice(c->device));
  const long long nn = static_cast<long long>(n);
  DevBuf<double> S, rows;
  JOFC_CUDA(S.ensure(n * n));
  JOFC_CUDA(rows.ensure(n));
  JOFC_CUDA(cudaMemcpyAsync(S.p, s, n * n * sizeof(double), cudaMemcpyDefault, c->stream));
  init::row_sumsq_kernel<<<static_cast<unsigned>((nn * 32 + 255) / 256), 256, 0, c->stream>>>(
      S.p, nn, rows.p);
  JOFC_CUDA(cudaGetLastError());
  ++c->launches;
  std::vector<double> rs(n);
  JOFC_TRY(copy_sync(c, rs.data(), rows.p, n * sizeof(double), cudaMemcpyDeviceToHost));
  double f2 = 0.0;
  for (double v : rs) f2 += v;
  std::vector<double> vals;
  init::Mat vecs;
  int sweeps = 0;
  double t_sync = 0.0;
  JOFC_TRY(eigen_top_device(c, S.p, nn, k, std::sqrt(f2), 64, vals, vecs, sweeps, t_sync));
  std::vector<double> out(k * n);
  for (size_t cc = 0; cc < k; ++cc)
    for (size_t r = 0; r < n; ++r) out[cc * n + r] = vecs(r, cc);
  JOFC_TRY(copy_sync(c, values, vals.data(), k * sizeof(double), cudaMemcpyDefault));
  JOFC_TRY(copy_sync(c, vectors, out.data(), out.size() * sizeof(double), cudaMemcpyDefault));
  return JOFC_OK;
}

int jofc_init_imputed_cmds(jofc_ctx* c, size_t d, size_t dense_cap, double* x_out) {
  int rc = require_full_problem(c);
  if (rc) return rc;
  const size_t m = static_cast<size_t>(c->lay.m), n = static_cast<size_t>(c->lay.n);
  if (m * n > dense_cap)
    return set_error(JOFC_EINVAL, "imputed_omnibus_init: mn exceeds the dense cap");
  JOFC_CUDA(cudaSetDevice(c->device));
  init::Mat x;
  rc = cmds_gpu(c, kOmnibus, d, x);
  if (rc) return rc;
  // Configuration::from_stacked, then each block re-centred (init.cpp:111-114)
  std::vector<double> out(m * n * d);
  for (size_t l = 0; l < m; ++l) {
    init::Mat blk(n, d);
    std::copy(x.a.begin() + l * n * d, x.a.begin() + (l + 1) * n * d, blk.a.begin());
    init::center_columns(blk);
    std::copy(blk.a.begin(), blk.a.end(), out.begin() + l * n * d);
  }
  JOFC_TRY(copy_sync(c, x_out, out.data(), out.size() * sizeof(double), cudaMemcpyDefault));
  return JOFC_OK;
}

int jofc_init_averaged_procrustes(jofc_ctx* c, size_t d, double* x_out) {
  int rc = require_full_problem(c);
  if (rc) return rc;
  JOFC_CUDA(cudaSetDevice(c->device));
  init::Mat anchor;
  rc = cmds_gpu(c, -1, d, anchor);
  if (rc) return rc;
  init::center_columns(anchor);
  const size_t block = static_cast<size_t>(c->lay.n) * d;
  std::vector<double> out(static_cast<size_t>(c->lay.m) * block);
  for (int l = 0; l < c->lay.m; ++l) {
    init::Mat xl;
    rc = cmds_gpu(c, l, d, xl);
    if (rc) return rc;
    init::center_columns(xl);
    const init::Mat rot = init::procrustes(xl, anchor);
    std::copy(rot.a.begin(), rot.a.end(), out.begin() + l * block);
  }
  JOFC_TRY(copy_sync(c, x_out, out.data(), out.size() * sizeof(double), cudaMemcpyDefault));
  return JOFC_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- streaming ingest
// load_dissimilarities (proj/src/io.cpp:152-215) straight into the packed
// device layout: files are read in 128-row panels into two pinned host
// buffers, copied asynchronously, and packed by jofc_pack_kernel (upper
// part, raw) and jofc_ingest_combine_kernel (lower part: symmetry check and
// averaging against the mirror).  Entry checks (non-finite, negative) and the
// diagonal run on the host rows while the previous panel is on the device.
// Errors are reported in the reference's order and wording: parse errors of
// any file first (files are read in order), then per file: shape, size,
// entries, symmetry; then the diagonal warnings; then OmnibusProblem's own
// checks (proj/src/problem.cpp:8-32).
namespace {

struct InputCheck {
  std::string name;
  long long rows = 0, cols = 0;
  bool bad = false, nonfinite = false;
  long long bi = 0, bj = 0;
  double bv = 0.0;
  std::vector<std::pair<long long, double>> diag;  // nonzero diagonal entries
};

void check_row(InputCheck& ck, long long r, const double* v, long long cols) {
  if (!ck.bad)
    for (long long j = 0; j < cols; ++j) {
      const double x = v[j];
      if (!std::isfinite(x) || x < 0.0) {
        ck.bad = true;
        ck.nonfinite = !std::isfinite(x);
        ck.bi = r;
        ck.bj = j;
        ck.bv = x;
        break;
      }
    }
  if (r < cols && v[r] != 0.0) ck.diag.emplace_back(r, v[r]);
}

int load_files(jofc_ctx* c, const std::vector<std::string>& paths, int normalize) {
  using namespace ingest;
  if (paths.empty()) return set_error(JOFC_EINVAL, "load_dissimilarities: no input files");
  const std::string& p0 = paths.front();
  const bool binary = paths.size() == 1 && p0.size() >= 5 && p0.compare(p0.size() - 5, 5, ".jofc") == 0;
  c->has_problem = false;
  std::string err;
  std::FILE* bf = nullptr;
  struct Closer {
    std::FILE*& f;
    ~Closer() {
      if (f) std::fclose(f);
    }
  } closer{bf};
  JofcHeader hdr;
  std::unique_ptr<CsvRows> csv(new CsvRows);
  std::vector<double> row;
  long long m = 0, n = 0;
  if (binary) {
    if (!open_jofc(p0, bf, hdr, err)) return set_error(JOFC_EINVAL, "%s", err.c_str());
    if (hdr.d != 0)
      return set_error(JOFC_EINVAL, "'%s': file holds an embedding, not a problem", p0.c_str());
    m = hdr.m;
    n = hdr.n;
  } else {
    m = static_cast<long long>(paths.size());
    if (!csv->open(p0, err)) return set_error(JOFC_EINVAL, "%s", err.c_str());
    const int rc = csv->next(row, err);
    if (rc < 0) return set_error(JOFC_EINVAL, "%s", err.c_str());
    if (rc == 0) return set_error(JOFC_EINVAL, "'%s': empty matrix", p0.c_str());
    n = static_cast<long long>(row.size());
  }
  const bool device = m >= 1 && n >= 2;
  if (normalize && c->world > 1)
    return set_error(JOFC_EINVAL, "load with normalize needs an unsharded context");
  // panels of whole row blocks, ~64 MB each
  const long long panel_rows =
      std::max<long long>(1, (64LL << 20) / (8LL * std::max<long long>(n, 1)) / kRows) * kRows;
  DevBuf<unsigned long long> keys;
  IngestPanels& pin = c->ingest;
  if (device) {
    make_layout(c, static_cast<size_t>(m), static_cast<size_t>(n));
    JOFC_CUDA(c->delta.ensure(static_cast<size_t>(std::max<long long>(c->lay.local(), 1)) *
                              kBlockElems));
    JOFC_CUDA(pin.ensure(static_cast<size_t>(panel_rows) * n));
    JOFC_CUDA(keys.ensure(static_cast<size_t>(m)));
    JOFC_CUDA(cudaMemsetAsync(keys.p, 0xff, m * sizeof(unsigned long long), c->stream));
  }
  const Layout& L = c->lay;
  long long panels = 0;
  // ships host panel k (rows [r0, r0 + rows) of modality l; r0 a multiple of
  // 128) to the device and packs it row block by row block
  auto flush = [&](int k, int l, long long r0, long long rows) -> int {
    JOFC_CUDA(cudaMemcpyAsync(pin.stage[k].p, pin.host[k], static_cast<size_t>(rows) * n * sizeof(double),
                              cudaMemcpyHostToDevice, c->stream));
    JOFC_CUDA(cudaEventRecord(pin.copied[k], c->stream));
    for (long long rb = r0; rb < r0 + rows; rb += kRows) {
      const int B = static_cast<int>(rb / kRows);
      const double* st = pin.stage[k].p + (rb - r0) * n;
      PackParams pk{};
      pk.stage = st;
      pk.pitch = n;
      pk.r0 = rb;
      pk.c0 = 0;
      pk.n = n;
      pk.nT = L.nT;
      pk.bpm = L.bpm;
      pk.g_first = static_cast<long long>(l) * L.bpm + row_first(L.nT, B);
      pk.begin = L.begin;
      pk.end = L.end;
      pk.dst = c->delta.p;
      pk.norm = 0.0;
      pk.bad = nullptr;
      jofc_pack_kernel<<<static_cast<unsigned>(L.nT - 2 * B), 256, 0, c->stream>>>(pk);
      JOFC_CUDA(cudaGetLastError());
      CombineParams cb{};
      cb.stage = st;
      cb.n = n;
      cb.nT = L.nT;
      cb.bpm = L.bpm;
      cb.l = l;
      cb.Bp = B;
      cb.rows = static_cast<int>(std::min<long long>(kRows, r0 + rows - rb));
      cb.begin = L.begin;
      cb.end = L.end;
      cb.dst = c->delta.p;
      cb.asym_key = keys.p + l;
      jofc_ingest_combine_kernel<<<static_cast<unsigned>(2 * (B + 1)), 256, 0, c->stream>>>(cb);
      JOFC_CUDA(cudaGetLastError());
      c->launches += 2;
    }
    return JOFC_OK;
  };
  auto acquire = [&](int k) -> int {  // host panel k free again (its last copy landed)
    if (panels >= 2) JOFC_CUDA(cudaEventSynchronize(pin.copied[k]));
    return JOFC_OK;
  };

  std::vector<InputCheck> checks(static_cast<size_t>(m));
  for (long long l = 0; l < m; ++l) {
    InputCheck& ck = checks[l];
    ck.name = binary ? p0 : paths[l];
    if (binary) {
      ck.rows = ck.cols = n;
      const int fd = fileno(bf);
      std::vector<double> scratch;
      for (long long r0 = 0; r0 < n; r0 += panel_rows) {
        const long long rows = std::min<long long>(panel_rows, n - r0);
        const int k = static_cast<int>(panels & 1);
        int rc = acquire(k);
        if (rc) return rc;
        double* dst = pin.host[k];
        if (!device) {
          scratch.resize(static_cast<size_t>(rows) * n);
          dst = scratch.data();
        }
        // parallel positioned reads + entry checks, one slab of rows per thread
        const int nt = std::max(1, std::min(16, omp_get_max_threads()));
        std::vector<InputCheck> part(nt);
        int io_err = 0;
#pragma omp parallel num_threads(nt)
        {
          const int t = omp_get_thread_num();
          const long long a = rows * t / nt, b = rows * (t + 1) / nt;
          const size_t bytes = static_cast<size_t>(b - a) * n * sizeof(double);
          const off_t off = 20 + static_cast<off_t>((l * n + r0 + a) * n) * 8;
          size_t done = 0;
          while (done < bytes) {
            const ssize_t got = pread(fd, reinterpret_cast<char*>(dst + (a * n)) + done,
                                      bytes - done, off + static_cast<off_t>(done));
            if (got <= 0) {
#pragma omp atomic write
              io_err = 1;
              break;
            }
            done += static_cast<size_t>(got);
          }
          if (done == bytes)
            for (long long i = a; i < b; ++i) check_row(part[t], r0 + i, dst + i * n, n);
        }
        if (io_err) return set_error(JOFC_EINVAL, "'%s': truncated payload", p0.c_str());
        for (const InputCheck& pc : part) {  // merge in row order
          if (pc.bad && !ck.bad) {
            ck.bad = true;
            ck.nonfinite = pc.nonfinite;
            ck.bi = pc.bi;
            ck.bj = pc.bj;
            ck.bv = pc.bv;
          }
          ck.diag.insert(ck.diag.end(), pc.diag.begin(), pc.diag.end());
        }
        if (device && !ck.bad) {
          rc = flush(k, static_cast<int>(l), r0, rows);
          if (rc) return rc;
          ++panels;
        }
      }
      continue;
    }
    // CSV: file l (file 0 is open with its first row parsed)
    if (l > 0) {
      csv.reset(new CsvRows);
      if (!csv->open(paths[l], err)) return set_error(JOFC_EINVAL, "%s", err.c_str());
      const int rc = csv->next(row, err);
      if (rc < 0) return set_error(JOFC_EINVAL, "%s", err.c_str());
      if (rc == 0) return set_error(JOFC_EINVAL, "'%s': empty matrix", paths[l].c_str());
    }
    ck.cols = static_cast<long long>(row.size());
    const bool packable = device && ck.cols == n;
    long long filled = 0;
    int k = static_cast<int>(panels & 1);
    bool have = true;
    for (long long r = 0;; ++r) {
      if (!have) {
        const int rc = csv->next(row, err);
        if (rc < 0) return set_error(JOFC_EINVAL, "%s", err.c_str());
        if (rc == 0) break;
        if (static_cast<long long>(row.size()) != ck.cols)
          return set_error(JOFC_EINVAL, "'%s' line %zu: ragged row", paths[l].c_str(),
                           csv->line());
      }
      have = false;
      ck.rows = r + 1;
      check_row(ck, r, row.data(), ck.cols);
      if (packable && r < n && !ck.bad) {
        if (filled == 0) {
          k = static_cast<int>(panels & 1);
          const int rc = acquire(k);
          if (rc) return rc;
        }
        std::memcpy(pin.host[k] + static_cast<size_t>(filled) * n, row.data(), n * sizeof(double));
        if (++filled == panel_rows || r == n - 1) {
          const int rc = flush(k, static_cast<int>(l), r + 1 - filled, filled);
          if (rc) return rc;
          ++panels;
          filled = 0;
        }
      }
    }
  }
  // the reference's per-file validation, in file order
  std::vector<unsigned long long> hkeys(static_cast<size_t>(m), ~0ull);
  if (device) {
    JOFC_CUDA(cudaMemcpyAsync(hkeys.data(), keys.p, m * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, c->stream));
    JOFC_CUDA(cudaStreamSynchronize(c->stream));
  }
  for (long long l = 0; l < m; ++l) {
    const InputCheck& ck = checks[l];
    const char* nm = ck.name.c_str();
    if (ck.rows != ck.cols)
      return set_error(JOFC_EINVAL, "'%s': matrix is %lldx%lld, expected square", nm, ck.rows,
                       ck.cols);
    if (l > 0 && ck.rows != n)
      return set_error(JOFC_EINVAL, "'%s': size %lld differs from earlier modalities (%lld)", nm,
                       ck.rows, n);
    if (ck.bad && ck.nonfinite)
      return set_error(JOFC_EINVAL, "'%s': non-finite entry at (%lld,%lld)", nm, ck.bi, ck.bj);
    if (ck.bad)
      return set_error(JOFC_EINVAL, "'%s': negative entry %s at (%lld,%lld)", nm,
                       std::to_string(ck.bv).c_str(), ck.bi, ck.bj);
    if (hkeys[l] != ~0ull)
      return set_error(JOFC_EINVAL, "'%s': asymmetry beyond tolerance at (%llu,%llu)", nm,
                       hkeys[l] / static_cast<unsigned long long>(n),
                       hkeys[l] % static_cast<unsigned long long>(n));
    for (const auto& dg : ck.diag)
      std::fprintf(stderr, "warning: '%s' diagonal entry (%lld,%lld) = %g forced to 0\n", nm,
                   dg.first, dg.first, dg.second);
  }
  if (m == 0) return set_error(JOFC_EINVAL, "OmnibusProblem: at least one modality required");
  if (n < 2) return set_error(JOFC_EINVAL, "OmnibusProblem: need at least two objects");
  if (normalize) {  // Frobenius norm of each (averaged, zero-diagonal) modality
    const int grid = c->num_sms * 4;
    DevBuf<double> part;
    JOFC_CUDA(part.ensure(grid));
    std::vector<double> hp(grid);
    for (long long l = 0; l < m; ++l) {
      jofc_sumsq_kernel<<<grid, 256, 0, c->stream>>>(c->delta.p, l * L.bpm, L.bpm, part.p);
      JOFC_CUDA(cudaGetLastError());
      JOFC_TRY(copy_sync(c, hp.data(), part.p, grid * sizeof(double), cudaMemcpyDeviceToHost));
      double s = 0.0;
      for (double v : hp) s += v;
      const double norm = std::sqrt(2.0 * s);
      if (norm != 0.0) {
        jofc_scale_kernel<<<grid, 256, 0, c->stream>>>(c->delta.p, l * L.bpm, L.bpm, norm);
        JOFC_CUDA(cudaGetLastError());
      }
      c->launches += 2;
    }
  }
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  c->has_problem = true;
  return JOFC_OK;
}

}  // namespace

extern "C" int jofc_problem_shape(jofc_ctx* c, size_t* m, size_t* n) {
  const int rc = require_problem(c);
  if (rc) return rc;
  if (m) *m = static_cast<size_t>(c->lay.m);
  if (n) *n = static_cast<size_t>(c->lay.n);
  return JOFC_OK;
}

extern "C" int jofc_load_problem_files(jofc_ctx* c, size_t count, const char* const* paths,
                                       int normalize) {
  if (!c) return set_error(JOFC_EINVAL, "null context");
  if (count && !paths) return set_error(JOFC_EINVAL, "null path list");
  std::vector<std::string> ps;
  for (size_t i = 0; i < count; ++i) {
    if (!paths[i]) return set_error(JOFC_EINVAL, "null path %zu", i);
    ps.emplace_back(paths[i]);
  }
  JOFC_CUDA(cudaSetDevice(c->device));
  return load_files(c, ps, normalize);
}
