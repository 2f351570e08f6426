// jofc_capi.cu -- host side of libjofc_gpu.so: the C ABI in include/jofc_gpu.h.
//
// Owns the device state of one solve context: the packed Delta shard, the
// ping-pong configuration buffers, the product/fidelity exchange buffer, the
// control block, and the launch sequence
//
//     for t = 0 .. max_it:   pass(t) -> [all-reduce hook] -> epilogue(t)
//     (peer exchange:        pass(t) -> peer mix(t) -> peer decide(t), capi_peer.cu)
//     (small, one GPU:       one jofc_solve_persistent_kernel launch for all t)
//
// enqueued without host synchronisation: termination (the reference's
// decrease < eps rule, proj/src/solver.cpp:138-143) is decided on the device
// and later launches exit at entry once the control block says done.
#include <cuda_runtime.h>
#include <omp.h>
#include <unistd.h>

#include <chrono>

#include <algorithm>
#include <climits>
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
#include "jofc_weights.h"

#include "capi_internal.h"

using namespace jofc_gpu;
using namespace jofc_gpu::capi;

namespace jofc_gpu {
namespace capi {

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

int delta_sumsq(jofc_ctx* c) {
  const Layout& L = c->lay;
  const int G = c->num_sms;
  JOFC_CUDA(c->sumsq.ensure(L.m));
  JOFC_CUDA(c->sumsq_part.ensure(static_cast<size_t>(G) * L.m));
  jofc_modality_sumsq_kernel<<<dim3(G, L.m), 256, 0, c->stream>>>(c->delta.p, L.bpm, L.begin,
                                                                   L.end, c->sumsq_part.p);
  JOFC_CUDA(cudaGetLastError());
  jofc_fold_partials_kernel<<<1, 128, 0, c->stream>>>(c->sumsq_part.p, G, L.m, c->sumsq.p);
  JOFC_CUDA(cudaGetLastError());
  c->launches += 2;
  return JOFC_OK;
}

bool rho_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("JOFC_FIDELITY");
    return !(e && std::string(e) == "direct");
  }();
  return v;
}

int require_problem(jofc_ctx* c) {
  if (!c) return set_error(JOFC_EINVAL, "null context");
  if (!c->has_problem) return set_error(JOFC_EINVAL, "no problem uploaded (jofc_set_problem)");
  return JOFC_OK;
}

// Estimated pass-kernel cost of one block, in units of an interior block: masked
// blocks (diagonal-crossing or padded) +0.1, the first block a CTA processes
// of a row band +band_cost() (flush of the row sums, X row-block staging, two
// CTA barriers; 1.0 measured best at C3/C4/C5 among 0, 0.5, 1, 1.5, 2, 4, 8).
// Experiment switches, read once per process: JOFC_DIAG (pass-kernel timing
// modes; results are wrong when set), JOFC_FUSE_EPI_N (fused-epilogue limit).
int diag_mode() {
  static const int v = [] {
    const char* e = std::getenv("JOFC_DIAG");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

long long fuse_epilogue_max_n() {
  static const long long v = [] {
    const char* e = std::getenv("JOFC_FUSE_EPI_N");
    return e ? std::atoll(e) : kFuseEpilogueMaxN;
  }();
  return v;
}

// Chunk length of the synchronous solves' early stop (0: off); JOFC_STOP_CHUNK
// overrides kStopChunk (experiments).
size_t stop_chunk() {
  static const size_t v = [] {
    const char* e = std::getenv("JOFC_STOP_CHUNK");
    return e ? static_cast<size_t>(std::atoll(e)) : kStopChunk;
  }();
  return v;
}

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

}  // namespace capi
}  // namespace jofc_gpu


namespace {

double* exchange(jofc_ctx* c) {
  const size_t need = static_cast<size_t>(c->lay.m) * c->lay.n_pad * c->d + 1;
  return (c->ext_P && c->ext_cap >= need) ? c->ext_P : c->P.p;
}

}  // namespace

double* jofc_gpu::capi::xbuf(jofc_ctx* c, int k) {
  if (c->peer.active) return c->peer.slab + c->peer.x_off[k];
  return k ? c->x1.p : c->x0.p;
}

namespace {

size_t fid_slot(const jofc_ctx* c) { return static_cast<size_t>(c->lay.m) * c->lay.n_pad * c->d; }

template <int D>
int setup_pass(int device) {
  JOFC_CUDA(ensure_smem_attr(jofc_pass_kernel<D>, static_cast<int>(sizeof(PassSmem<D>)), device));
  return JOFC_OK;
}

template <int D>
int launch_pass(jofc_ctx* c, const PassParams& pp) {
  int rc = setup_pass<D>(c->device);
  if (rc) return rc;
  jofc_pass_kernel<D><<<c->pass_grid, kPassThreads, sizeof(PassSmem<D>), c->stream>>>(pp);
  JOFC_CUDA(cudaGetLastError());
  return JOFC_OK;
}

template <int D>
int setup_for(jofc_ctx* c) {
  return setup_pass<D>(c->device);
}

// 256-thread identity-form epilogue for m <= 8 (JOFC_WIDE_SMALL=0: the
// 1024-thread form, comparisons)
bool wide_small_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("JOFC_WIDE_SMALL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int D>
int launch_epi(jofc_ctx* c, const EpiParams& ep) {
  if (ep.rho && ep.m <= kWideSmallMaxM && wide_small_enabled())
    jofc_epilogue_wide_kernel<D, kWideSmallThreads><<<c->rho_grid, kWideSmallThreads, 0, c->stream>>>(ep);
  else if (ep.rho && ep.m <= kWideMaxM)
    jofc_epilogue_wide_kernel<D><<<c->rho_grid, kWideThreads, 0, c->stream>>>(ep);
  else
    jofc_epilogue_kernel<D><<<c->epi_grid, kEpiThreads, 0, c->stream>>>(ep);
  JOFC_CUDA(cudaGetLastError());
  return JOFC_OK;
}

template <int D>
int launch_rho_decide(jofc_ctx* c, const EpiParams& ep) {
  jofc_rho_decide_kernel<D><<<1, 32, 0, c->stream>>>(ep, static_cast<unsigned>(c->rho_grid));
  JOFC_CUDA(cudaGetLastError());
  return JOFC_OK;
}




}  // namespace

int jofc_gpu::capi::pass_for_d(jofc_ctx* c, const PassParams& pp) {
  JOFC_DISPATCH_D(c->d, launch_pass, c, pp);
}

namespace {

// The whole solve as one cooperative launch (jofc_solve_persistent_kernel).
template <int D>
int launch_persistent(jofc_ctx* c, const PassParams& pp) {
  JOFC_CUDA(ensure_smem_attr(jofc_solve_persistent_kernel<D>,
                             static_cast<int>(sizeof(PassSmem<D>)), c->device));
  PassParams arg = pp;
  void* args[] = {&arg};
  JOFC_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(jofc_solve_persistent_kernel<D>),
                                        dim3(c->pass_grid), dim3(kPassThreads), args,
                                        sizeof(PassSmem<D>), c->stream));
  return JOFC_OK;
}

int persistent_for_d(jofc_ctx* c, const PassParams& pp) {
  JOFC_DISPATCH_D(c->d, launch_persistent, c, pp);
}

// Single-launch solves for problems whose pass is short (JOFC_PERSISTENT=0/1
// forces it off / on for experiments).
bool use_persistent(const jofc_ctx* c) {
  static const char* env = std::getenv("JOFC_PERSISTENT");
  if (env && env[0] == '0') return false;
  if (env && env[0] == '1') return true;
  return c->lay.local() <= kPersistentMaxBlocks;
}

int setup_for_d(jofc_ctx* c) { JOFC_DISPATCH_D(c->d, setup_for, c); }
int epi_for_d(jofc_ctx* c, const EpiParams& ep) { JOFC_DISPATCH_D(c->d, launch_epi, c, ep); }
int rho_decide_for_d(jofc_ctx* c, const EpiParams& ep) {
  JOFC_DISPATCH_D(c->d, launch_rho_decide, c, ep);
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
  if (L.local() <= NG) {  // one block per CTA (cost cuts would pair some up)
    for (int i = 0; i <= NG; ++i) b[i] = std::min(L.end, L.begin + i);
    JOFC_CUDA(c->bounds.ensure(NG + 1));
    JOFC_TRY(copy_sync(c, c->bounds.p, b.data(), (NG + 1) * sizeof(long long),
                       cudaMemcpyHostToDevice));
    c->bounds_key = key;
    return JOFC_OK;
  }
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
  const bool peer = c->peer.active;
  const bool resize = !peer && ((d != c->d) || !c->x0.p || c->x0.n < cfg);
  c->d = d;
  if (!peer) {  // (peer exchange: X and P live in the context's slab)
    JOFC_CUDA(c->x0.ensure(cfg));
    JOFC_CUDA(c->x1.ensure(cfg));
    if (c->ext_P && c->ext_cap >= cfg + 1) {
      c->P.release();
    } else {
      JOFC_CUDA(c->P.ensure(cfg + 1));
    }
  }
  c->pass_grid = static_cast<int>(std::max<long long>(1, std::min<long long>(c->num_sms, L.local())));
  c->epi_grid = static_cast<int>((L.n + kEpiThreads - 1) / kEpiThreads);
  JOFC_CUDA(c->fid_part.ensure(2 * static_cast<size_t>(c->pass_grid)));
  JOFC_TRY(pass_bounds(c));
  // (the persistent kernel keeps one commensurability partial per pass CTA)
  JOFC_CUDA(c->com_part.ensure(std::max(c->epi_grid, c->pass_grid)));
  JOFC_CUDA(c->trace.ensure(max_it + 1));
  if (!c->ctrl.p) {  // (zeroed once: the evaluation counter lives in it)
    JOFC_CUDA(c->ctrl.ensure(1));
    JOFC_CUDA(cudaMemsetAsync(c->ctrl.p, 0, sizeof(Control), c->stream));
  }
  JOFC_CUDA(c->consts.ensure(3 * static_cast<size_t>(L.m) * L.m + L.m));
  if (resize) {
    JOFC_CUDA(cudaMemsetAsync(c->x0.p, 0, cfg * sizeof(double), c->stream));
    JOFC_CUDA(cudaMemsetAsync(c->x1.p, 0, cfg * sizeof(double), c->stream));
  }
  // (peer exchange: the protocol leaves the next solve's P region zeroed)
  if (!peer) JOFC_CUDA(cudaMemsetAsync(exchange(c), 0, (cfg + 1) * sizeof(double), c->stream));
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
}  // namespace

int jofc_gpu::capi::prepare_solve(jofc_ctx* c, const jofc_weights* spec, size_t d,
                                  const double* x0, double eps, size_t max_it, PassParams* ppo,
                                  EpiParams* epo) {
  int rc = require_problem(c);
  if (rc) return rc;
  if (d < 1 || d > static_cast<size_t>(kMaxD))
    return set_error(JOFC_EINVAL, "dim %zu unsupported (1..%d)", d, kMaxD);
  if (!(eps > 0.0)) return set_error(JOFC_EINVAL, "SolveOptions: eps must be positive");
  if (!x0) return set_error(JOFC_EINVAL, "null configuration");
  if (max_it >= static_cast<size_t>(INT_MAX))
    return set_error(JOFC_EINVAL, "max_iterations %zu too large (< %d)", max_it, INT_MAX);
  const Layout& L = c->lay;
  HostWeights hw;
  std::string msg;
  rc = build_weights(spec, static_cast<size_t>(L.m), static_cast<size_t>(L.n), &hw, &msg);
  if (rc) return set_error(rc, "%s", msg.c_str());
  if (c->peer.active) {
    if (c->peer.pending) {  // the previous solve fixes this one's P parity
      Control prev;
      finish_solve(c, &prev);
    }
    JOFC_TRY(peer_check(c));
  }
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
  rc = upload_config(c, x0, xbuf(c, 0));
  if (rc) return rc;

  Control h;
  std::memset(&h, 0, sizeof(Control));
  h.max_it = static_cast<int>(max_it);
  h.eps = eps;
  if (c->peer.active) {
    h.epoch = ++c->peer.epoch;
    c->peer.pending = true;
  }
  const double mn = static_cast<double>(L.m) * static_cast<double>(L.n);
  h.pairs = mn * (mn - 1.0) / 2.0;
  jofc_control_init_kernel<<<1, 1, 0, c->stream>>>(c->ctrl.p, h);
  JOFC_CUDA(cudaGetLastError());
  ++c->launches;

  PassParams pp{};
  pp.delta = c->delta.p;
  pp.x0 = xbuf(c, 0);
  pp.x1 = xbuf(c, 1);
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
  pp.diag = diag_mode();

  EpiParams ep{};
  ep.x0 = xbuf(c, 0);
  ep.x1 = xbuf(c, 1);
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
  ep.mix_lo = 0;
  ep.mix_hi = L.n;
  if (c->nccl_comm) {  // this rank mixes its own row chunk (capi_nccl.cu)
    JOFC_TRY(nccl_check(c));
    const long long rows = nccl_chunk_rows(c);
    ep.mix_lo = std::min<long long>(L.n, rows * c->rank);
    ep.mix_hi = std::min<long long>(L.n, rows * (c->rank + 1));
  }

  // Small problems on one GPU: the pass kernel's last CTA runs the epilogue
  // too (one launch per iteration instead of two).  The threshold keeps the
  // one-CTA epilogue below the cost of a second launch.
  pp.fuse_epilogue = (c->world == 1 && !c->nccl_comm && L.n <= fuse_epilogue_max_n()) ? 1 : 0;
  // Identity-form fidelity (jofc_kernels.cuh, rho_decide): the one-GPU route
  // with a separate epilogue kernel.  (The fused and persistent epilogues,
  // the NCCL, hook and peer exchanges keep the per-pair sum.)
  if (rho_enabled() && c->fidelity_form == JOFC_FIDELITY_AUTO &&
      (c->world == 1 || c->nccl_comm) && !c->peer.active && !pp.fuse_epilogue && c->sumsq.p) {
    const size_t K = 1 + static_cast<size_t>(L.m) * (d + 3);
    const int wthreads = wide_small_enabled() ? wide_threads(L.m) : kWideThreads;
    const long long wide_objs = static_cast<long long>(wthreads / 32 / L.m) * 32;
    // (one wave of resident CTAs: 2048 / wthreads per SM)
    const long long max_ctas = static_cast<long long>(c->num_sms) * (2048 / wthreads);
    c->rho_grid = L.m <= kWideMaxM
                      ? static_cast<int>(std::min<long long>(max_ctas,
                                                             (L.n + wide_objs - 1) / wide_objs))
                      : c->epi_grid;
    JOFC_CUDA(c->rho_part.ensure((static_cast<size_t>(c->rho_grid) + 1) * K));
    ep.rho = 1;
    ep.rho_split = c->nccl_comm ? 1 : 0;
    ep.rho_partials = c->rho_part.p;
    ep.sumsq = c->sumsq.p;
    ep.within = c->consts.p + 3 * mm;
  }
  pp.rho = ep.rho;
  pp.epi = ep;
  *ppo = pp;
  *epo = ep;
  return JOFC_OK;
}

namespace {

int enqueue_solve(jofc_ctx* c, const jofc_weights* spec, size_t d, const double* x0, double eps,
                  size_t max_it, std::vector<cudaEvent_t>* events, bool early_stop = false) {
  PassParams pp;
  EpiParams ep;
  int rc = prepare_solve(c, spec, d, x0, eps, max_it, &pp, &ep);
  if (rc) return rc;
  const Layout& L = c->lay;
  const bool fused = pp.fuse_epilogue != 0;

  // Single GPU, no per-launch events: replay a captured CUDA graph of the
  // whole 2(max_it + 1)-kernel sequence (kernel parameters only hold buffer
  // pointers; everything iteration-dependent lives in the control block).
  // (the NCCL exchange is captured with the kernels: its calls are on the
  // context stream with fixed buffers per iteration parity)
  const bool nccl_x = c->nccl_comm != nullptr;
  const bool graphable = c->use_graphs && (c->world == 1 || nccl_x) && !c->peer.active &&
                         !events && !c->profiling;
  // iteration t's collectives: the reduce-scatter after its pass, the
  // all-gather of X_{t+1} after its epilogue
  auto exchange_pre = [&]() -> int {
    return nccl_x ? nccl_reduce(c, exchange(c), fid_slot(c)) : JOFC_OK;
  };
  // (identity-form fidelity: the ranks' folded sums ride in the all-gather
  // group, then the decision kernel)
  const size_t rho_k = 1 + static_cast<size_t>(L.m) * (d + 3);
  double* rho_sums = ep.rho_split ? ep.rho_partials + static_cast<size_t>(c->rho_grid) * rho_k
                                  : nullptr;
  auto exchange_post = [&](size_t t) -> int {
    if (!nccl_x) return JOFC_OK;
    JOFC_TRY(nccl_gather(c, xbuf(c, static_cast<int>((t + 1) & 1)), rho_sums, rho_k));
    if (rho_sums) JOFC_TRY(rho_decide_for_d(c, ep));
    return JOFC_OK;
  };
  if (early_stop && !c->stop_flag) {
    JOFC_CUDA(cudaMallocHost(&c->stop_flag, 2 * sizeof(int)));
    for (int k = 0; k < 2; ++k)
      JOFC_CUDA(cudaEventCreateWithFlags(&c->stop_ev[k], cudaEventDisableTiming));
  }
  // early stop: after enqueuing chunk `ch` (0-based) of iterations, send its
  // done flag to the host and look at the previous chunk's; true = stop
  auto chunk_done = [&](size_t ch, bool* stop) -> int {
    const int k = static_cast<int>(ch & 1);
    JOFC_CUDA(cudaMemcpyAsync(&c->stop_flag[k], &c->ctrl.p->done, sizeof(int),
                              cudaMemcpyDeviceToHost, c->stream));
    JOFC_CUDA(cudaEventRecord(c->stop_ev[k], c->stream));
    *stop = false;
    if (ch >= 1) {
      JOFC_CUDA(cudaEventSynchronize(c->stop_ev[k ^ 1]));
      *stop = c->stop_flag[k ^ 1] != 0;
    }
    return JOFC_OK;
  };
  if (graphable && !nccl_x && use_persistent(c)) {
    // (a cooperative launch is refused when the SMs are shared, e.g. under
    // MPS: the per-iteration launches below then run the solve)
    if (persistent_for_d(c, pp) == JOFC_OK) {
      ++c->launches;
      c->max_it_enqueued = max_it;
      return JOFC_OK;
    }
    cudaGetLastError();
  }
  if (graphable) {
    // one graph of the whole sequence, or (early stop) of one chunk replayed
    // until the device says done: later iterations are no-ops on the device
    // anyway (the control block), this stops paying their launches
    size_t per_graph = early_stop ? std::min(stop_chunk(), max_it + 1) : max_it + 1;
    // a chunk graph replayed for later iterations must keep their X-buffer
    // parity (the all-gather targets are baked in): even length
    if (nccl_x && early_stop && per_graph < max_it + 1 && (per_graph & 1)) ++per_graph;
    std::vector<uintptr_t> key = {c->d, per_graph, static_cast<uintptr_t>(c->pass_grid),
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
                                  static_cast<uintptr_t>(pp.diag),
                                  static_cast<uintptr_t>(pp.fuse_epilogue),
                                  reinterpret_cast<uintptr_t>(c->nccl_comm),
                                  static_cast<uintptr_t>(ep.mix_lo),
                                  static_cast<uintptr_t>(ep.mix_hi),
                                  static_cast<uintptr_t>(ep.rho),
                                  reinterpret_cast<uintptr_t>(ep.rho_partials),
                                  reinterpret_cast<uintptr_t>(ep.sumsq)};
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
      for (size_t t = 0; t < per_graph && !lrc; ++t) {
        lrc = pass_for_d(c, pp);
        if (!lrc) lrc = exchange_pre();
        if (!lrc && !fused) lrc = epi_for_d(c, ep);
        if (!lrc) lrc = exchange_post(t);
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
    for (size_t ch = 0; ch * per_graph <= max_it; ++ch) {
      JOFC_CUDA(cudaGraphLaunch(it->second, c->stream));
      c->launches += (fused ? 1 : rho_sums ? 3 : 2) * per_graph;  // (ours; NCCL's not counted)
      if (early_stop) {
        bool stop = false;
        JOFC_TRY(chunk_done(ch, &stop));
        if (stop) break;
      }
    }
    c->max_it_enqueued = max_it;
    return JOFC_OK;
  }

  for (size_t t = 0; t <= max_it; ++t) {
    if (early_stop && t > 0 && t % stop_chunk() == 0) {
      bool stop = false;
      JOFC_TRY(chunk_done(t / stop_chunk() - 1, &stop));
      if (stop) break;
    }
    if (events) JOFC_CUDA(cudaEventRecord((*events)[t], c->stream));
    cudaEvent_t pe1 = nullptr;
    rc = prof_begin(c, &pe1);
    if (rc) return rc;
    if (c->peer.active) {  // pass + peer mix + decide (jofc_peer.cuh)
      for (int stage = 0; stage < 3; ++stage) {
        JOFC_TRY(peer_stage(c, pp, t, stage));
        if (stage == 0 && pe1) JOFC_CUDA(cudaEventRecord(pe1, c->stream));
      }
      continue;
    }
    rc = pass_for_d(c, pp);
    if (rc) return rc;
    if (pe1) JOFC_CUDA(cudaEventRecord(pe1, c->stream));
    ++c->launches;
    if (nccl_x) {
      JOFC_TRY(exchange_pre());
    } else if (c->world > 1) {
      if (!c->allreduce)
        return set_error(JOFC_ECOMM, "sharded context (world %d) without an all-reduce hook",
                         c->world);
      if (c->allreduce(exchange(c), fid_slot(c) + 1, c->stream, c->allreduce_user) != 0)
        return set_error(JOFC_ECOMM, "all-reduce hook failed at iteration %zu", t);
    }
    if (!fused) {
      rc = epi_for_d(c, ep);
      if (rc) return rc;
      ++c->launches;
    }
    JOFC_TRY(exchange_post(t));
    if (rho_sums) ++c->launches;
  }
  if (events) JOFC_CUDA(cudaEventRecord((*events)[max_it + 1], c->stream));
  c->max_it_enqueued = max_it;
  return JOFC_OK;
}

}  // namespace

// Synchronise, then fetch the control block; maps device status to errors.
int jofc_gpu::capi::finish_solve(jofc_ctx* c, Control* out) {
  JOFC_CUDA(cudaMemcpyAsync(c->ctrl_host, c->ctrl.p, sizeof(Control), cudaMemcpyDeviceToHost,
                            c->stream));
  if (c->nccl_comm)
    JOFC_TRY(nccl_wait(c));  // polls the communicator's async error meanwhile
  else
    JOFC_CUDA(cudaStreamSynchronize(c->stream));
  *out = *c->ctrl_host;
  if (c->peer.active && c->peer.pending) {
    // the last evaluated iteration T left P region (T + phase) & 1 dirty and
    // zeroed the other one: the next solve starts on the clean region
    const int last = (out->status == 2) ? out->err_iter : out->iterations;
    c->peer.phase = (c->peer.phase + last + 1) & 1;
    c->peer.pending = false;
  }
  if (out->status == 3 || out->status == 4) {
    peer_release(c);  // the group's exchange state is unknown: attach again
    if (out->status == 4)
      return set_error(JOFC_ECOMM,
                       "peer exchange: the ranks disagree on the solve count (epoch mismatch at "
                       "iteration %d); re-attach the group",
                       out->err_iter);
    return set_error(JOFC_ECOMM, "peer exchange: a rank did not arrive within 20 s (iteration %d)",
                     out->err_iter);
  }
  if (out->status == 2) {
    if (out->err_iter == 0)
      return set_error(JOFC_ENUMERIC, "embed: non-finite stress at the initial configuration");
    return set_error(JOFC_ENUMERIC, "embed: non-finite stress at iteration %d", out->err_iter);
  }
  if (!out->done) return set_error(JOFC_ECUDA, "solve did not terminate (internal)");
  return JOFC_OK;
}

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
  peer_release(c);
  nccl_release(c);
  for (DevBuf<double>* b : {&c->delta, &c->x0, &c->x1, &c->P, &c->fid_part, &c->com_part,
                            &c->trace, &c->consts, &c->oos_x, &c->oos_delta, &c->oos_y0,
                            &c->oos_y1, &c->oos_part, &c->oos_trace, &c->oos_delta_t,
                            &c->oos_delta_p})
    b->release();
  c->ctrl.release();
  c->up_bad.release();
  c->ingest_keys.release();
  c->oos_st.release();
  for (auto& e : c->prof_events) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
  if (c->ctrl_host) cudaFreeHost(c->ctrl_host);
  c->ingest.release();
  if (c->stop_flag) cudaFreeHost(c->stop_flag);
  for (auto& e : c->stop_ev)
    if (e) cudaEventDestroy(e);
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

int jofc_stress_evaluations(jofc_ctx* c, uint64_t* out) {
  if (!c || !out) return set_error(JOFC_EINVAL, "null argument");
  *out = 0;
  if (!c->ctrl.p) return JOFC_OK;
  JOFC_CUDA(cudaSetDevice(c->device));
  unsigned long long v = 0;
  JOFC_CUDA(cudaMemcpyAsync(&v, &c->ctrl.p->evals, sizeof(v), cudaMemcpyDeviceToHost, c->stream));
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  *out = static_cast<uint64_t>(v);
  return JOFC_OK;
}

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
  JOFC_CUDA(cudaSetDevice(c->device));
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  peer_release(c);  // a new shard needs a new problem and a new peer group
  nccl_release(c);  // ... and a new communicator
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
  const NvtxScope nvtx_scope("jofc_set_problem");
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

  // Frobenius norms over the full dense matrix (OmnibusProblem::normalized,
  // proj/src/problem.cpp:34-42): row sums on all host threads, then added in
  // row order -- deterministic and identical on every rank of a sharded
  // context; it differs from the reference's one serial n^2 sum only by
  // rounding (the serial loop took ~0.5 s per C3 modality).
  std::vector<double> norms(m, 0.0);
  if (normalize)
    for (size_t l = 0; l < m; ++l) {
      const double* dl = delta[l];
      std::vector<double> rows(n);
#pragma omp parallel for schedule(static)
      for (long long i = 0; i < static_cast<long long>(n); ++i) {
        double s = 0.0;
        const double* row = dl + static_cast<size_t>(i) * n;
        for (size_t j = 0; j < n; ++j) s += row[j] * row[j];
        rows[static_cast<size_t>(i)] = s;
      }
      double s = 0.0;
      for (double v : rows) s += v;
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
  // (device staging shared with file ingest, kept across uploads: no
  // cudaMalloc / synchronising cudaFree per call)
  DevBuf<double>* stage = c->ingest.stage;
  DevBuf<int>& bad = c->up_bad;
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
  JOFC_TRY(delta_sumsq(c));
  int hbad = 0;
  JOFC_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  if (hbad) return set_error(JOFC_EINVAL, "OmnibusProblem: delta has a non-finite or negative entry");
  c->has_problem = true;
  return JOFC_OK;
}

int jofc_set_problem_features(jofc_ctx* c, size_t m, size_t n, size_t p, const double* feats) {
  const NvtxScope nvtx_scope("jofc_set_problem_features");
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
  JOFC_TRY(delta_sumsq(c));
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  f.release();
  c->has_problem = true;
  return JOFC_OK;
}

int jofc_fjofc_enqueue(jofc_ctx* c, const jofc_weights* spec, size_t d, const double* x0,
                       double eps, size_t max_it) {
  const NvtxScope nvtx_scope("jofc_fjofc_enqueue");
  if (!c) return set_error(JOFC_EINVAL, "null context");
  JOFC_CUDA(cudaSetDevice(c->device));
  return enqueue_solve(c, spec, d, x0, eps, max_it, nullptr);
}

int jofc_fetch_result(jofc_ctx* c, double* x_out, double* trace_out, size_t* iterations,
                      int* converged) {
  const NvtxScope nvtx_scope("jofc_fetch_result");
  int rc = require_problem(c);
  if (rc) return rc;
  if (!c->ctrl.p) return set_error(JOFC_EINVAL, "fetch: no solve was enqueued");
  Control h;
  rc = finish_solve(c, &h);
  if (rc) return rc;
  if (x_out) {
    rc = download_config(c, xbuf(c, h.iterations & 1), x_out);
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
  const NvtxScope nvtx_scope("jofc_fjofc_embed");
  if (!c) return set_error(JOFC_EINVAL, "null context");
  JOFC_CUDA(cudaSetDevice(c->device));
  // step_seconds: two events around the whole solve (it keeps the CUDA-graph
  // and single-launch routes; per-iteration events would force stream
  // launches).  Every entry is the solve's mean device time per iteration --
  // one fused pass + epilogue, i.e. the transform together with the stress
  // of its input iterate, which the fused kernel cannot time apart
  // (the reference times fast_step alone, proj/src/solver.cpp:123-127).
  cudaEvent_t ev[2] = {nullptr, nullptr};
  if (step_seconds)
    for (auto& e : ev) JOFC_CUDA(cudaEventCreate(&e));
  if (ev[0]) JOFC_CUDA(cudaEventRecord(ev[0], c->stream));
  int rc = enqueue_solve(c, spec, d, x0, eps, max_it, nullptr, /*early_stop=*/stop_chunk() > 0);
  if (!rc && ev[1]) rc = cudaEventRecord(ev[1], c->stream) == cudaSuccess
                             ? JOFC_OK
                             : set_error(JOFC_ECUDA, "event record failed");
  size_t its = 0;
  if (!rc) rc = jofc_fetch_result(c, x_out, trace_out, &its, converged);
  if (!rc && iterations) *iterations = its;
  if (!rc && step_seconds && its > 0) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev[0], ev[1]);
    const double per = ms * 1e-3 / static_cast<double>(its + 1);  // its + 1 passes
    for (size_t t = 0; t < its; ++t) step_seconds[t] = per;
  }
  for (auto& e : ev)
    if (e) cudaEventDestroy(e);
  return rc;
}

int jofc_set_oos_route(jofc_ctx* c, int route) {
  if (!c) return set_error(JOFC_EINVAL, "null context");
  if (route != JOFC_OOS_AUTO && route != JOFC_OOS_PERSISTENT && route != JOFC_OOS_PER_UPDATE)
    return set_error(JOFC_EINVAL, "oos route %d unknown (0 auto, 1 persistent, 2 per update)",
                     route);
  c->oos_route = route;
  return JOFC_OK;
}

int jofc_set_fidelity_form(jofc_ctx* c, int form) {
  if (!c) return set_error(JOFC_EINVAL, "null context");
  if (form != JOFC_FIDELITY_AUTO && form != JOFC_FIDELITY_DIRECT)
    return set_error(JOFC_EINVAL, "fidelity form %d unknown (0 auto, 1 direct)", form);
  c->fidelity_form = form;
  return JOFC_OK;
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
  rc = download_config(c, xbuf(c, 1), x_next);
  if (rc) return rc;
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  return JOFC_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- out-of-sample
namespace {

// Kernels of the out-of-sample loop: 3 = one fused step kernel per update
// (jofc_oos_step_kernel, default); 1 = pass (warp per point, lanes over rows)
// + update kernel, the round-2 pair; 2 = the lanes-over-points pass on the
// transposed delta + update kernel.  JOFC_OOS_KERNEL=1/2 for comparisons.
// 4 (default) = the persistent solve (jofc_oos_solve_kernel: one launch per
// batch) where its shared-memory plan fits, else 3.
int oos_kernel_version() {
  static const int v = [] {
    const char* e = std::getenv("JOFC_OOS_KERNEL");
    return (e && e[0] >= '1' && e[0] <= '3') ? e[0] - '0' : 4;
  }();
  return v;
}

// Slices of the in-sample range per (point group, modality): kOosSplits, or
// JOFC_OOS_SPLITS (experiments).
long long oos_splits() {
  static const long long v = [] {
    const char* e = std::getenv("JOFC_OOS_SPLITS");
    return e ? std::max(1LL, std::atoll(e)) : static_cast<long long>(kOosSplits);
  }();
  return v;
}

template <int D>
int oos_launch(jofc_ctx* c, const OosParams& op, int steps) {
  const bool v2 = oos_kernel_version() == 2;
  const bool fused = oos_kernel_version() >= 3;  // (4: the persistent solve did not apply)
  // v1: 4 slices of the in-sample range (measured best at C5 among 2..16)
  const dim3 pg((op.k + kOosWarps - 1) / kOosWarps, op.m,
                static_cast<unsigned>(std::min<long long>(oos_splits(), std::max<long long>(1, op.n / 256))));
  // v2: (point group, modality) x slices -- one wave of resident CTAs
  constexpr int smem2 = oos2_smem_bytes<D>();
  int per_sm = 1;
  if (v2) {
    JOFC_CUDA(ensure_smem_attr(jofc_oos_pass2_kernel<D>, smem2, c->device));
    JOFC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jofc_oos_pass2_kernel<D>,
                                                            kOos2Warps * 32, smem2));
  }
  const long long gm = static_cast<long long>(op.groups) * op.m;
  static const long long waves = [] {  // CTAs of the v2 pass per resident slot (experiments)
    const char* e = std::getenv("JOFC_OOS2_WAVES");
    return e ? std::max(1LL, std::atoll(e)) : 1LL;
  }();
  const long long slices = std::max<long long>(
      1, std::min<long long>(op.n / kOos2Rows,
                             waves * std::max<long long>(1, per_sm) * c->num_sms / gm));
  const dim3 pg2(static_cast<unsigned>(gm), static_cast<unsigned>(slices));
  const unsigned ug = (op.k + 127) / 128;
  // The launches are replayed from a captured CUDA graph of `per_graph` steps
  // (all per-step state is in the device-side point records), chunk after
  // chunk until every point is done: the count of finished points is read one
  // chunk behind, so at most ~2 chunks of no-op launches follow the last point.
  // (fixed iteration counts cannot stop early: one graph of all steps)
  // (fused: launches 0 .. steps + 1, the last one only finishes the points)
  const size_t launches_needed = static_cast<size_t>(steps) + (fused ? 2 : 1);
  const size_t chunk =
      (stop_chunk() && !op.fixed) ? stop_chunk() : launches_needed;
  const size_t per_graph = std::min(chunk, launches_needed);
  if (!c->stop_flag) {
    JOFC_CUDA(cudaMallocHost(&c->stop_flag, 2 * sizeof(int)));
    for (int k = 0; k < 2; ++k)
      JOFC_CUDA(cudaEventCreateWithFlags(&c->stop_ev[k], cudaEventDisableTiming));
  }
  std::vector<uintptr_t> key = {0x0005u, static_cast<uintptr_t>(D), static_cast<uintptr_t>(op.k),
                                static_cast<uintptr_t>(op.m), static_cast<uintptr_t>(op.n),
                                static_cast<uintptr_t>(per_graph), static_cast<uintptr_t>(op.fixed),
                                static_cast<uintptr_t>(op.max_it),
                                reinterpret_cast<uintptr_t>(op.x),
                                reinterpret_cast<uintptr_t>(op.deltas),
                                reinterpret_cast<uintptr_t>(op.y0),
                                reinterpret_cast<uintptr_t>(op.y1),
                                reinterpret_cast<uintptr_t>(op.part),
                                reinterpret_cast<uintptr_t>(op.st),
                                reinterpret_cast<uintptr_t>(op.traces),
                                reinterpret_cast<uintptr_t>(op.done_count),
                                reinterpret_cast<uintptr_t>(op.deltas_t),
                                static_cast<uintptr_t>(oos_kernel_version())};
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
    if (fused && smem > 48 * 1024)
      JOFC_CUDA(cudaFuncSetAttribute(jofc_oos_step_kernel<D>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    for (size_t t = 0; t < per_graph; ++t) {
      if (fused) {
        OosParams ot = op;
        ot.local_t = static_cast<int>(t);
        jofc_oos_step_kernel<D><<<pg, kOosWarps * 32, smem, c->stream>>>(ot);
        continue;
      }
      if (v2)
        jofc_oos_pass2_kernel<D><<<pg2, kOos2Warps * 32, smem2, c->stream>>>(op);
      else
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
  for (size_t ch = 0; ch * per_graph < launches_needed; ++ch) {
    if (fused) {  // this chunk's first launch index
      jofc_oos_set_base_kernel<<<1, 1, 0, c->stream>>>(c->oos_done.p + 1,
                                                       static_cast<unsigned>(ch * per_graph));
      JOFC_CUDA(cudaGetLastError());
      ++c->launches;
    }
    JOFC_CUDA(cudaGraphLaunch(it->second, c->stream));
    c->launches += (fused ? 1 : 2) * per_graph;
    const int kk = static_cast<int>(ch & 1);
    JOFC_CUDA(cudaMemcpyAsync(&c->stop_flag[kk], op.done_count, sizeof(unsigned),
                              cudaMemcpyDeviceToHost, c->stream));
    JOFC_CUDA(cudaEventRecord(c->stop_ev[kk], c->stream));
    if (ch >= 1) {
      JOFC_CUDA(cudaEventSynchronize(c->stop_ev[kk ^ 1]));
      if (static_cast<unsigned>(c->stop_flag[kk ^ 1]) >= static_cast<unsigned>(op.k)) break;
    }
  }
  return JOFC_OK;
}

// The persistent solve (jofc_oos_solve_kernel): one CTA per SM, each owning a
// contiguous range of <= G points for the whole solve.  Returns 1 (nothing
// launched) when the batch does not fit the kernel's shared-memory plan: the
// caller falls back to the per-update kernels.
// Dynamic shared memory a CTA may opt into on this device, less the block
// the driver reserves per CTA (B200: 232448 - 1024 bytes).
int smem_optin(int device) {
  static std::mutex mu;
  static std::map<int, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(device);
  if (it != cache.end()) return it->second;
  int optin = 0, reserved = 0;
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) != cudaSuccess)
    optin = 232448;
  if (cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, device) !=
      cudaSuccess)
    reserved = 1024;
  return cache[device] = optin - reserved;
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

template <int D>
int oos_launch_persistent(jofc_ctx* c, const OosParams& op, bool auto_route) {
  constexpr int Q = oosp_q<D>();
  constexpr int V = D + 2;
  const int m = op.m, k = op.k;
  static const long long rows_env = [] {  // experiments: rows per chunk
    const char* e = std::getenv("JOFC_OOSP_ROWS");
    return e ? std::atoll(e) : 0LL;
  }();
  static const long long g_env = [] {  // experiments: points per CTA
    const char* e = std::getenv("JOFC_OOSP_G");
    return e ? std::atoll(e) : 0LL;
  }();
  const int kSmemOptin = smem_optin(c->device);
  JOFC_CUDA(ensure_smem_attr(jofc_oos_solve_kernel<D>, kSmemOptin, c->device));
  int G = static_cast<int>(std::min<long long>((k + c->num_sms - 1) / c->num_sms, kOospConsumers * Q));
  if (g_env > 0) G = static_cast<int>(std::min<long long>(g_env, kOospConsumers * Q));
  int S = 1;  // slots: the smallest divisor of the consumer warps holding G points
  while (S * Q < G || kOospConsumers % S) ++S;
  const int ncta = (k + G - 1) / G;
  const int waves = (ncta + c->num_sms - 1) / c->num_sms;
  // AUTO: only batches that fill the point slots.  A CTA's time per update is
  // set by its S slots of Q points, used or not, and a second wave of CTAs
  // doubles it, so the persistent solve pays off only when the batch uses
  // >= 75% of waves x SMs x S x Q point slots; smaller or ragged batches run
  // the per-update kernels, which spread a point over several CTAs.  Device
  // time per 100-update solve, m = 2, n = 5000, d = 3, persistent vs
  // per-update (scripts/oos_small_k.py): k = 1 1.46 vs 0.98 ms, k = 300 1.50
  // vs 1.40, k = 450 1.28 vs 1.76, k = 600 2.36 vs 2.15, k = 1000 2.20 vs
  // 2.87, k = 2000 3.99 vs 6.03, k = 5000 (two waves) 15.1 vs 13.7; k = 1,
  // n = 200000 45 vs 22.
  const double used = static_cast<double>(k) /
                      (static_cast<double>(waves) * c->num_sms * S * Q);
  if (auto_route && g_env <= 0 && used < 0.75) return 1;
  OospParams pp{};
  // fixed part: part, y, warp sums, previous stresses, sums of X, done flags
  const size_t fixed_bytes = static_cast<size_t>(m) * G * V * 8 + 2ull * G * m * D * 8 +
                             static_cast<size_t>(kOospConsumers) * Q * V * 8 + static_cast<size_t>(G) * 8 +
                             static_cast<size_t>(m) * D * 8 + static_cast<size_t>(G) * 4 + 64;
  // Rows per chunk: as large as two ring stages allow, balanced over the
  // modality pass (the per-chunk cost -- wait, release, refill -- dominates
  // small chunks: C5 R = 512 x 5 stages 41.1k batch-it/s, 768 x 3 43.3k,
  // 1024 x 2 44.7k, 1280 x 2 45.4k), a multiple of the lanes of a slot.
  const int lanes_per_slot = 32 * (kOospConsumers / S);  // every lane the same rows
  const long long room = static_cast<long long>(kSmemOptin) - 128 - static_cast<long long>(fixed_bytes);
  const long long row_bytes = (static_cast<long long>(G) + D) * 8;
  long long r_max = (room / 2 - 16) / row_bytes / lanes_per_slot * lanes_per_slot;
  if (rows_env > 0) r_max = std::min<long long>(r_max, std::max<long long>(lanes_per_slot, rows_env));
  if (r_max < lanes_per_slot) return 1;  // (does not fit: the per-update kernels)
  const long long nch_min = (op.n + r_max - 1) / r_max;
  const int R = static_cast<int>(std::min<long long>(
      r_max, ((op.n + nch_min - 1) / nch_min + lanes_per_slot - 1) / lanes_per_slot * lanes_per_slot));
  const size_t stage_bytes = (static_cast<size_t>(G) * R + static_cast<size_t>(R) * D + 2) * 8;
  const int stages = static_cast<int>(
      std::min<long long>(kOospMaxStages, room / static_cast<long long>(stage_bytes)));
  if (stages < 2) return 1;

  pp.x = op.x;
  pp.deltas = op.deltas;
  pp.ystart = op.y0;
  pp.yout0 = op.y0;
  pp.yout1 = op.y1;
  pp.traces = op.traces;
  pp.st = op.st;
  pp.k = k;
  pp.m = m;
  pp.n = op.n;
  pp.w = op.w;
  pp.eps = op.eps;
  pp.term_count = op.term_count;
  pp.max_it = op.max_it;
  pp.fixed = op.fixed;
  pp.G = G;
  pp.S = S;
  pp.ncta = ncta;
  pp.R = R;
  pp.stages = stages;
  pp.nch = static_cast<int>((op.n + R - 1) / R);
  pp.stage_doubles = static_cast<unsigned>(static_cast<size_t>(G) * R + static_cast<size_t>(R) * D + 2);
  size_t o = 128;
  pp.off_ring = static_cast<unsigned>(o);
  o += static_cast<size_t>(stages) * pp.stage_doubles * 8;
  pp.off_part = static_cast<unsigned>(o);
  o += static_cast<size_t>(m) * G * V * 8;
  pp.off_y = static_cast<unsigned>(o);
  o += 2ull * G * m * D * 8;
  pp.off_red = static_cast<unsigned>(o);
  o += static_cast<size_t>(kOospConsumers) * Q * V * 8;
  pp.off_misc = static_cast<unsigned>(o);
  o += static_cast<size_t>(G) * 8 + static_cast<size_t>(m) * D * 8 + static_cast<size_t>(G) * 4;
  const size_t bytes = align_up(o, 16);
  if (bytes > static_cast<size_t>(kSmemOptin)) return 1;
  // delta in ring order (once per batch)
  const size_t nperm = static_cast<size_t>(pp.ncta) * m * pp.nch * G * R;
  JOFC_CUDA(c->oos_delta_p.ensure(nperm));
  pp.dperm = c->oos_delta_p.p;
  jofc_oos_permute_kernel<<<static_cast<unsigned>(nperm / R), 256, 0, c->stream>>>(
      op.deltas, c->oos_delta_p.p, k, m, op.n, pp.ncta, G, R, pp.nch);
  JOFC_CUDA(cudaGetLastError());
  ++c->launches;
  if (std::getenv("JOFC_OOSP_DEBUG"))
    std::fprintf(stderr, "oosp: k %d m %d n %lld D %d: G %d S %d R %d stages %d ncta %d nch %d smem %zu\n",
                 k, m, op.n, D, G, S, R, stages, pp.ncta, pp.nch, bytes);
  jofc_oos_solve_kernel<D><<<pp.ncta, kOospThreads, bytes, c->stream>>>(pp);
  const cudaError_t le = cudaGetLastError();
  if (le == cudaErrorLaunchOutOfResources || le == cudaErrorInvalidConfiguration) {
    return 1;  // (e.g. shared memory not available at this size: the per-update kernels)
  }
  JOFC_CUDA(le);
  ++c->launches;
  return JOFC_OK;
}

int oos_run(jofc_ctx* c, size_t k, size_t m, size_t n, size_t d, const double* x,
            const double* deltas, double w, const double* y0, double eps, size_t max_it,
            int fixed, double* y_out, double* traces, size_t* iterations, double* stress0) {
  const NvtxScope nvtx_scope("jofc_oos");
  if (!c) return set_error(JOFC_EINVAL, "null context");
  if (!(w > 0.0)) return set_error(JOFC_EINVAL, "oos: w must be strictly positive");
  if (!(eps > 0.0)) return set_error(JOFC_EINVAL, "OosOptions: eps must be positive");
  if (m == 0 || n == 0 || k == 0) return set_error(JOFC_EINVAL, "oos: empty input");
  if (d < 1 || d > static_cast<size_t>(kMaxD))
    return set_error(JOFC_EINVAL, "dim %zu unsupported (1..%d)", d, kMaxD);
  JOFC_CUDA(cudaSetDevice(c->device));
  JOFC_CUDA(c->oos_x.ensure(m * n * d + 4));  // + slack: chunk copies round up to 16 bytes
  JOFC_CUDA(c->oos_delta.ensure(k * m * n + 2));  // + slack: segment copies round up to 16 bytes
  const int groups = static_cast<int>((k + 31) / 32);
  if (oos_kernel_version() == 2)
    JOFC_CUDA(c->oos_delta_t.ensure(static_cast<size_t>(groups) * 32 * m * n));
  JOFC_CUDA(c->oos_y0.ensure(k * m * d));
  JOFC_CUDA(c->oos_y1.ensure(k * m * d));
  // partials: 3 x k x m x (d + 2) (the fused step kernel's triple buffer; the
  // two-kernel path uses the first) + 2 x k previous stresses
  const size_t kmd = k * m * (d + 2);
  JOFC_CUDA(c->oos_part.ensure(3 * kmd + 2 * k));
  JOFC_CUDA(c->oos_trace.ensure(k * (max_it + 1)));
  JOFC_CUDA(c->oos_st.ensure(k));
  JOFC_CUDA(c->oos_done.ensure(3));  // done count, launch index, arrivals
  JOFC_CUDA(cudaMemsetAsync(c->oos_done.p, 0, 3 * sizeof(unsigned), c->stream));
  JOFC_CUDA(cudaMemcpyAsync(c->oos_x.p, x, m * n * d * sizeof(double), cudaMemcpyDefault, c->stream));
  JOFC_CUDA(cudaMemcpyAsync(c->oos_delta.p, deltas, k * m * n * sizeof(double), cudaMemcpyDefault,
                            c->stream));
  JOFC_CUDA(cudaMemcpyAsync(c->oos_y0.p, y0, k * m * d * sizeof(double), cudaMemcpyDefault,
                            c->stream));
  JOFC_CUDA(cudaMemsetAsync(c->oos_st.p, 0, k * sizeof(OosPoint), c->stream));
  JOFC_CUDA(cudaMemsetAsync(c->oos_part.p, 0, (3 * kmd + 2 * k) * sizeof(double), c->stream));
  if (oos_kernel_version() == 2) {  // delta rows -> [j][point group][row][32 points], once per solve
    const dim3 tg(static_cast<unsigned>((n + 31) / 32), static_cast<unsigned>(m * groups));
    jofc_oos_transpose_kernel<<<tg, 256, 0, c->stream>>>(c->oos_delta.p, c->oos_delta_t.p,
                                                         static_cast<int>(k), static_cast<int>(m),
                                                         static_cast<long long>(n), groups);
    JOFC_CUDA(cudaGetLastError());
    ++c->launches;
  }
  OosParams op{};
  op.deltas_t = oos_kernel_version() == 2 ? c->oos_delta_t.p : nullptr;
  op.groups = groups;
  op.base = c->oos_done.p + 1;
  op.prev2 = c->oos_part.p + 3 * kmd;
  op.x = c->oos_x.p;
  op.deltas = c->oos_delta.p;
  op.y0 = c->oos_y0.p;
  op.y1 = c->oos_y1.p;
  op.part = c->oos_part.p;
  op.st = c->oos_st.p;
  op.done_count = c->oos_done.p;
  op.traces = c->oos_trace.p;
  op.k = static_cast<int>(k);
  op.m = static_cast<int>(m);
  op.n = static_cast<long long>(n);
  op.w = w;
  op.eps = eps;
  op.term_count = static_cast<double>(m * n) + 0.5 * static_cast<double>(m * (m - 1));
  op.max_it = static_cast<int>(max_it);
  op.fixed = fixed;
  int rc = 1;
  if (oos_kernel_version() == 4 && c->oos_route != JOFC_OOS_PER_UPDATE) {
    const bool auto_route = c->oos_route == JOFC_OOS_AUTO;
    switch (d) {
      case 1: rc = oos_launch_persistent<1>(c, op, auto_route); break;
      case 2: rc = oos_launch_persistent<2>(c, op, auto_route); break;
      case 3: rc = oos_launch_persistent<3>(c, op, auto_route); break;
      case 4: rc = oos_launch_persistent<4>(c, op, auto_route); break;
      case 5: rc = oos_launch_persistent<5>(c, op, auto_route); break;
      case 6: rc = oos_launch_persistent<6>(c, op, auto_route); break;
      case 7: rc = oos_launch_persistent<7>(c, op, auto_route); break;
      case 8: rc = oos_launch_persistent<8>(c, op, auto_route); break;
      case 9: rc = oos_launch_persistent<9>(c, op, auto_route); break;
      default: rc = oos_launch_persistent<10>(c, op, auto_route); break;
    }
    if (rc != JOFC_OK && rc != 1) return rc;
  }
  if (rc == 1) switch (d) {
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

