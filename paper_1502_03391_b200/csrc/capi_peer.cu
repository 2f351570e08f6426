// capi_peer.cu -- the peer-memory exchange of a sharded context (C ABI part
// of include/jofc_gpu.h; kernels and protocol in jofc_peer.cuh).
//
// The reference has no multi-GPU path: this replaces the
// per-iteration sum-all-reduce of the partial products + epilogue with a
// reduce-scatter read fused into the mix and an all-gather write of the new
// configuration, both through peer pointers.
#include <cuda_runtime.h>

#include <cstring>
#include <vector>

#include "capi_internal.h"
#include "jofc_gpu.h"

using namespace jofc_gpu;
using namespace jofc_gpu::capi;

namespace {

long long round32(long long v) { return (v + 31) & ~31LL; }

// Slab layout for the context's problem (m, n_pad); sized for kMaxD so that
// any solve dimension fits the same offsets on every rank.
void peer_layout(jofc_ctx* c) {
  PeerState& ps = c->peer;
  const long long cap = static_cast<long long>(c->lay.m) * c->lay.n_pad * kMaxD;
  ps.p_len = round32(cap + 1);
  const long long x_len = round32(cap);
  ps.p_off[0] = 0;
  ps.p_off[1] = ps.p_len;
  ps.x_off[0] = 2 * ps.p_len;
  ps.x_off[1] = ps.x_off[0] + x_len;
  ps.com_off = ps.x_off[1] + x_len;
  ps.flag1_off = ps.com_off + 32;
  ps.flag2_off = ps.flag1_off + kMaxPeers;
  ps.slab_doubles = static_cast<size_t>(ps.flag2_off + kMaxPeers);
  ps.key = {c->lay.m, c->lay.n_pad};
}

void close_opened(PeerState& ps) {
  for (void* p : ps.opened)
    if (p) cudaIpcCloseMemHandle(p);
  ps.opened.clear();
}

template <int D>
int launch_mix(jofc_ctx* c, const PeerParams& pe) {
  const size_t smem = static_cast<size_t>(c->lay.m) * pe.rows_cta * D * sizeof(double);
  jofc_peer_mix_kernel<D><<<c->peer.mix_grid, 256, smem, c->stream>>>(pe);
  JOFC_CUDA(cudaGetLastError());
  return JOFC_OK;
}

int mix_for_d(jofc_ctx* c, const PeerParams& pe) { JOFC_DISPATCH_D(c->d, launch_mix, c, pe); }

PeerParams peer_params(jofc_ctx* c, const PassParams& pp, size_t t) {
  const PeerState& ps = c->peer;
  const int k = static_cast<int>((t + ps.phase) & 1);
  PeerParams pe{};
  pe.slabs = ps.ptrs.p;
  pe.rank = ps.rank;
  pe.world = ps.world;
  pe.p_read = ps.p_off[k];
  pe.p_zero = ps.p_off[k ^ 1];
  pe.p_len = ps.p_len;
  pe.x_off0 = ps.x_off[0];
  pe.x_off1 = ps.x_off[1];
  pe.com_off = ps.com_off;
  pe.flag1_off = ps.flag1_off;
  pe.flag2_off = ps.flag2_off;
  pe.row_lo = ps.row_lo;
  pe.row_hi = ps.row_hi;
  pe.rows_cta = ps.rows_cta;
  pe.com_partials = ps.com_part.p;
  pe.trace = pp.epi.trace;
  pe.ctrl = pp.ctrl;
  pe.coef = pp.epi.coef;
  pe.cross = pp.epi.cross;
  pe.m = c->lay.m;
  pe.n_pad = c->lay.n_pad;
  pe.fid_slot = static_cast<long long>(pp.fid_slot);
  return pe;
}

// Every attach starts the group from a clean slab: both P regions, X, the
// flags and the epoch counter zeroed (a slab left by an earlier group holds a
// dirty P region and that group's flags).  All ranks must attach before any
// of them solves (dist.attach_peers puts a barrier there).
int attach_common(jofc_ctx* c, int rank, int world, const std::vector<double*>& bases) {
  PeerState& ps = c->peer;
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  JOFC_CUDA(cudaMemsetAsync(ps.slab, 0, ps.slab_doubles * sizeof(double), c->stream));
  ps.epoch = 0;
  JOFC_CUDA(ps.ptrs.ensure(world));
  JOFC_TRY(copy_sync(c, ps.ptrs.p, bases.data(), world * sizeof(double*), cudaMemcpyHostToDevice));
  ps.rank = rank;
  ps.world = world;
  ps.row_lo = c->lay.n * rank / world;
  ps.row_hi = c->lay.n * (rank + 1) / world;
  // objects per mix CTA: the world's products of m modalities x D coordinates
  // for rows_cta objects in 48 KB of shared memory
  ps.rows_cta = static_cast<int>(std::max<long long>(
      1, std::min<long long>(32, 6144 / (static_cast<long long>(c->lay.m) * kMaxD))));
  ps.mix_grid = static_cast<int>(std::max<long long>(
      1, (ps.row_hi - ps.row_lo + ps.rows_cta - 1) / ps.rows_cta));
  JOFC_CUDA(ps.com_part.ensure(ps.mix_grid));
  ps.phase = 0;
  ps.pending = false;
  ps.active = true;
  return JOFC_OK;
}

int attach_checks(jofc_ctx* c, int rank, int world) {
  if (!c) return set_error(JOFC_EINVAL, "null context");
  JOFC_TRY(require_problem(c));
  if (world < 2 || world > kMaxPeers || rank < 0 || rank >= world)
    return set_error(JOFC_EINVAL, "peer exchange: rank %d of world %d (2..%d ranks)", rank, world,
                     kMaxPeers);
  if (rank != c->rank || world != c->world)
    return set_error(JOFC_EINVAL, "peer exchange: rank %d of %d but the shard is %d of %d", rank,
                     world, c->rank, c->world);
  if (!c->peer.slab) return set_error(JOFC_EINVAL, "peer exchange: jofc_peer_export first");
  JOFC_CUDA(cudaSetDevice(c->device));
  return JOFC_OK;
}

}  // namespace

namespace jofc_gpu {
namespace capi {

int peer_check(jofc_ctx* c) {
  const std::vector<long long> key = {c->lay.m, c->lay.n_pad};
  if (key != c->peer.key)
    return set_error(JOFC_EINVAL,
                     "peer exchange: the slab was exported for another problem (export and attach "
                     "again)");
  return JOFC_OK;
}

void peer_release(jofc_ctx* c) {
  PeerState& ps = c->peer;
  close_opened(ps);
  ps.ptrs.release();
  ps.com_part.release();
  if (ps.slab) cudaFree(ps.slab);
  ps.slab = nullptr;
  ps.active = false;
  ps.pending = false;
}

int peer_stage(jofc_ctx* c, const PassParams& base, size_t t, int stage) {
  const PeerState& ps = c->peer;
  const PeerParams pe = peer_params(c, base, t);
  if (stage == 0) {
    PassParams pp = base;
    pp.P = ps.slab + pe.p_read;
    pp.peer_slabs = ps.ptrs.p;
    pp.flag1_off = ps.flag1_off;
    pp.peer_rank = ps.rank;
    pp.peer_world = ps.world;
    pp.fuse_epilogue = 0;
    JOFC_TRY(pass_for_d(c, pp));
  } else if (stage == 1) {
    JOFC_TRY(mix_for_d(c, pe));
  } else {
    jofc_peer_decide_kernel<<<1, 32, 0, c->stream>>>(pe);
    JOFC_CUDA(cudaGetLastError());
  }
  ++c->launches;
  return JOFC_OK;
}

}  // namespace capi
}  // namespace jofc_gpu

extern "C" {

int jofc_peer_export(jofc_ctx* c, void* ipc_handle_out, void** slab_out) {
  if (!c) return set_error(JOFC_EINVAL, "null context");
  JOFC_TRY(require_problem(c));
  JOFC_CUDA(cudaSetDevice(c->device));
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  peer_release(c);
  peer_layout(c);
  PeerState& ps = c->peer;
  JOFC_CUDA(cudaMalloc(&ps.slab, ps.slab_doubles * sizeof(double)));
  JOFC_CUDA(cudaMemsetAsync(ps.slab, 0, ps.slab_doubles * sizeof(double), c->stream));
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  if (ipc_handle_out) {
    cudaIpcMemHandle_t h;
    JOFC_CUDA(cudaIpcGetMemHandle(&h, ps.slab));
    static_assert(sizeof(h) == 64, "CUDA IPC handle size");
    std::memcpy(ipc_handle_out, &h, sizeof(h));
  }
  if (slab_out) *slab_out = ps.slab;
  return JOFC_OK;
}

int jofc_peer_attach(jofc_ctx* c, int rank, int world, const void* handles) {
  JOFC_TRY(attach_checks(c, rank, world));
  if (!handles) return set_error(JOFC_EINVAL, "peer exchange: null handles");
  PeerState& ps = c->peer;
  close_opened(ps);
  std::vector<double*> bases(world, nullptr);
  for (int q = 0; q < world; ++q) {
    if (q == rank) {
      bases[q] = ps.slab;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + 64 * q, sizeof(h));
    void* p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      close_opened(ps);
      return set_error(JOFC_ECOMM, "peer exchange: opening rank %d's slab: %s", q,
                       cudaGetErrorString(e));
    }
    ps.opened.push_back(p);
    bases[q] = static_cast<double*>(p);
  }
  nccl_release(c);  // one exchange at a time
  return attach_common(c, rank, world, bases);
}

int jofc_peer_attach_pointers(jofc_ctx* c, int rank, int world, void* const* slabs) {
  JOFC_TRY(attach_checks(c, rank, world));
  if (!slabs) return set_error(JOFC_EINVAL, "peer exchange: null slabs");
  close_opened(c->peer);  // (mappings of an earlier IPC attach)
  std::vector<double*> bases(world);
  for (int q = 0; q < world; ++q) bases[q] = static_cast<double*>(slabs[q]);
  if (bases[rank] != c->peer.slab)
    return set_error(JOFC_EINVAL, "peer exchange: slab %d is not this context's", rank);
  nccl_release(c);  // one exchange at a time
  return attach_common(c, rank, world, bases);
}

void* jofc_peer_address(jofc_ctx* c, int q) {
  if (!c || !c->peer.active || q < 0 || q >= c->peer.world) return nullptr;
  if (q == c->peer.rank) return c->peer.slab;
  // the opened mappings are stored in rank order without this rank's own slab
  const int idx = q < c->peer.rank ? q : q - 1;
  return idx < static_cast<int>(c->peer.opened.size()) ? c->peer.opened[idx] : nullptr;
}

int jofc_peer_detach(jofc_ctx* c) {
  if (!c) return set_error(JOFC_EINVAL, "null context");
  JOFC_CUDA(cudaSetDevice(c->device));
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  peer_release(c);
  return JOFC_OK;
}

int jofc_peer_lockstep_solve(jofc_ctx* const* ctxs, int world, const jofc_weights* spec, size_t d,
                             const double* x0, double eps, size_t max_it) {
  if (!ctxs || world < 2) return set_error(JOFC_EINVAL, "lockstep: need >= 2 contexts");
  for (int r = 0; r < world; ++r)
    if (!ctxs[r] || !ctxs[r]->peer.active || ctxs[r]->peer.rank != r ||
        ctxs[r]->peer.world != world)
      return set_error(JOFC_EINVAL, "lockstep: context %d is not rank %d of a %d-rank peer group",
                       r, r, world);
  std::vector<PassParams> pp(world);
  std::vector<EpiParams> ep(world);
  for (int r = 0; r < world; ++r) {
    JOFC_CUDA(cudaSetDevice(ctxs[r]->device));
    JOFC_TRY(prepare_solve(ctxs[r], spec, d, x0, eps, max_it, &pp[r], &ep[r]));
  }
  // stage s of every rank waits for stage s - 1 of every rank (events): each
  // flag a kernel polls was raised before it starts
  std::vector<cudaEvent_t> ev(2 * world, nullptr);
  int rc = JOFC_OK;
  for (auto& e : ev)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
      rc = set_error(JOFC_ECUDA, "lockstep: event creation failed");
  for (size_t t = 0; t <= max_it && !rc; ++t) {
    for (int stage = 0; stage < 3 && !rc; ++stage) {
      for (int r = 0; r < world && !rc; ++r) {
        jofc_ctx* c = ctxs[r];
        cudaSetDevice(c->device);
        if (stage > 0)
          for (int q = 0; q < world; ++q)
            if (cudaStreamWaitEvent(c->stream, ev[(stage - 1) * world + q], 0) != cudaSuccess)
              rc = set_error(JOFC_ECUDA, "lockstep: stream wait failed");
        if (!rc) rc = peer_stage(c, pp[r], t, stage);
        if (!rc && stage < 2 && cudaEventRecord(ev[stage * world + r], c->stream) != cudaSuccess)
          rc = set_error(JOFC_ECUDA, "lockstep: event record failed");
      }
    }
  }
  for (int r = 0; r < world; ++r) cudaStreamSynchronize(ctxs[r]->stream);
  for (auto& e : ev)
    if (e) cudaEventDestroy(e);
  return rc;
}

}  // extern "C"
