// capi_nccl.cu -- the C-native NCCL exchange of a sharded context (C ABI part
// of include/jofc_gpu.h).
//
// The reference has no multi-GPU path; its data-parallel site
// is the per-(modality, object) loop of block_guttman_products
// (proj/src/solver.cpp:27-49).  Here every rank streams its shard of the
// packed Delta into a partial P = B(X)X over ALL objects plus a partial
// fidelity; per iteration
//
//   pass                      partial P (all rows), partial fidelity
//   NCCL group: m x ncclReduceScatter(P_l -> own row chunk of P_l, in place)
//               + ncclAllReduce(fidelity, 1 double)
//   epilogue                  W^-1 mix of the OWN rows only (X_{t+1}), P
//                             zeroed, commensurability of X_t over all rows
//                             (X_t is replicated: every rank sums it in the
//                             same order), sigma_t and the stop rule -- the
//                             same decision on every rank
//   NCCL group: m x ncclAllGather(own rows of X_{t+1}_l -> X_{t+1}_l, in place)
//
// With the identity-form fidelity (jofc_kernels.cuh, rho_decide) the pass
// skips the per-pair fidelity; the epilogue folds its own rows' sums
// (commensurability, x_i . P_i, |x_i - x_0|^2, x_i - x_0 per modality), the
// all-gather group all-reduces that vector (1 + m (d + 2) doubles), and
// jofc_rho_decide_kernel takes the same decision on every rank.
//
// so each rank moves (W-1)/W of P in and of X out per iteration -- the
// north star's all-gather of X -- and mixes 1/W of the objects.  Every call is
// on the context stream, so the whole sequence is captured in the same CUDA
// graph as the single-GPU loop (jofc_capi.cu, enqueue_solve).
//
// NCCL itself is resolved at run time (dlopen of libnccl.so.2: the copy the
// process already loaded, e.g. torch's, else the system NCCL 2.27 of this
// image), so libjofc_gpu.so has no link-time NCCL dependency and still loads
// where NCCL is absent; the types come from the system <nccl.h>.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>

#include "capi_internal.h"
#include "jofc_gpu.h"

using namespace jofc_gpu;
using namespace jofc_gpu::capi;

namespace {

struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                                ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  std::string error;
};

template <class F>
bool bind(void* h, const char* name, F*& fn) {
  fn = reinterpret_cast<F*>(dlsym(h, name));
  return fn != nullptr;
}

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // a copy already in the process first (one NCCL instance per process)
    // then JOFC_NCCL_LIB, then the loader's libnccl.so.2.  (A process that
    // will also use torch should import torch first: once loaded here, a
    // libnccl.so.2 satisfies torch's own dependency by soname, and an older
    // system copy lacks symbols torch's build needs -- api.py does that.)
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    const char* env = std::getenv("JOFC_NCCL_LIB");
    if (!h && env && *env) h = dlopen(env, RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      api.error = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return;
    }
    bool ok = bind(h, "ncclGetUniqueId", api.GetUniqueId) &&
              bind(h, "ncclCommInitRank", api.CommInitRank) &&
              bind(h, "ncclCommDestroy", api.CommDestroy) &&
              bind(h, "ncclCommAbort", api.CommAbort) &&
              bind(h, "ncclReduceScatter", api.ReduceScatter) &&
              bind(h, "ncclAllGather", api.AllGather) &&
              bind(h, "ncclAllReduce", api.AllReduce) &&
              bind(h, "ncclGroupStart", api.GroupStart) && bind(h, "ncclGroupEnd", api.GroupEnd) &&
              bind(h, "ncclGetErrorString", api.GetErrorString) &&
              bind(h, "ncclGetVersion", api.GetVersion) &&
              bind(h, "ncclCommGetAsyncError", api.CommGetAsyncError);
    if (!ok) {
      api.error = "libnccl.so.2 lacks a required symbol";
      return;
    }
    api.handle = h;
  });
  return api;
}

#define JOFC_NCCL(call)                                                                        \
  do {                                                                                         \
    const ncclResult_t r_ = (call);                                                            \
    if (r_ != ncclSuccess)                                                                     \
      return set_error(JOFC_ECOMM, "%s failed: %s", #call, nccl().GetErrorString(r_));         \
  } while (0)

}  // namespace

namespace jofc_gpu {
namespace capi {

long long nccl_chunk_rows(const jofc_ctx* c) { return c->lay.n_pad / c->nccl_world; }

int nccl_check(jofc_ctx* c) {
  if (c->lay.n_pad % c->nccl_world != 0)
    return set_error(JOFC_EINVAL,
                     "NCCL exchange: world %d must divide the padded object count %lld "
                     "(use a power-of-two world, or the peer / hook exchange)",
                     c->nccl_world, c->lay.n_pad);
  return JOFC_OK;
}

// The exchange after pass t: reduce-scatter of P's row chunks (+ fidelity sum).
int nccl_reduce(jofc_ctx* c, double* P, size_t fid_slot) {
  const NcclApi& api = nccl();
  const long long rows = nccl_chunk_rows(c);
  const size_t cnt = static_cast<size_t>(rows) * c->d;
  const size_t per_mod = static_cast<size_t>(c->lay.n_pad) * c->d;
  JOFC_NCCL(api.GroupStart());
  for (int l = 0; l < c->lay.m; ++l) {
    double* Pl = P + l * per_mod;
    JOFC_NCCL(api.ReduceScatter(Pl, Pl + c->rank * cnt, cnt, ncclFloat64, ncclSum,
                                static_cast<ncclComm_t>(c->nccl_comm), c->stream));
  }
  JOFC_NCCL(api.AllReduce(P + fid_slot, P + fid_slot, 1, ncclFloat64, ncclSum,
                          static_cast<ncclComm_t>(c->nccl_comm), c->stream));
  JOFC_NCCL(api.GroupEnd());
  return JOFC_OK;
}

// After the epilogue of t: all-gather of the own rows of X_{t+1}, plus (the
// identity-form fidelity) the all-reduce of the ranks' folded sums, `sums`
// (count doubles; null: none) in the same group.
int nccl_gather(jofc_ctx* c, double* xn, double* sums, size_t count) {
  const NcclApi& api = nccl();
  const size_t cnt = static_cast<size_t>(nccl_chunk_rows(c)) * c->d;
  const size_t per_mod = static_cast<size_t>(c->lay.n_pad) * c->d;
  JOFC_NCCL(api.GroupStart());
  for (int l = 0; l < c->lay.m; ++l) {
    double* Xl = xn + l * per_mod;
    JOFC_NCCL(api.AllGather(Xl + c->rank * cnt, Xl, cnt, ncclFloat64,
                            static_cast<ncclComm_t>(c->nccl_comm), c->stream));
  }
  if (sums)
    JOFC_NCCL(api.AllReduce(sums, sums, count, ncclFloat64, ncclSum,
                            static_cast<ncclComm_t>(c->nccl_comm), c->stream));
  JOFC_NCCL(api.GroupEnd());
  return JOFC_OK;
}

// Waits for the context stream of an NCCL-exchanging context.  A plain
// cudaStreamSynchronize would block forever if a peer died or the network
// failed (the collective kernels never complete), so the stream is polled and
// the communicator's asynchronous error checked between polls; on an error
// the communicator is aborted (which lets the stream drain) and released, and
// the call returns JOFC_ECOMM -- the caller re-initialises the exchange.
int nccl_wait(jofc_ctx* c) {
  const NcclApi& api = nccl();
  auto comm = static_cast<ncclComm_t>(c->nccl_comm);
  for (int spin = 0;; ++spin) {
    const cudaError_t q = cudaStreamQuery(c->stream);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady)
      return set_error(JOFC_ECUDA, "stream wait: %s", cudaGetErrorString(q));
    ncclResult_t async = ncclSuccess;
    const ncclResult_t r = api.CommGetAsyncError(comm, &async);
    if (r != ncclSuccess || async != ncclSuccess) {
      const ncclResult_t bad = (r != ncclSuccess) ? r : async;
      api.CommAbort(comm);
      c->nccl_comm = nullptr;
      c->nccl_world = 0;
      for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
      c->graphs.clear();
      return set_error(JOFC_ECOMM, "NCCL exchange failed: %s (communicator aborted; call "
                       "jofc_nccl_init again)", api.GetErrorString(bad));
    }
    // spin briefly (a solve ends within microseconds of the first poll when
    // the host enqueued it long ago), then back off to 50 us sleeps
    if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
  return JOFC_OK;
}

void nccl_release(jofc_ctx* c) {
  if (c->nccl_comm) {
    cudaStreamSynchronize(c->stream);
    nccl().CommDestroy(static_cast<ncclComm_t>(c->nccl_comm));
  }
  c->nccl_comm = nullptr;
  c->nccl_world = 0;
}

}  // namespace capi
}  // namespace jofc_gpu

extern "C" {

int jofc_nccl_version(int* version) {
  if (!version) return set_error(JOFC_EINVAL, "null argument");
  const NcclApi& api = nccl();
  if (!api.handle) return set_error(JOFC_ECOMM, "%s", api.error.c_str());
  JOFC_NCCL(api.GetVersion(version));
  return JOFC_OK;
}

int jofc_nccl_unique_id(void* id_out) {
  if (!id_out) return set_error(JOFC_EINVAL, "null argument");
  const NcclApi& api = nccl();
  if (!api.handle) return set_error(JOFC_ECOMM, "%s", api.error.c_str());
  ncclUniqueId id;
  JOFC_NCCL(api.GetUniqueId(&id));
  static_assert(sizeof(id) == JOFC_NCCL_ID_BYTES, "ncclUniqueId size");
  std::memcpy(id_out, &id, sizeof(id));
  return JOFC_OK;
}

int jofc_nccl_init(jofc_ctx* c, const void* id, int rank, int world) {
  if (!c || !id) return set_error(JOFC_EINVAL, "null argument");
  if (world < 1 || rank < 0 || rank >= world)
    return set_error(JOFC_EINVAL, "NCCL exchange: rank %d of world %d invalid", rank, world);
  if (rank != c->rank || world != c->world)
    return set_error(JOFC_EINVAL, "NCCL exchange: rank %d of %d but the shard is %d of %d", rank,
                     world, c->rank, c->world);
  const NcclApi& api = nccl();
  if (!api.handle) return set_error(JOFC_ECOMM, "%s", api.error.c_str());
  JOFC_CUDA(cudaSetDevice(c->device));
  nccl_release(c);
  peer_release(c);  // one exchange at a time
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm = nullptr;
  JOFC_NCCL(api.CommInitRank(&comm, world, uid, rank));
  c->nccl_comm = comm;
  c->nccl_world = world;
  for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);  // (no graph of the old route)
  c->graphs.clear();
  return JOFC_OK;
}

int jofc_nccl_release(jofc_ctx* c) {
  if (!c) return set_error(JOFC_EINVAL, "null context");
  JOFC_CUDA(cudaSetDevice(c->device));
  for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
  c->graphs.clear();
  nccl_release(c);
  return JOFC_OK;
}

}  // extern "C"
