// jofc_peer.cuh -- the multi-GPU exchange of the Guttman loop over peer
// memory (NVLink / NVSwitch), without NCCL.
//
// Each rank streams its shard of the packed Delta (jofc_pass_kernel) into
// its own copy of P = B(X)X (all objects, partial over the shard) and a
// partial fidelity.  The collective the loop needs is a sum of the world's
// P followed by the W^-1 mix (proj/src/solver.cpp:52-72) and the stress /
// stop rule (proj/src/solver.cpp:129-143).  Here it is a reduce-scatter read
// fused with the mix and an all-gather write fused with it too:
//
//   pass (each rank)   products into P[t] of its slab; the last CTA raises
//                      flag1[rank] = (epoch, t) in every rank's slab
//   jofc_peer_mix_kernel<D>   waits for flag1 of all ranks, reads ITS rows of
//                      every rank's P[t] (peer loads, summed in rank order),
//                      mixes them into X_{t+1} and stores those rows into
//                      every rank's X_{t+1}; commensurability of X_t over its
//                      rows; zeroes its own P[t + 1]; the last CTA raises
//                      flag2[rank] everywhere
//   jofc_peer_decide_kernel   waits for flag2 of all ranks, sums the ranks'
//                      fidelity and commensurability in rank order: the same
//                      sigma_t and stop decision on every rank
//
// Ranks hold bitwise-identical X and control state, so no rank ever waits
// for a kernel that another rank will not launch.  Buffer reuse is safe
// without further barriers: P alternates between two regions by iteration
// parity (region t + 1 is zeroed only after every rank's pass t started,
// i.e. after every rank finished reading it at iteration t - 1), and a rank
// writes into a peer's X_{t+1} only after that peer's pass t -- the last
// reader of the buffer's previous contents -- finished.
//
// Slab of a rank (one cudaMalloc, exported by CUDA IPC), offsets in doubles
// (PeerLayout): P[0], P[1] (each m * n_pad * kMaxD + 1 with the fidelity
// slot at m * n_pad * d), X[0], X[1], the commensurability slot, flag1[],
// flag2[] (u64 per rank).
#pragma once

#include "jofc_kernels.cuh"

namespace jofc_gpu {

constexpr int kMaxPeers = 16;

struct PeerParams {
  double* const* slabs;   // [world] slab bases (device pointers, own = slabs[rank])
  int rank, world;
  long long p_read;       // this iteration's P region
  long long p_zero;       // the other P region: zeroed for the next pass
  long long p_len;        // doubles zeroed
  long long x_off0, x_off1;  // X buffers (X_t lives in buffer t & 1)
  long long com_off, flag1_off, flag2_off;
  long long row_lo, row_hi;  // the objects this rank mixes
  int rows_cta;              // objects per CTA of the mix (shared-memory bound)
  double* com_partials;      // one per mix CTA (own memory)
  double* trace;
  Control* ctrl;
  const double* coef;   // m*m: Winv(j,l) * a_l
  const double* cross;  // m*m: w_ll'
  int m;
  long long n_pad;
  long long fid_slot;
};

// A rank that never arrives fails the solve instead of hanging it: after
// kPeerTimeoutNs of polling the waiting kernel marks the control block
// (status 3, done) and returns; finish_solve reports JOFC_ECOMM.
constexpr unsigned long long kPeerTimeoutNs = 20ull * 1000 * 1000 * 1000;

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  return v;
}

// Wait until flag f reaches target = (epoch, t + 1).  In a consistent group
// a flag never runs ahead of the value a waiter needs (a rank raises (e, t+2)
// only after every rank's decide of (e, t), which follows this wait), so a
// larger value means the ranks disagree on the solve count -- e.g. one rank's
// solve failed validation before it took an epoch -- and the solve fails
// instead of reading another solve's products.
// Returns 0 arrived, 1 timed out, 2 epoch mismatch.
__device__ __forceinline__ int wait_flag(const unsigned long long* f, unsigned long long target) {
  unsigned long long v = ld_acquire_sys(f);
  const unsigned long long t0 = global_ns();
  while (v < target) {
    __nanosleep(32);
    if (global_ns() - t0 > kPeerTimeoutNs) return 1;
    v = ld_acquire_sys(f);
  }
  return v == target ? 0 : 2;
}

// status 3: a rank did not arrive in time; 4: the ranks' epochs disagree
__device__ __forceinline__ void peer_fail(Control* ctrl, int t, int why) {
  ctrl->status = why == 2 ? 4 : 3;
  ctrl->err_iter = t;
  ctrl->done = 1;
}

template <int D>
__global__ void __launch_bounds__(256) jofc_peer_mix_kernel(const PeerParams p) {
  Control* ctrl = p.ctrl;
  if (ctrl->done) return;
  extern __shared__ double s_sum[];  // [m][rows_cta * D]: the world's P for this CTA's objects
  __shared__ double red[8];
  __shared__ bool last;
  __shared__ int timed_out;
  const int t = ctrl->t;
  const unsigned long long target = flag_value(ctrl->epoch, t);
  double* own = p.slabs[p.rank];
  if (threadIdx.x == 0) timed_out = 0;
  __syncthreads();
  if (threadIdx.x < p.world) {
    const int w = wait_flag(reinterpret_cast<const unsigned long long*>(own + p.flag1_off) +
                                threadIdx.x, target);
    if (w) atomicMax(&timed_out, w);
  }
  __syncthreads();
  if (timed_out) {
    if (threadIdx.x == 0) peer_fail(ctrl, t, timed_out);
    return;
  }

  const long long i0 = p.row_lo + static_cast<long long>(blockIdx.x) * p.rows_cta;
  const int rows = static_cast<int>(
      max(0LL, min(static_cast<long long>(p.rows_cta), p.row_hi - i0)));
  const int per = rows * D;
  // 1. P of these objects summed over the ranks in rank order (all of a
  //    thread's peer loads in flight before the first add)
  for (int e = threadIdx.x; e < p.m * per; e += blockDim.x) {
    const int l = e / per, q = e - l * per;
    const long long off = p.p_read + (static_cast<long long>(l) * p.n_pad + i0) * D + q;
    double v[kMaxPeers];
#pragma unroll
    for (int r = 0; r < kMaxPeers; ++r)
      if (r < p.world) v[r] = ld_relaxed_sys(p.slabs[r] + off);
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < kMaxPeers; ++r)
      if (r < p.world) s += v[r];
    s_sum[e] = s;
  }
  __syncthreads();

  // 2. X_{t+1} of these objects (the W^-1 mix, accumulated from 0 in l order
  //    as proj/src/solver.cpp:63-68), stored into every rank's copy
  const long long xn = ((t + 1) & 1) ? p.x_off1 : p.x_off0;
  for (int e = threadIdx.x; e < p.m * per; e += blockDim.x) {
    const int j = e / per, q = e - j * per;
    double acc = 0.0;
    for (int l = 0; l < p.m; ++l) acc = fma(__ldg(p.coef + j * p.m + l), s_sum[l * per + q], acc);
    const long long off = xn + (static_cast<long long>(j) * p.n_pad + i0) * D + q;
    for (int r = 0; r < p.world; ++r) p.slabs[r][off] = acc;
  }

  // 3. commensurability of X_t over these objects
  const double* xc = own + ((t & 1) ? p.x_off1 : p.x_off0);
  double com = 0.0;
  for (int ii = threadIdx.x; ii < rows; ii += blockDim.x)
    com += row_commensurability<D>(xc, p.cross, p.m, p.n_pad, i0 + ii);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) com += __shfl_xor_sync(0xffffffffu, com, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = com;

  // 4. the other P region of this rank, zero for pass t + 1
  double* pz = own + p.p_zero;
  for (long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; e < p.p_len;
       e += static_cast<long long>(gridDim.x) * blockDim.x)
    pz[e] = 0.0;
  __syncthreads();

  // 5. CTA partials in a fixed order into the slot peers read; flag2 once
  //    every CTA's X stores are visible system-wide
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int w = 0; w < (blockDim.x >> 5); ++w) v += red[w];
    p.com_partials[blockIdx.x] = v;
    __threadfence_system();
    const unsigned prev = atomicAdd(&ctrl->epi_counter, 1u);
    last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence_system();
    const volatile double* vp = p.com_partials;
    double s = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) s += vp[b];
    own[p.com_off] = s;
    ctrl->epi_counter = 0;
    __threadfence_system();
    for (int q = 0; q < p.world; ++q)
      st_release_sys(reinterpret_cast<unsigned long long*>(p.slabs[q] + p.flag2_off) + p.rank,
                     target);
  }
}

// One warp: sigma_t = sum_r fidelity_r + sum_r commensurability_r (rank
// order on every rank), trace write and the stop rule.
static __global__ void __launch_bounds__(32) jofc_peer_decide_kernel(const PeerParams p) {
  Control* ctrl = p.ctrl;
  if (ctrl->done) return;
  const int t = ctrl->t;
  const unsigned long long target = flag_value(ctrl->epoch, t);
  const double* own = p.slabs[p.rank];
  double f = 0.0, c = 0.0;
  const int q = threadIdx.x;
  int w = 0;
  if (q < p.world) {
    w = wait_flag(reinterpret_cast<const unsigned long long*>(own + p.flag2_off) + q, target);
    f = ld_relaxed_sys(p.slabs[q] + p.p_read + p.fid_slot);
    c = ld_relaxed_sys(p.slabs[q] + p.com_off);
  }
  const int why = __reduce_max_sync(0xffffffffu, w);
  if (why) {
    if (threadIdx.x == 0) peer_fail(ctrl, t, why);
    return;
  }
  double fid = 0.0, com = 0.0;
  for (int r = 0; r < p.world; ++r) {
    fid += __shfl_sync(0xffffffffu, f, r);
    com += __shfl_sync(0xffffffffu, c, r);
  }
  if (threadIdx.x == 0) decide_sigma(p.trace, ctrl, t, fid + com);
}

}  // namespace jofc_gpu
