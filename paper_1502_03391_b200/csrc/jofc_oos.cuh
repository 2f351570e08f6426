// jofc_oos.cuh -- batched out-of-sample Guttman updates (sm_100a).
//
// k new objects, each with m views, embedded against a frozen in-sample
// configuration X (m x n x d).  Per point and modality j the reference
// (proj/src/oos.cpp:83-96) needs, for the current y_j,
//   r_k = [dist != 0] delta_j(k) / dist(X^(j)_k, y_j),
//   psi_j = sum_k r_k,   xi_j = sum_k (1 - r_k) X^(j)_k,
// and oos_stress (proj/src/oos.cpp:50-57) needs sum_k (delta_j(k) - dist)^2
// from the same distances, so one streaming pass over delta yields both
// (fused like the in-sample pass); the closed-form corner update
// (proj/src/oos.cpp:98-111), the commensurability term and the per-point stop
// rule (proj/src/oos.cpp:221-226) follow.
//
// Kernels (jofc_capi.cu, oos_run):
//   jofc_oos_solve_kernel    (default) the whole batch solve in ONE launch:
//                            CTAs own point ranges for every iteration, a
//                            producer warp streams delta/X chunks through a
//                            TMA ring, consumer warps run pass, fold and update
//                            (bottom of this file);
//   jofc_oos_step_kernel     one fused launch per update (pass of y_t after
//                            update step t - 1), replayed from CUDA graphs --
//                            the fallback when the persistent plan does not
//                            fit, or JOFC_OOS_KERNEL=3;
//   jofc_oos_pass_kernel / jofc_oos_pass2_kernel + jofc_oos_update_kernel
//                            the earlier two-kernel forms (JOFC_OOS_KERNEL=1/2,
//                            comparisons only).
//
// Per-update pass layout (jofc_oos_pass_kernel / jofc_oos_step_kernel): CTA =
// 8 warps = 8 points of one modality (blockIdx.y) and one of kOosSplits slices
// of the in-sample range (blockIdx.z); X^(j) streams through two shared-memory
// chunk buffers (512 rows each, filled by the TMA bulk engine, double
// buffered) shared by the 8 warps; lanes stride the n in-sample rows
// (coalesced delta reads, 4 in flight per lane), warp shuffles finish the sums.
#pragma once

#include "jofc_kernels.cuh"

namespace jofc_gpu {

struct OosPoint {
  int t;
  int done;
  int iterations;
  int status;  // 0 ok, 2 non-finite stress
};

struct OosParams {
  const double* x;       // m x n x d
  const double* deltas;  // k x m x n
  double* y0;            // ping-pong k x m x d
  double* y1;
  double* part;          // k x m x (d + 2): psi, fid, xi[d]
  OosPoint* st;
  double* traces;        // k x (max_it + 1) or null
  int k, m;
  long long n;
  double w, eps, term_count;
  int max_it;
  int fixed;
  unsigned* done_count;  // points finished (the host stops enqueuing at k)
  // v2 pass (lanes = points): delta transposed to [j][g][n][32], g = point group
  const double* deltas_t;
  int groups;
  // fused step kernel: launch index = *base + local_t (base: one device word
  // set per replayed chunk of launches; local_t: the launch's place in the
  // captured chunk), the previous stress per point by parity (2 x k)
  const unsigned* base;
  int local_t;
  double* prev2;
};

// The first launch index of a replayed chunk of fused steps (the value rides
// in the kernel parameter: no host staging buffer).
static __global__ void jofc_oos_set_base_kernel(unsigned* base, unsigned v) { *base = v; }

constexpr int kOosWarps = 8;
constexpr int kOosChunk = 512;
constexpr int kOosSplits = 4;  // n-range slices per (point, modality): 4x the warps in flight
#ifndef JOFC_OOS_UNROLL
#define JOFC_OOS_UNROLL 4
#endif
constexpr int kOosUnroll = JOFC_OOS_UNROLL;  // delta entries per lane per step

// X staging: two chunk buffers filled by the TMA bulk engine (double
// buffered: chunk c + 2 streams in while chunk c + 1 is consumed).  Each buffer
// has 2 spare doubles: a chunk's global start is rounded down to 16 bytes.
template <int D>
__host__ __device__ constexpr int oos_buf_doubles() { return kOosChunk * D + 2; }
template <int D>
__host__ __device__ constexpr int oos_smem_bytes() { return 128 + 2 * oos_buf_doubles<D>() * 8; }

template <int D>
__global__ void __launch_bounds__(kOosWarps * 32) jofc_oos_pass_kernel(const OosParams p) {
  extern __shared__ __align__(128) unsigned char oos_smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(oos_smem);
  double* xbuf = reinterpret_cast<double*>(oos_smem + 128);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pt = blockIdx.x * kOosWarps + warp;
  const int j = blockIdx.y;
  const long long k_lo = p.n * blockIdx.z / gridDim.z;
  const long long k_hi = p.n * (blockIdx.z + 1) / gridDim.z;
  const int nch = static_cast<int>((k_hi - k_lo + kOosChunk - 1) / kOosChunk);
  bool active = pt < p.k;
  int t = 0;
  if (active) {
    const OosPoint s = p.st[pt];
    active = !s.done;
    t = s.t;
  }
  double y[D];
  const double* yb = ((t & 1) ? p.y1 : p.y0) + (static_cast<long long>(pt) * p.m + j) * D;
#pragma unroll
  for (int c = 0; c < D; ++c) y[c] = active ? yb[c] : 0.0;
  const long long xbase = static_cast<long long>(j) * p.n * D;  // X^(j) in doubles
  const double* dl = p.deltas + (static_cast<long long>(pt) * p.m + j) * p.n;
  auto issue = [&](int ch) {  // thread 0: chunk ch -> buffer ch & 1
    const long long k0 = k_lo + static_cast<long long>(ch) * kOosChunk;
    const int rows = static_cast<int>(min(static_cast<long long>(kOosChunk), k_hi - k0));
    const long long first = xbase + k0 * D;
    const long long start = first & ~1LL;  // 16-byte aligned
    const uint32_t bytes = static_cast<uint32_t>(((first - start + rows * D) * 8 + 15) & ~15LL);
    mbar_expect_tx(&bar[ch & 1], bytes);
    bulk_g2s(xbuf + (ch & 1) * oos_buf_doubles<D>(), p.x + start, bytes, &bar[ch & 1]);
  };
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
    if (nch > 0) issue(0);
    if (nch > 1) issue(1);
  }
  __syncthreads();
  double psi[2] = {0.0, 0.0}, fid[2] = {0.0, 0.0}, xi[2][D];
#pragma unroll
  for (int c = 0; c < D; ++c) xi[0][c] = xi[1][c] = 0.0;
  for (int ch = 0; ch < nch; ++ch) {
    const long long k0 = k_lo + static_cast<long long>(ch) * kOosChunk;
    const int rows = static_cast<int>(min(static_cast<long long>(kOosChunk), k_hi - k0));
    mbar_wait(&bar[ch & 1], (ch >> 1) & 1);
    const double* xs = xbuf + (ch & 1) * oos_buf_doubles<D>() + ((xbase + k0 * D) & 1);
    if (active) {
      // kOosUnroll delta loads in flight per lane, two accumulator sets
      for (int kk0 = lane; kk0 < rows; kk0 += 32 * kOosUnroll) {
        double dv[kOosUnroll];
#pragma unroll
        for (int u = 0; u < kOosUnroll; ++u) {
          const int kk = kk0 + 32 * u;
          dv[u] = (kk < rows) ? dl[k0 + kk] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kOosUnroll; ++u) {
          const int kk = kk0 + 32 * u;
          if (kk >= rows) break;
          double s = 0.0, xk[D];
#pragma unroll
          for (int c = 0; c < D; ++c) {
            xk[c] = xs[kk * D + c];
            const double df = xk[c] - y[c];
            s = (c == 0) ? df * df : fma(df, df, s);
          }
          const double inv = (s > 0.0) ? rsqrt_nr(s) : 0.0;
          const double r = dv[u] * inv;
          const double resid = dv[u] - s * inv;
          const int a = u & 1;
          fid[a] = fma(resid, resid, fid[a]);
          psi[a] += r;
          const double cf = 1.0 - r;
#pragma unroll
          for (int c = 0; c < D; ++c) xi[a][c] = fma(cf, xk[c], xi[a][c]);
        }
      }
    }
    __syncthreads();  // every warp is done with this buffer
    if (threadIdx.x == 0 && ch + 2 < nch) {
      fence_proxy_async_smem();
      issue(ch + 2);
    }
  }
  if (!active) return;
  double spsi = psi[0] + psi[1], sfid = fid[0] + fid[1], sxi[D];
#pragma unroll
  for (int c = 0; c < D; ++c) sxi[c] = xi[0][c] + xi[1][c];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    spsi += __shfl_xor_sync(0xffffffffu, spsi, o);
    sfid += __shfl_xor_sync(0xffffffffu, sfid, o);
#pragma unroll
    for (int c = 0; c < D; ++c) sxi[c] += __shfl_xor_sync(0xffffffffu, sxi[c], o);
  }
  if (lane == 0) {  // slices of the n range meet in `part` (zeroed by the update kernel)
    double* out = p.part + (static_cast<long long>(pt) * p.m + j) * (D + 2);
    atomicAdd(out, spsi);
    atomicAdd(out + 1, sfid);
#pragma unroll
    for (int c = 0; c < D; ++c) atomicAdd(out + 2 + c, sxi[c]);
  }
}

template <int D>
__global__ void __launch_bounds__(128) jofc_oos_update_kernel(const OosParams p) {
  const int pt = blockIdx.x * blockDim.x + threadIdx.x;
  if (pt >= p.k) return;
  OosPoint st = p.st[pt];
  if (st.done) return;
  const int t = st.t, m = p.m;
  const double* y = ((t & 1) ? p.y1 : p.y0) + static_cast<long long>(pt) * m * D;
  double* yn = ((t & 1) ? p.y0 : p.y1) + static_cast<long long>(pt) * m * D;
  const double* part = p.part + static_cast<long long>(pt) * m * (D + 2);
  double fid = 0.0, com = 0.0;
  double xi_sum[D], psi_y[D];
#pragma unroll
  for (int c = 0; c < D; ++c) xi_sum[c] = psi_y[c] = 0.0;
  for (int j = 0; j < m; ++j) {
    fid += part[j * (D + 2) + 1];
    const double psi = part[j * (D + 2)];
#pragma unroll
    for (int c = 0; c < D; ++c) {
      xi_sum[c] += part[j * (D + 2) + 2 + c];
      psi_y[c] = fma(psi, y[j * D + c], psi_y[c]);
    }
    for (int i2 = j + 1; i2 < m; ++i2) {
#pragma unroll
      for (int c = 0; c < D; ++c) {
        const double df = y[j * D + c] - y[i2 * D + c];
        com = fma(df, df, com);
      }
    }
  }
  const double sigma = fid + p.w * com;
  if (p.traces) p.traces[static_cast<long long>(pt) * (p.max_it + 1) + t] = sigma;
  if (!isfinite(sigma)) {
    st.status = 2;
    st.done = 1;
    st.iterations = t;
    p.st[pt] = st;
    atomicAdd(p.done_count, 1u);
    return;
  }
  st.iterations = t;
  double* prev_slot = p.part + static_cast<long long>(p.k) * m * (D + 2) + pt;
  if (t >= 1 && !p.fixed && (*prev_slot - sigma) / p.term_count < p.eps) st.done = 1;
  if (t >= p.max_it) st.done = 1;
  if (st.done) atomicAdd(p.done_count, 1u);
  *prev_slot = sigma;
  if (!st.done) {
    const double nn = static_cast<double>(p.n);
    const double mw = static_cast<double>(m) * p.w;
    const double direct = 1.0 / (nn + mw);
    const double spread = p.w / (nn * (nn + mw));
    for (int j = 0; j < m; ++j) {
      const double psi = part[j * (D + 2)];
#pragma unroll
      for (int c = 0; c < D; ++c)
        yn[j * D + c] = direct * (part[j * (D + 2) + 2 + c] + psi * y[j * D + c]) +
                        spread * (xi_sum[c] + psi_y[c]);
    }
  }
  double* pz = p.part + static_cast<long long>(pt) * m * (D + 2);
  for (int e = 0; e < m * (D + 2); ++e) pz[e] = 0.0;
  st.t = t + 1;
  p.st[pt] = st;
}

// ------------------------------------------------------------- pass, v2
// Lanes = points.  The batch's delta rows are transposed once per solve to
// [modality j][point group g][in-sample row k][32 points] (jofc_oos_transpose_
// kernel), so a chunk of R rows x 32 points is one contiguous 1-D bulk copy;
// the matching R rows of X^(j) ride along.  CTA = (point group, modality,
// slice of the in-sample range); its 8 warps take the chunk's rows
// round-robin, every lane computing its own point's entry for the row
// (x_k a shared-memory broadcast, delta a conflict-free 32-wide read) and
// keeping psi, the fidelity and xi in registers -- no per-entry reductions,
// and the ring keeps ~70 KB of delta in flight per CTA (the v1 kernel, one
// warp per point with lanes over rows, was L2-latency bound: long-scoreboard
// 40% of its samples).  The 8 warps' sums meet in shared memory; one add per
// (point, modality, value) and CTA goes to `part`.
#ifndef JOFC_OOS2_ROWS
#define JOFC_OOS2_ROWS 64
#endif
#ifndef JOFC_OOS2_STAGES
#define JOFC_OOS2_STAGES 4
#endif
constexpr int kOos2Rows = JOFC_OOS2_ROWS;
constexpr int kOos2Warps = 8;
template <int D>
__host__ __device__ constexpr int oos2_stages() { return D >= 8 ? 3 : JOFC_OOS2_STAGES; }
template <int D>
__host__ __device__ constexpr int oos2_x_doubles() { return kOos2Rows * D + 2; }
template <int D>
__host__ __device__ constexpr int oos2_smem_bytes() {
  return 128 + oos2_stages<D>() * (kOos2Rows * 32 + oos2_x_doubles<D>()) * 8 +
         kOos2Warps * (D + 2) * 32 * 8;
}

static __global__ void __launch_bounds__(256) jofc_oos_transpose_kernel(const double* __restrict__ d,
                                                                        double* __restrict__ dt,
                                                                        int k, int m, long long n,
                                                                        int groups) {
  // CTA: (modality j, group g, 32-row tile of n); d is k x m x n
  __shared__ double tile[32][33];
  const int j = blockIdx.y / groups, g = blockIdx.y % groups;
  const long long k0 = static_cast<long long>(blockIdx.x) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int q = ty; q < 32; q += 8) {  // read point q's rows k0 .. k0 + 31
    const int pt = g * 32 + q;
    const long long kk = k0 + tx;
    tile[q][tx] = (pt < k && kk < n) ? d[(static_cast<long long>(pt) * m + j) * n + kk] : 0.0;
  }
  __syncthreads();
  double* out = dt + ((static_cast<long long>(j) * groups + g) * n) * 32;
  for (int r = ty; r < 32; r += 8) {
    const long long kk = k0 + r;
    if (kk < n) out[kk * 32 + tx] = tile[tx][r];
  }
}

template <int D>
__global__ void __launch_bounds__(kOos2Warps * 32) jofc_oos_pass2_kernel(const OosParams p) {
  constexpr int kSt = oos2_stages<D>();
  constexpr int R = kOos2Rows;
  constexpr int XD = oos2_x_doubles<D>();
  extern __shared__ __align__(128) unsigned char oos2_smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(oos2_smem);
  unsigned* done = reinterpret_cast<unsigned*>(oos2_smem + 64);
  double* sd = reinterpret_cast<double*>(oos2_smem + 128);
  double* sx = sd + kSt * R * 32;
  double* sred = sx + kSt * XD;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x % p.groups, j = blockIdx.x / p.groups;
  const int pt = g * 32 + lane;
  bool active = pt < p.k;
  int t = 0;
  if (active) {
    const OosPoint st = p.st[pt];
    active = !st.done;
    t = st.t;
  }
  if (!__any_sync(0xffffffffu, active)) return;  // (the same 32 points in every warp)
  const long long k_lo = p.n * blockIdx.y / gridDim.y;
  const long long k_hi = p.n * (blockIdx.y + 1) / gridDim.y;
  const int nch = static_cast<int>((k_hi - k_lo + R - 1) / R);
  double y[D];
  const double* yb = ((t & 1) ? p.y1 : p.y0) + (static_cast<long long>(pt) * p.m + j) * D;
#pragma unroll
  for (int c = 0; c < D; ++c) y[c] = active ? yb[c] : 0.0;
  const double* dt = p.deltas_t + ((static_cast<long long>(j) * p.groups + g) * p.n) * 32;
  const long long xbase = static_cast<long long>(j) * p.n * D;
  auto issue = [&](int ch) {
    const int st = ch % kSt;
    const long long k0 = k_lo + static_cast<long long>(ch) * R;
    const int rows = static_cast<int>(min(static_cast<long long>(R), k_hi - k0));
    const uint32_t bd = static_cast<uint32_t>(rows) * 32u * 8u;
    const long long first = xbase + k0 * D;
    const long long start = first & ~1LL;  // 16-byte aligned
    const uint32_t bx = static_cast<uint32_t>(((first - start + rows * D) * 8 + 15) & ~15LL);
    mbar_expect_tx(&full[st], bd + bx);
    bulk_g2s(sd + st * R * 32, dt + k0 * 32, bd, &full[st]);
    bulk_g2s(sx + st * XD, p.x + start, bx, &full[st]);
  };
  if (threadIdx.x == 0) {
    for (int st = 0; st < kSt; ++st) {
      mbar_init(&full[st], 1);
      done[st] = 0;
    }
    mbar_fence_init();
    for (int ch = 0; ch < nch && ch < kSt; ++ch) issue(ch);
  }
  __syncthreads();
  double psi = 0.0, fid = 0.0, xi[D];
#pragma unroll
  for (int c = 0; c < D; ++c) xi[c] = 0.0;
  for (int ch = 0; ch < nch; ++ch) {
    const int st = ch % kSt;
    const long long k0 = k_lo + static_cast<long long>(ch) * R;
    const int rows = static_cast<int>(min(static_cast<long long>(R), k_hi - k0));
    mbar_wait(&full[st], static_cast<uint32_t>((ch / kSt) & 1));
    const double* xs = sx + st * XD + ((xbase + k0 * D) & 1);
    const double* ds = sd + st * R * 32 + lane;
#pragma unroll 4
    for (int rr = warp; rr < rows; rr += kOos2Warps) {
      const double dv = ds[rr * 32];
      double s = 0.0, xk[D];
#pragma unroll
      for (int c = 0; c < D; ++c) {
        xk[c] = xs[rr * D + c];
        const double df = xk[c] - y[c];
        s = (c == 0) ? df * df : fma(df, df, s);
      }
      const double inv = (s > 0.0) ? rsqrt_nr(s) : 0.0;  // dist == 0 guard (proj/src/oos.cpp:88)
      const double r = dv * inv;
      const double resid = dv - s * inv;
      fid = fma(resid, resid, fid);
      psi += r;
      const double cf = 1.0 - r;
#pragma unroll
      for (int c = 0; c < D; ++c) xi[c] = fma(cf, xk[c], xi[c]);
    }
    // the last warp done with the stage refills it (formal release/acquire as
    // the in-sample ring)
    __syncwarp();
    if (lane == 0 && smem_arrive_count(&done[st]) == kOos2Warps - 1) {
      done[st] = 0;
      fence_acquire_cta();
      if (ch + kSt < nch) {
        fence_proxy_async_smem();
        issue(ch + kSt);
      }
    }
  }
  // the 8 warps' partial sums of each point, then one add per value to `part`
  double* mine = sred + warp * (D + 2) * 32 + lane;
  mine[0] = psi;
  mine[32] = fid;
#pragma unroll
  for (int c = 0; c < D; ++c) mine[(2 + c) * 32] = xi[c];
  __syncthreads();
  if (active) {
    for (int v = warp; v < D + 2; v += kOos2Warps) {
      double acc = 0.0;
#pragma unroll
      for (int w = 0; w < kOos2Warps; ++w) acc += sred[(w * (D + 2) + v) * 32 + lane];
      red_add(p.part + (static_cast<long long>(pt) * p.m + j) * (D + 2) + v, acc);
    }
  }
}

// ------------------------------------------------------------- fused step
// One kernel per Guttman update instead of pass + update: launch t first
// applies update step s = t - 1 of every point its CTA touches -- sigma_s from
// the triple-buffered partials part[s % 3] (proj/src/oos.cpp:50-70), the stop
// rule (:221-226) and y_t (:98-111), each CTA redundantly for its own points
// (a few dozen FP64 operations) -- then streams the pass for y_t into
// part[t % 3].  The CTA of modality 0 and slice 0 of a point is its
// bookkeeper: trace, previous stress (by parity), state, y_t to memory (the
// next launch's start), part[(t + 1) % 3] zeroed (last read by launch t - 1).
// The launch index is *base + local_t (a captured chunk of launches is
// replayed with a new base).  The X chunks of the pass are requested before
// the update step, so its loads overlap the first TMA copies.  Launch 0 is a
// pure pass; launch max_it + 1 only finishes the points.  Decisions are
// identical in every CTA: same inputs, same order.
template <int D>
__global__ void __launch_bounds__(kOosWarps * 32) jofc_oos_step_kernel(const OosParams p) {
  extern __shared__ __align__(128) unsigned char oos_smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(oos_smem);
  double* xbuf = reinterpret_cast<double*>(oos_smem + 128);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pt = blockIdx.x * kOosWarps + warp;
  const int j = blockIdx.y;
  const int t = static_cast<int>(*p.base) + p.local_t;
  const long long kmd = static_cast<long long>(p.k) * p.m * (D + 2);
  const long long k_lo = p.n * blockIdx.z / gridDim.z;
  const long long k_hi = p.n * (blockIdx.z + 1) / gridDim.z;
  const int nch = static_cast<int>((k_hi - k_lo + kOosChunk - 1) / kOosChunk);
  const long long xbase = static_cast<long long>(j) * p.n * D;
  auto issue = [&](int ch) {
    const long long k0 = k_lo + static_cast<long long>(ch) * kOosChunk;
    const int rows = static_cast<int>(min(static_cast<long long>(kOosChunk), k_hi - k0));
    const long long first = xbase + k0 * D;
    const long long start = first & ~1LL;
    const uint32_t bytes = static_cast<uint32_t>(((first - start + rows * D) * 8 + 15) & ~15LL);
    mbar_expect_tx(&bar[ch & 1], bytes);
    bulk_g2s(xbuf + (ch & 1) * oos_buf_doubles<D>(), p.x + start, bytes, &bar[ch & 1]);
  };
  // every CTA runs the chunk ring (a CTA whose points are all done only
  // drains it): the X copies start before the update step's loads
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
    if (nch > 0) issue(0);
    if (nch > 1) issue(1);
  }
  bool active = pt < p.k && !p.st[pt].done;
  double y[D];
#pragma unroll
  for (int c = 0; c < D; ++c) y[c] = 0.0;
  if (active && t == 0) {
    const double* yb = p.y0 + (static_cast<long long>(pt) * p.m + j) * D;
#pragma unroll
    for (int c = 0; c < D; ++c) y[c] = yb[c];
  } else if (active) {
    // ---- update step s = t - 1 (every lane, same values)
    const int s = t - 1;
    const int m = p.m;
    const double* part = p.part + (s % 3) * kmd + static_cast<long long>(pt) * m * (D + 2);
    const double* yp = ((s & 1) ? p.y1 : p.y0) + static_cast<long long>(pt) * m * D;
    double fid = 0.0, com = 0.0, xi_sum[D], psi_y[D];
#pragma unroll
    for (int c = 0; c < D; ++c) xi_sum[c] = psi_y[c] = 0.0;
    for (int l = 0; l < m; ++l) {
      fid += part[l * (D + 2) + 1];
      const double psi = part[l * (D + 2)];
#pragma unroll
      for (int c = 0; c < D; ++c) {
        xi_sum[c] += part[l * (D + 2) + 2 + c];
        psi_y[c] = fma(psi, yp[l * D + c], psi_y[c]);
      }
      for (int l2 = l + 1; l2 < m; ++l2) {
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const double df = yp[l * D + c] - yp[l2 * D + c];
          com = fma(df, df, com);
        }
      }
    }
    const double sigma = fid + p.w * com;
    bool finished = false;
    int status = 0;
    if (!isfinite(sigma)) {
      finished = true;
      status = 2;
    } else {
      if (s >= 1 && !p.fixed && (p.prev2[((s - 1) & 1) * p.k + pt] - sigma) / p.term_count < p.eps)
        finished = true;
      if (s >= p.max_it) finished = true;
    }
    const bool keeper = j == 0 && blockIdx.z == 0 && lane == 0;
    const double nn = static_cast<double>(p.n);
    const double mw = static_cast<double>(m) * p.w;
    const double direct = 1.0 / (nn + mw);
    const double spread = p.w / (nn * (nn + mw));
    if (!finished) {
      const double psi_j = part[j * (D + 2)];
#pragma unroll
      for (int c = 0; c < D; ++c)
        y[c] = direct * (part[j * (D + 2) + 2 + c] + psi_j * yp[j * D + c]) +
               spread * (xi_sum[c] + psi_y[c]);
    }
    if (keeper) {
      if (p.traces) p.traces[static_cast<long long>(pt) * (p.max_it + 1) + s] = sigma;
      p.prev2[(s & 1) * p.k + pt] = sigma;
      double* yn = ((t & 1) ? p.y1 : p.y0) + static_cast<long long>(pt) * m * D;
      if (!finished)
        for (int l = 0; l < m; ++l) {
          const double psi = part[l * (D + 2)];
#pragma unroll
          for (int c = 0; c < D; ++c)
            yn[l * D + c] = direct * (part[l * (D + 2) + 2 + c] + psi * yp[l * D + c]) +
                            spread * (xi_sum[c] + psi_y[c]);
        }
      double* pz = p.part + ((t + 1) % 3) * kmd + static_cast<long long>(pt) * m * (D + 2);
      for (int e = 0; e < m * (D + 2); ++e) pz[e] = 0.0;
      OosPoint st = p.st[pt];
      st.t = t;
      st.iterations = s;
      if (finished) {
        st.done = 1;
        st.status = status;
        atomicAdd(p.done_count, 1u);
      }
      p.st[pt] = st;
    }
    active = !finished;
  }
  // ---- pass for y_t (the v1 layout: warp = point, lanes over rows)
  const double* dl = p.deltas + (static_cast<long long>(min(pt, p.k - 1)) * p.m + j) * p.n;
  __syncthreads();
  {
    double psi[2] = {0.0, 0.0}, fid[2] = {0.0, 0.0}, xi[2][D];
#pragma unroll
    for (int c = 0; c < D; ++c) xi[0][c] = xi[1][c] = 0.0;
    for (int ch = 0; ch < nch; ++ch) {
      const long long k0 = k_lo + static_cast<long long>(ch) * kOosChunk;
      const int rows = static_cast<int>(min(static_cast<long long>(kOosChunk), k_hi - k0));
      mbar_wait(&bar[ch & 1], (ch >> 1) & 1);
      const double* xs = xbuf + (ch & 1) * oos_buf_doubles<D>() + ((xbase + k0 * D) & 1);
      if (active) {
        for (int kk0 = lane; kk0 < rows; kk0 += 32 * kOosUnroll) {
          double dv[kOosUnroll];
#pragma unroll
          for (int u = 0; u < kOosUnroll; ++u) {
            const int kk = kk0 + 32 * u;
            dv[u] = (kk < rows) ? dl[k0 + kk] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < kOosUnroll; ++u) {
            const int kk = kk0 + 32 * u;
            if (kk >= rows) break;
            double sq = 0.0, xk[D];
#pragma unroll
            for (int c = 0; c < D; ++c) {
              xk[c] = xs[kk * D + c];
              const double df = xk[c] - y[c];
              sq = (c == 0) ? df * df : fma(df, df, sq);
            }
            const double inv = (sq > 0.0) ? rsqrt_nr(sq) : 0.0;  // dist == 0 guard
            const double r = dv[u] * inv;
            const double resid = dv[u] - sq * inv;
            const int a = u & 1;
            fid[a] = fma(resid, resid, fid[a]);
            psi[a] += r;
            const double cf = 1.0 - r;
#pragma unroll
            for (int c = 0; c < D; ++c) xi[a][c] = fma(cf, xk[c], xi[a][c]);
          }
        }
      }
      __syncthreads();  // every warp is done with this buffer
      if (threadIdx.x == 0 && ch + 2 < nch) {
        fence_proxy_async_smem();
        issue(ch + 2);
      }
    }
    if (active) {
      double spsi = psi[0] + psi[1], sfid = fid[0] + fid[1], sxi[D];
#pragma unroll
      for (int c = 0; c < D; ++c) sxi[c] = xi[0][c] + xi[1][c];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        spsi += __shfl_xor_sync(0xffffffffu, spsi, o);
        sfid += __shfl_xor_sync(0xffffffffu, sfid, o);
#pragma unroll
        for (int c = 0; c < D; ++c) sxi[c] += __shfl_xor_sync(0xffffffffu, sxi[c], o);
      }
      if (lane == 0) {
        double* out = p.part + (t % 3) * kmd + (static_cast<long long>(pt) * p.m + j) * (D + 2);
        red_add(out, spsi);
        red_add(out + 1, sfid);
#pragma unroll
        for (int c = 0; c < D; ++c) red_add(out + 2 + c, sxi[c]);
      }
    }
  }
}

// ------------------------------------------------------ persistent solve
// The whole out-of-sample batch solve in ONE launch.  Points are independent
// (proj/src/oos.cpp:180-229 runs one oos_embed per point), so each CTA (one
// per SM) owns a contiguous range of at most G points for every iteration --
// no grid-wide synchronisation, no per-iteration launches.  A producer warp
// streams chunks of R in-sample rows through a TMA ring: for modality l, the
// G points' delta rows (one bulk copy: the batch's delta is permuted into
// ring order once, jofc_oos_permute_kernel) and the rows of X^(l) (one
// more), in the order (iteration, modality, chunk); delta and X do not
// depend on y, so the ring runs on across the update steps.  8 consumer
// warps, per iteration:
//   pass    lanes over rows; a lane keeps Q points of its warp's slot in
//           registers (register u holds point u ^ pi(lane): the fold below is
//           a select-free reduce-scatter) and, per row and point:
//           r = [dist != 0] delta / dist, psi += r, fidelity += (delta -
//           dist)^2, xi' += r x_k (xi = sum_k x_k - xi', one FP64 operation
//           per entry less than (1 - r) x_k);
//   fold    per modality: lanes -> warp (log2 Q reduce-scatter levels + a
//           butterfly), warps -> point in a fixed order, into part[l][q];
//   update  thread q: sigma_t (proj/src/oos.cpp:50-70), the stop rule
//           (:221-226) and y_{t+1} of every modality (:98-111); the trace,
//           the state and the final y go to global memory.
// Ring protocol: full[s] (TMA completion, waited by the consumers), empty[s]
// (one release-arrive per consumer warp, acquired by the producer before
// its fence.proxy.async and the bulk copies that overwrite the stage).
// (9 warps: 168 registers per thread, 4 points per lane at d <= 4.  Measured
// per C5 update (batch of 1000, `scripts/gpu_oosp_ab.sh`): 8 consumers x 4
// points 24.7 us; 16 x 2 26.5 us; 12 x 2 or 12 x 4 (128 registers) 27-29 us;
// 24 x 2 (72 registers) 35.7 us; two rows per lane in flight: slower)
#ifndef JOFC_OOSP_CONSUMERS
#define JOFC_OOSP_CONSUMERS 8
#endif
constexpr int kOospConsumers = JOFC_OOSP_CONSUMERS;     // consumer warps
constexpr int kOospThreads = (kOospConsumers + 1) * 32;  // + the producer warp
constexpr int kOospMaxStages = 6;
#ifndef JOFC_OOSP_UNROLL
#define JOFC_OOSP_UNROLL 1
#endif
constexpr int kOospUnroll = JOFC_OOSP_UNROLL;  // rows per lane in flight (experiments)

// Points per warp slot (a power of 2): Q (D + 2) accumulators and Q D
// coordinates of y per lane (<= 168 registers at 9 warps).
template <int D>
__host__ __device__ constexpr int oosp_q() {
#ifdef JOFC_OOSP_Q
  return D <= 4 ? JOFC_OOSP_Q : 1;  // (experiments)
#else
  return D <= 4 ? 4 : (D <= 8 ? 2 : 1);
#endif
}

struct OospParams {
  const double* x;       // m x n x D (the frozen in-sample configuration)
  const double* deltas;  // k x m x n
  const double* ystart;  // k x m x D
  double* yout0;         // final y of a point -> buffer (iterations & 1)
  double* yout1;
  double* traces;        // k x (max_it + 1)
  OosPoint* st;
  int k, m;
  long long n;
  double w, eps, term_count;
  int max_it, fixed;
  int ncta;    // CTA b owns points [b k / ncta, (b + 1) k / ncta)
  int G;       // max points per CTA
  int S;       // point slots (divides kOospConsumers): point q -> slot q % S, register q / S
  int R;       // rows per chunk (even)
  int stages;  // ring depth (<= kOospMaxStages)
  int nch;     // chunks per modality pass, ceil(n / R)
  unsigned stage_doubles;  // G R delta + (R D + 2) X
  // delta rows in ring order (jofc_oos_permute_kernel): for CTA b, modality
  // l, chunk ch one contiguous G x R block (point-major, zero padded)
  const double* dperm;
  // dynamic shared-memory layout (byte offsets from the base)
  unsigned off_ring, off_part, off_y, off_red, off_misc;
};

__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kOospConsumers * 32) : "memory");
}

// Consumer-wide OR (named barrier 1, the producer warp excluded).
__device__ __forceinline__ int consumers_or(int v) {
  int r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.s32 p, %1, 0;\n\t"
      "bar.red.or.pred q, 1, %2, p;\n\t"
      "selp.s32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"(v), "n"(kOospConsumers * 32)
      : "memory");
  return r;
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// delta (k x m x n) -> the persistent solve's ring order: block
// (b, l, ch) = rows [ch R, ch R + R) of modality l for CTA b's G point slots,
// point-major, zeros past n and past the CTA's points.  Once per batch.
static __global__ void __launch_bounds__(256) jofc_oos_permute_kernel(const double* __restrict__ d,
                                                                      double* __restrict__ out,
                                                                      int k, int m, long long n,
                                                                      int ncta, int G, int R,
                                                                      int nch) {
  // CTA = one segment (b, l, ch, q): R consecutive doubles of the output
  const long long seg = blockIdx.x;
  const int q = static_cast<int>(seg % G);
  long long rest = seg / G;
  const int ch = static_cast<int>(rest % nch);
  rest /= nch;
  const int l = static_cast<int>(rest % m);
  const int b = static_cast<int>(rest / m);
  const int p_lo = static_cast<int>(static_cast<long long>(b) * k / ncta);
  const int g = static_cast<int>(static_cast<long long>(b + 1) * k / ncta) - p_lo;
  const long long row0 = static_cast<long long>(ch) * R;
  const double* src = d + (static_cast<long long>(p_lo + q) * m + l) * n + row0;
  double* dst = out + seg * R;
  const long long rows = (q < g) ? min(static_cast<long long>(R), n - row0) : 0;
  for (int r = threadIdx.x; r < R; r += blockDim.x) dst[r] = (r < rows) ? __ldcs(src + r) : 0.0;
}

template <int D>
__global__ void __launch_bounds__(kOospThreads, 1) jofc_oos_solve_kernel(const OospParams p) {
  constexpr int Q = oosp_q<D>();
  constexpr int V = D + 2;  // per (point, modality): psi, fidelity, xi[D]
  constexpr int kLanesPerPt = 32 / Q;  // lanes that end up holding one point's sums
  extern __shared__ __align__(128) unsigned char oosp_smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(oosp_smem);       // kOospMaxStages
  uint64_t* empty = full + kOospMaxStages;                         // kOospMaxStages
  volatile int* stop = reinterpret_cast<volatile int*>(empty + kOospMaxStages);
  volatile long long* consumed = reinterpret_cast<volatile long long*>(oosp_smem + 112);
  double* ring = reinterpret_cast<double*>(oosp_smem + p.off_ring);
  double* part = reinterpret_cast<double*>(oosp_smem + p.off_part);  // m x G x V
  double* ybuf = reinterpret_cast<double*>(oosp_smem + p.off_y);     // 2 x G x m x D
  double* sred = reinterpret_cast<double*>(oosp_smem + p.off_red);   // warps x Q x V
  double* prev = reinterpret_cast<double*>(oosp_smem + p.off_misc);  // G: sigma_{t-1}
  double* sx = prev + p.G;                                           // m x D: sum_k x_k
  int* pdone = reinterpret_cast<int*>(sx + p.m * D);                 // G

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = p.m, kSt = p.stages;
  const int p_lo = static_cast<int>(static_cast<long long>(blockIdx.x) * p.k / p.ncta);
  const int g = static_cast<int>(static_cast<long long>(blockIdx.x + 1) * p.k / p.ncta) - p_lo;
  const long long n = p.n;
  const int R = p.R, nch = p.nch;
  const long long total_chunks = static_cast<long long>(p.max_it + 1) * m * nch;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kSt; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kOospConsumers);
    }
    *stop = 0;
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == kOospConsumers) {
    // ---- producer: chunk gc (order: iteration, modality, rows) into stage
    // gc % kSt once the consumers released its previous use: the CTA's G x R
    // delta block of the permuted copy, then the X^(l) rows (started at the
    // even index below them: 16-byte aligned bulk copies)
    if (lane != 0) return;
    long long gc = 0;
    int stg = 0;
    uint32_t ph = 0;  // (gc / kSt) & 1
    for (int l = 0, ch = 0; gc < total_chunks; ++gc) {
      if (gc >= kSt) {
        bool ok;
        // (the stage's previous use, chunk gc - kSt, completed phase ph ^ 1)
        while (!(ok = mbar_try_wait(&empty[stg], ph ^ 1u)) && !*stop) {
        }
        if (!ok) break;  // the solve ended: nothing more is consumed
        fence_proxy_async_smem();
      }
      // two bulk copies per chunk: the TMA engine's cost is per copy (one
      // 4 KB copy per point measured ~0.9 us per chunk whatever its size)
      const long long k0 = static_cast<long long>(ch) * R;
      const int rows = static_cast<int>(min(static_cast<long long>(R), n - k0));
      double* base = ring + static_cast<long long>(stg) * p.stage_doubles;
      const long long xfirst = (static_cast<long long>(l) * n + k0) * D;
      const uint32_t xbytes = static_cast<uint32_t>((((xfirst & 1) + rows * D) * 8 + 15) & ~15LL);
      const uint32_t dbytes = static_cast<uint32_t>(p.G) * R * 8;
      mbar_expect_tx(&full[stg], xbytes + dbytes);
      bulk_g2s(base, p.dperm + ((static_cast<long long>(blockIdx.x) * m + l) * nch + ch) * p.G * R,
               dbytes, &full[stg]);
      bulk_g2s(base + static_cast<long long>(p.G) * R, p.x + (xfirst & ~1LL), xbytes, &full[stg]);
      if (++stg == kSt) {
        stg = 0;
        ph ^= 1u;
      }
      if (++ch == nch) {
        ch = 0;
        if (++l == m) l = 0;
      }
    }
    // drain: every chunk issued but never consumed must land before the CTA
    // (and its shared memory) goes away
    while (!*stop) {
    }
    __threadfence_block();
    for (long long q = *consumed; q < gc; ++q)
      mbar_wait(&full[q % kSt], static_cast<uint32_t>((q / kSt) & 1));
    return;
  }

  // ---- consumers
  const int S = p.S, WS = kOospConsumers / S;
  const int slot = warp % S, wi = warp / S;
  const int pi = lane / kLanesPerPt;  // this lane's point permutation (0 .. Q-1)
  constexpr int kT = kOospConsumers * 32;
  for (int e = threadIdx.x; e < g * m * D; e += kT)
    ybuf[e] = p.ystart[static_cast<long long>(p_lo) * m * D + e];
  for (int q = threadIdx.x; q < g; q += kT) pdone[q] = 0;
  // sum_k x_k of every modality (fixed order; warp l sums modality l, ...)
  for (int l = warp; l < m; l += kOospConsumers) {
    double a[D];
#pragma unroll
    for (int c = 0; c < D; ++c) a[c] = 0.0;
    const double* xl = p.x + static_cast<long long>(l) * n * D;
    for (long long r = lane; r < n; r += 32)
#pragma unroll
      for (int c = 0; c < D; ++c) a[c] += xl[r * D + c];
#pragma unroll
    for (int c = 0; c < D; ++c) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a[c] += __shfl_xor_sync(0xffffffffu, a[c], o);
      if (lane == 0) sx[l * D + c] = a[c];
    }
  }
  consumers_sync();

  const double nn = static_cast<double>(n);
  const double mw = static_cast<double>(m) * p.w;
  const double direct = 1.0 / (nn + mw);
  const double spread = p.w / (nn * (nn + mw));
  long long gc = 0;  // chunks consumed
  int stg = 0;
  uint32_t ph = 0;
  for (int t = 0;; ++t) {
    for (int l = 0; l < m; ++l) {
      // ---- pass of modality l for y_t: register u holds point
      // q_u = slot + S (u ^ pi) (points past g or finished compute on a
      // clamped segment and are never read)
      double yv[Q][D], acc[Q][V];
      int seg[Q];  // a point's delta segment in a stage (doubles; 32-bit offsets)
#pragma unroll
      for (int u = 0; u < Q; ++u) {
        const int q = min(slot + S * (u ^ pi), g - 1);
        seg[u] = q * R;
#pragma unroll
        for (int c = 0; c < D; ++c) yv[u][c] = ybuf[((t & 1) * p.G + q) * m * D + l * D + c];
#pragma unroll
        for (int v = 0; v < V; ++v) acc[u][v] = 0.0;
      }
      const int xpar = static_cast<int>((static_cast<long long>(l) * n * D) & 1);
      for (int ch = 0; ch < nch; ++ch, ++gc) {
        const int rows = static_cast<int>(min(static_cast<long long>(R), n - static_cast<long long>(ch) * R));
        mbar_wait(&full[stg], ph);
        const double* base = ring + static_cast<long long>(stg) * p.stage_doubles;
        const double* xk0 = base + static_cast<long long>(p.G) * R + ((xpar + ch * R * D) & 1);
#ifdef JOFC_OOSP_DIAG  // timing experiment: streaming only (results wrong)
        if (rows > 0) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[stg]);
          if (++stg == kSt) {
            stg = 0;
            ph ^= 1u;
          }
          continue;
        }
#endif
#pragma unroll kOospUnroll
        for (int r = lane + 32 * wi; r < rows; r += 32 * WS) {
          double xk[D];
#pragma unroll
          for (int c = 0; c < D; ++c) xk[c] = xk0[r * D + c];
#pragma unroll
          for (int u = 0; u < Q; ++u) {
            const double dv = base[seg[u] + r];
            double s = 0.0;
#pragma unroll
            for (int c = 0; c < D; ++c) {
              const double df = xk[c] - yv[u][c];
              s = (c == 0) ? df * df : fma(df, df, s);
            }
            // dist == 0 guard (proj/src/oos.cpp:88) as an integer test of the
            // high word (s >= 0; s = 0 and the flushed denormals give 0)
            const double y = rsqrt_nr(s);
            const double inv = (__double2hiint(s) > 0) ? y : 0.0;
            const double rt = dv * inv;
            const double resid = fma(-s, inv, dv);
            acc[u][0] += rt;
            acc[u][1] = fma(resid, resid, acc[u][1]);
#pragma unroll
            for (int c = 0; c < D; ++c) acc[u][2 + c] = fma(rt, xk[c], acc[u][2 + c]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stg]);  // (release: this warp's reads of the stage)
        if (++stg == kSt) {
          stg = 0;
          ph ^= 1u;
        }
      }
      // ---- fold of modality l.  Reduce-scatter over the lane bits of pi:
      // at the level of point bit h, register u (bit h clear) adds the
      // partner's register u ^ h, which holds the same point.
#pragma unroll
      for (int h = Q / 2; h >= 1; h >>= 1) {
#pragma unroll
        for (int u = 0; u < h; ++u)
#pragma unroll
          for (int v = 0; v < V; ++v)
            acc[u][v] += __shfl_xor_sync(0xffffffffu, acc[u + h][v], h * kLanesPerPt);
      }
      // register 0 now holds point slot + S pi over the lanes sharing pi
#pragma unroll
      for (int o = kLanesPerPt / 2; o >= 1; o >>= 1)
#pragma unroll
        for (int v = 0; v < V; ++v) acc[0][v] += __shfl_xor_sync(0xffffffffu, acc[0][v], o);
      if ((lane & (kLanesPerPt - 1)) == 0)
#pragma unroll
        for (int v = 0; v < V; ++v) sred[(warp * Q + pi) * V + v] = acc[0][v];
      consumers_sync();
      for (int e = threadIdx.x; e < g * V; e += kT) {
        const int q = e / V, v = e - q * V;
        const int s = q % S, u = q / S;
        double a = 0.0;
        for (int w2 = 0; w2 < WS; ++w2) a += sred[((s + S * w2) * Q + u) * V + v];
        // xi = sum_k x_k - sum_k r_k x_k
        part[(l * p.G + q) * V + v] = (v >= 2) ? sx[l * D + v - 2] - a : a;
      }
      consumers_sync();
    }
    // ---- update step t of each point
    int active = 0;
    if (threadIdx.x < g && !pdone[threadIdx.x]) {
      const int q = threadIdx.x;
      const int pt = p_lo + q;
      const double* yc = ybuf + ((t & 1) * p.G + q) * m * D;
      double* yn = ybuf + (((t + 1) & 1) * p.G + q) * m * D;
      double fid = 0.0, com = 0.0, xi_sum[D], psi_y[D];
#pragma unroll
      for (int c = 0; c < D; ++c) xi_sum[c] = psi_y[c] = 0.0;
      for (int l = 0; l < m; ++l) {
        const double* pl = part + (l * p.G + q) * V;
        fid += pl[1];
#pragma unroll
        for (int c = 0; c < D; ++c) {
          xi_sum[c] += pl[2 + c];
          psi_y[c] = fma(pl[0], yc[l * D + c], psi_y[c]);
        }
        for (int l2 = l + 1; l2 < m; ++l2) {
#pragma unroll
          for (int c = 0; c < D; ++c) {
            const double df = yc[l * D + c] - yc[l2 * D + c];
            com = fma(df, df, com);
          }
        }
      }
      const double sigma = fid + p.w * com;
      bool finished = false;
      int status = 0;
      if (!isfinite(sigma)) {
        finished = true;
        status = 2;
      } else {
        if (t >= 1 && !p.fixed && (prev[q] - sigma) / p.term_count < p.eps) finished = true;
        if (t >= p.max_it) finished = true;
      }
      if (!finished)
        for (int l = 0; l < m; ++l) {
          const double* pl = part + (l * p.G + q) * V;
#pragma unroll
          for (int c = 0; c < D; ++c)
            yn[l * D + c] = direct * (pl[2 + c] + pl[0] * yc[l * D + c]) +
                            spread * (xi_sum[c] + psi_y[c]);
        }
      prev[q] = sigma;
      if (p.traces) p.traces[static_cast<long long>(pt) * (p.max_it + 1) + t] = sigma;
      if (finished) {
        double* yo = ((t & 1) ? p.yout1 : p.yout0) + static_cast<long long>(pt) * m * D;
        for (int e = 0; e < m * D; ++e) yo[e] = yc[e];
        OosPoint s;
        s.t = t;
        s.done = 1;
        s.iterations = t;
        s.status = status;
        p.st[pt] = s;
        pdone[q] = 1;
      }
      active = !finished;
    }
    if (!consumers_or(active)) break;
  }
  // tell the producer where the solve ended (it drains what it issued past it)
  if (threadIdx.x == 0) {
    *consumed = gc;
    __threadfence_block();
    *stop = 1;
  }
}

}  // namespace jofc_gpu
