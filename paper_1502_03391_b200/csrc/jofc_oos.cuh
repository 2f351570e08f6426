// jofc_oos.cuh -- batched out-of-sample Guttman updates (sm_100a).
//
// k new objects, each with m views, embedded against a frozen in-sample
// configuration X (m x n x d).  Per point and modality j the reference
// (proj/src/oos.cpp:83-96) needs, for the current y_j,
//   r_k = [dist != 0] delta_j(k) / dist(X^(j)_k, y_j),
//   psi_j = sum_k r_k,   xi_j = sum_k (1 - r_k) X^(j)_k,
// and oos_stress (proj/src/oos.cpp:50-57) needs sum_k (delta_j(k) - dist)^2
// from the same distances, so one streaming pass over delta yields both
// (fused like the in-sample pass).  jofc_oos_update_kernel then applies the
// closed-form corner update (proj/src/oos.cpp:98-111), the commensurability
// term and the per-point stop rule (proj/src/oos.cpp:221-226).
//
// Pass layout: CTA = 8 warps = 8 points of one modality (blockIdx.y) and one
// of kOosSplits slices of the in-sample range (blockIdx.z); X^(j) streams
// through two shared-memory chunk buffers (512 rows each, filled by the TMA
// bulk engine, double buffered) shared by the 8 warps; lanes stride the n
// in-sample rows (coalesced delta reads, 4 in flight per lane), warp shuffles
// finish the sums.
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
};

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

}  // namespace jofc_gpu
