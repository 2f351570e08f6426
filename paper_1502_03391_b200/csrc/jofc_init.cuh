// jofc_init.cuh -- GPU initialisation for fjofc_embed.
//
// averaged_procrustes_init (proj/src/init.cpp:57-88): cMDS of the modality
// average, cMDS of every modality, each Procrustes-rotated onto the average.
// cmds (proj/src/init.cpp:21-42) = top-d eigenpairs of the double-centred
// squared dissimilarities S = -1/2 J (Delta o Delta) J.
//
// Device side: S is materialised densely in HBM from the resident packed
// Delta (3.2 GB at n = 20000), its Frobenius norm reduced, and the reference's
// shifted orthogonal iteration with Rayleigh-Ritz (proj/src/linalg.cpp:167-271)
// runs with its n x p panels resident: S Q as a bandwidth-bound tiled kernel,
// the Ritz/Gram products and the re-orthogonalisation as O(n p^2) kernels.
// Same start (Rng(0x9e3779b97f4a7c15) normals, Gram-Schmidt on the host), same
// cyclic Jacobi on the p x p Ritz matrix (host, host_linalg.h), same
// stopping residual 1e-9 ||S||_F.  The reference re-orthogonalises with Gram-Schmidt plus one
// re-orthogonalisation; here it is Cholesky-QR twice (same Q in exact
// arithmetic, rounding-level difference), falling back to host Gram-Schmidt
// when the panel is too ill-conditioned for Cholesky.  For n <= 320 the
// reference's route -- cyclic Jacobi on the whole S -- runs on the host; the
// d x d Procrustes rotation comes from a one-sided Jacobi SVD (the shared
// host_linalg.h routines, proj/src/linalg.cpp's contracts).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <numeric>
#include <random>
#include <stdexcept>
#include <vector>

#include "host_linalg.h"
#include "jofc_layout.h"
#include "jofc_rng.h"

namespace jofc_gpu {
namespace init {

// ------------------------------------------------------------------- kernels
// Dense D2 (n x n) from the packed blocks: for modality `which`, or the
// modality average when which < 0 (sum in modality order, then / m, as
// proj/src/init.cpp:62-67), squared (proj/src/init.cpp:26-28).  The diagonal
// is left to a prior memset.
static __global__ void __launch_bounds__(256) dense_d2_kernel(const double* __restrict__ packed,
                                                       long long n, int nT, long long bpm, int m,
                                                       int which, double* __restrict__ d2) {
  const long long g0 = blockIdx.x;  // block index within one modality
  int l0, B, J;
  block_coords(g0, nT, bpm, l0, B, J);
  const long long gi0 = static_cast<long long>(kRows) * B, gj0 = static_cast<long long>(kCols) * J;
  for (int e = threadIdx.x; e < kBlockElems; e += blockDim.x) {
    const int jl = e >> 7, il = e & 127;
    const long long i = gi0 + il, j = gj0 + jl;
    if (!(i < j && j < n)) continue;
    double v;
    if (which >= 0) {
      v = packed[(static_cast<long long>(which) * bpm + g0) * kBlockElems + e];
    } else {
      double s = 0.0;
      for (int l = 0; l < m; ++l) s += packed[(static_cast<long long>(l) * bpm + g0) * kBlockElems + e];
      v = s / static_cast<double>(m);
    }
    const double sq = v * v;
    d2[j * n + i] = sq;  // coalesced along i
    d2[i * n + j] = sq;
  }
}

// Dense squared omnibus dissimilarity (N = m n) of imputed_omnibus_init
// (proj/src/init.cpp:90-116): block (bi, bj) holds Delta_bi for bi == bj and
// 0.5 (Delta_bi + Delta_bj) otherwise (same rounding as the host), each entry
// then squared as cmds does.  One CTA per packed block of modality 0's stream
// coordinates; every unordered modality pair writes its four mirror entries.
static __global__ void __launch_bounds__(256) omnibus_d2_kernel(const double* __restrict__ packed,
                                                         long long n, int nT, long long bpm, int m,
                                                         double* __restrict__ d2) {
  const long long g0 = blockIdx.x;
  int l0, B, J;
  block_coords(g0, nT, bpm, l0, B, J);
  const long long N = static_cast<long long>(m) * n;
  const long long gi0 = static_cast<long long>(kRows) * B, gj0 = static_cast<long long>(kCols) * J;
  for (int e = threadIdx.x; e < kBlockElems; e += blockDim.x) {
    const int jl = e >> 7, il = e & 127;
    const long long i = gi0 + il, j = gj0 + jl;
    if (!(i < j && j < n)) continue;
    for (int bi = 0; bi < m; ++bi) {
      const double a = packed[(static_cast<long long>(bi) * bpm + g0) * kBlockElems + e];
      for (int bj = bi; bj < m; ++bj) {
        double v = a;
        if (bj != bi)
          v = __dmul_rn(0.5, __dadd_rn(a, packed[(static_cast<long long>(bj) * bpm + g0) * kBlockElems + e]));
        const double sq = __dmul_rn(v, v);
        const long long ri = bi * n, rj = static_cast<long long>(bj) * n;
        d2[(rj + j) * N + ri + i] = sq;
        d2[(ri + i) * N + rj + j] = sq;
        if (bj != bi) {
          d2[(rj + i) * N + ri + j] = sq;
          d2[(ri + j) * N + rj + i] = sq;
        }
      }
    }
  }
}

// Row sums of a dense n x n matrix: one warp per row.
static __global__ void __launch_bounds__(256) row_sums_kernel(const double* __restrict__ a, long long n,
                                                       double* __restrict__ out) {
  const long long row = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  double s = 0.0;
  for (long long j = lane; j < n; j += 32) s += a[row * n + j];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[row] = s;
}

// Row sums of squares of a dense n x n matrix (||S||_F by the host, in row
// order): one warp per row.
static __global__ void __launch_bounds__(256) row_sumsq_kernel(const double* __restrict__ a, long long n,
                                                        double* __restrict__ out) {
  const long long row = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  double s = 0.0;
  for (long long j = lane; j < n; j += 32) s = fma(a[row * n + j], a[row * n + j], s);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[row] = s;
}

// In place: S_ij = -1/2 (D2_ij - rm_i - rm_j + tm) (proj/src/distance.cpp:31-53),
// accumulating sum S_ij^2 for ||S||_F.
static __global__ void __launch_bounds__(256) double_center_kernel(double* __restrict__ a, long long n,
                                                            const double* __restrict__ rm,
                                                            double tm, double* __restrict__ fro2) {
  const long long total = n * n;
  double acc = 0.0;
  for (long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = e / n, j = e - i * n;
    const double v = -0.5 * (a[e] - rm[i] - rm[j] + tm);
    a[e] = v;
    acc = fma(v, v, acc);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int w = 0; w < (blockDim.x >> 5); ++w) v += red[w];
    atomicAdd(fro2, v);
  }
}

// out[e] = sum over b of part[b * per + e], b ascending (the order the host
// summed the per-CTA partials in).
static __global__ void __launch_bounds__(256) sum_partials_kernel(const double* __restrict__ part,
                                                               int blocks, int per,
                                                               double* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= per) return;
  double s = 0.0;
  int b = 0;
  for (; b + 16 <= blocks; b += 16) {  // 16 loads in flight, then the in-order adds
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = __ldcg(part + static_cast<long long>(b + u) * per + e);
#pragma unroll
    for (int u = 0; u < 16; ++u) s += v[u];
  }
  for (; b < blocks; ++b) s += __ldcg(part + static_cast<long long>(b) * per + e);
  out[e] = s;
}

// ------------------------------------------------- device subspace iteration
// The n x p panels (Q, Z = S Q, W = Z + shift Q) stay in HBM; only p x p
// Gram/Ritz matrices and per-CTA partial sums cross to the host each sweep.
constexpr int kMvRows = 512;    // rows of Z per CTA (two per thread: r and r + 256)
constexpr int kMvChunk = 128;   // columns of S per staged Q chunk
constexpr int kMvMaxSplits = 32;  // column ranges per row block (deterministic partials)
constexpr int kMaxP = 14;       // widest panel: d <= 10, p = d + 4

// Partial Z_s = S[:, J_s] Q[J_s, :] for column range J_s = blockIdx.y.  S is
// symmetric, so thread t reads S[j][r] for its rows r = base + t, base + 256 + t
// -- consecutive threads, consecutive addresses -- streamed once with
// evict-first.  The Q rows of the range are staged in shared memory at an even
// stride and read as warp-uniform 16-byte broadcasts, each feeding both rows.
// The partials zp[s] (n x p each) are summed in split order by
// gram_shift_kernel.
template <int P>
__global__ void __launch_bounds__(256) matvec_sym_kernel(const double* __restrict__ s,
                                                         long long n,
                                                         const double* __restrict__ q,
                                                         double* __restrict__ zp) {
  constexpr int PP = (P + 1) & ~1;
  __shared__ __align__(16) double qs[kMvChunk * PP];
  const long long r0 = static_cast<long long>(blockIdx.x) * kMvRows + threadIdx.x;
  const long long r1 = r0 + 256;
  const long long span = (n + gridDim.y - 1) / gridDim.y;
  const long long j0 = span * blockIdx.y, j1 = (j0 + span < n) ? j0 + span : n;
  const bool live0 = r0 < n, live1 = r1 < n;
  const double* col0 = s + (live0 ? r0 : 0);
  const double* col1 = s + (live1 ? r1 : 0);
  double acc0[PP], acc1[PP];
#pragma unroll
  for (int c = 0; c < PP; ++c) acc0[c] = acc1[c] = 0.0;
  for (long long c0 = j0; c0 < j1; c0 += kMvChunk) {
    const int cnt = static_cast<int>(j1 - c0 < kMvChunk ? j1 - c0 : kMvChunk);
    __syncthreads();
    for (int e = threadIdx.x; e < cnt * PP; e += blockDim.x) {
      const int jj = e / PP, c = e - jj * PP;
      qs[e] = (c < P) ? q[(c0 + jj) * P + c] : 0.0;
    }
    __syncthreads();
    int jj = 0;
    for (; jj < cnt; jj += 16) {
      const int u_end = (cnt - jj < 16) ? cnt - jj : 16;
      double sv0[16], sv1[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const long long off = (c0 + jj + u) * n;
        sv0[u] = (live0 && u < u_end) ? __ldcs(col0 + off) : 0.0;
        sv1[u] = (live1 && u < u_end) ? __ldcs(col1 + off) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        if (u >= u_end) break;
        const double2* qv = reinterpret_cast<const double2*>(qs + (jj + u) * PP);
#pragma unroll
        for (int c2 = 0; c2 < PP / 2; ++c2) {
          const double2 v = qv[c2];
          acc0[2 * c2] = fma(sv0[u], v.x, acc0[2 * c2]);
          acc0[2 * c2 + 1] = fma(sv0[u], v.y, acc0[2 * c2 + 1]);
          acc1[2 * c2] = fma(sv1[u], v.x, acc1[2 * c2]);
          acc1[2 * c2 + 1] = fma(sv1[u], v.y, acc1[2 * c2 + 1]);
        }
      }
    }
  }
  double* out = zp + static_cast<long long>(blockIdx.y) * n * P;
  if (live0)
#pragma unroll
    for (int c = 0; c < P; ++c) out[r0 * P + c] = acc0[c];
  if (live1)
#pragma unroll
    for (int c = 0; c < P; ++c) out[r1 * P + c] = acc1[c];
}

// Accumulates two p x p Gram products over 64-row chunks staged in shared
// memory: thread e < 2 p^2 owns one entry.  a/b/c/d are chunk pointers.
template <int P>
__device__ __forceinline__ void gram_pair_accumulate(const double* sa, const double* sb,
                                                     const double* sc, const double* sd, int rows,
                                                     double (&acc)[2]) {
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int e = threadIdx.x + s * blockDim.x;
    if (e >= 2 * P * P) continue;
    const int which = e / (P * P), ij = e - which * P * P, i = ij / P, j = ij - i * P;
    const double* x = which ? sc : sa;
    const double* y = which ? sd : sb;
    double v = acc[s];
    for (int r = 0; r < rows; ++r) v = fma(x[r * P + i], y[r * P + j], v);
    acc[s] = v;
  }
}

// Rayleigh-Ritz + shift pass: Z = sum of the `splits` partials (written out),
// T = Q^T Z and, with W = Z + shift Q (written out), G = W^T W.
// part[blk] = {T (p x p), G (p x p)}.
template <int P>
__global__ void __launch_bounds__(256) gram_shift_kernel(const double* __restrict__ q,
                                                         const double* __restrict__ zp,
                                                         double* __restrict__ z,
                                                         double* __restrict__ w, long long n,
                                                         int splits, double shift,
                                                         double* __restrict__ part) {
  __shared__ double sq[64 * P], sz[64 * P], sw[64 * P];
  double acc[2] = {0.0, 0.0};
  const long long chunks = (n + 63) / 64;
  for (long long ch = blockIdx.x; ch < chunks; ch += gridDim.x) {
    const long long r0 = ch * 64;
    const int rows = static_cast<int>(n - r0 < 64 ? n - r0 : 64);
    __syncthreads();
    for (int e = threadIdx.x; e < rows * P; e += blockDim.x) {
      const double qv = q[r0 * P + e];
      double zv = zp[r0 * P + e];
      for (int sp = 1; sp < splits; ++sp) zv += zp[static_cast<long long>(sp) * n * P + r0 * P + e];
      z[r0 * P + e] = zv;
      const double wv = zv + shift * qv;  // the reference's z += shift * q
      sq[e] = qv;
      sz[e] = zv;
      sw[e] = wv;
      w[r0 * P + e] = wv;
    }
    __syncthreads();
    gram_pair_accumulate<P>(sq, sz, sw, sw, rows, acc);
  }
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int e = threadIdx.x + s * blockDim.x;
    if (e < 2 * P * P) part[static_cast<long long>(blockIdx.x) * 2 * P * P + e] = acc[s];
  }
}

struct RitzParams {
  double u[kMaxP * kMaxP];     // p x k: the top-k Ritz coefficient columns
  double theta[kMaxP];         // their Ritz values
  double rinv[kMaxP * kMaxP];  // p x p upper-triangular R^{-1} of W = Q1 R
};

// Per row: Ritz vectors Q u_c (written to ritz, n x k), residual partials
// sum_r ((Z u_c)_r - theta_c (Q u_c)_r)^2, and the re-orthogonalised panel
// Q1 = W R^{-1} (written over Q) with the Gram partial Q1^T Q1 for the second
// Cholesky-QR sweep.  part[blk] = {res (k), G2 (p x p)}.
template <int P>
__global__ void __launch_bounds__(256) ritz_orth_kernel(double* __restrict__ q,
                                                        const double* __restrict__ z,
                                                        const double* __restrict__ w, long long n,
                                                        int k, const RitzParams prm,
                                                        double* __restrict__ ritz,
                                                        double* __restrict__ part) {
  __shared__ double s1[256 * P];
  __shared__ double red[8 * P];
  double res[P];
#pragma unroll
  for (int c = 0; c < P; ++c) res[c] = 0.0;
  double acc[2] = {0.0, 0.0};
  const long long tiles = (n + 255) / 256;
  for (long long tl = blockIdx.x; tl < tiles; tl += gridDim.x) {
    const long long row = tl * 256 + threadIdx.x;
    const int rows = static_cast<int>(n - tl * 256 < 256 ? n - tl * 256 : 256);
    __syncthreads();
    if (row < n) {
      double qr[P], zr[P], wr[P];
#pragma unroll
      for (int j = 0; j < P; ++j) {
        qr[j] = q[row * P + j];
        zr[j] = z[row * P + j];
        wr[j] = w[row * P + j];
      }
#pragma unroll
      for (int c = 0; c < P; ++c) {
        if (c < k) {
          double rv = 0.0, zv = 0.0;
#pragma unroll
          for (int j = 0; j < P; ++j) {
            rv = fma(qr[j], prm.u[j * kMaxP + c], rv);
            zv = fma(zr[j], prm.u[j * kMaxP + c], zv);
          }
          ritz[row * k + c] = rv;
          const double df = zv - prm.theta[c] * rv;
          res[c] = fma(df, df, res[c]);
        }
      }
#pragma unroll
      for (int j = 0; j < P; ++j) {
        double v = 0.0;
#pragma unroll
        for (int i = 0; i <= j; ++i) v = fma(wr[i], prm.rinv[i * kMaxP + j], v);
        s1[threadIdx.x * P + j] = v;
        q[row * P + j] = v;
      }
    }
    __syncthreads();
    gram_pair_accumulate<P>(s1, s1, s1, s1, rows, acc);
  }
  // residual partials: warp reduce, then across warps in fixed order
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int c = 0; c < P; ++c) {
    double v = res[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp * P + c] = v;
  }
  __syncthreads();
  double* out = part + static_cast<long long>(blockIdx.x) * (P + P * P);
  if (threadIdx.x < P) {
    double v = 0.0;
    for (int wi = 0; wi < static_cast<int>(blockDim.x >> 5); ++wi) v += red[wi * P + threadIdx.x];
    out[threadIdx.x] = v;
  }
  // only the first p^2 entries (sa = sb = s1) are meaningful
  if (threadIdx.x < P * P) out[P + threadIdx.x] = acc[0];
}

// Q = Q1 R2^{-1} in place (second Cholesky-QR sweep).
template <int P>
__global__ void __launch_bounds__(256) apply_rinv_kernel(double* __restrict__ q, long long n,
                                                         const RitzParams prm) {
  const long long row = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (row >= n) return;
  double qr[P];
#pragma unroll
  for (int j = 0; j < P; ++j) qr[j] = q[row * P + j];
#pragma unroll
  for (int j = 0; j < P; ++j) {
    double v = 0.0;
#pragma unroll
    for (int i = 0; i <= j; ++i) v = fma(qr[i], prm.rinv[i * kMaxP + j], v);
    q[row * P + j] = v;
  }
}

// ------------------------------------------------------------- host algebra
// Row-major n x p helpers.
struct Mat {
  std::size_t r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(std::size_t rows, std::size_t cols) : r(rows), c(cols), a(rows * cols, 0.0) {}
  double& operator()(std::size_t i, std::size_t j) { return a[i * c + j]; }
  double operator()(std::size_t i, std::size_t j) const { return a[i * c + j]; }
};

// The start panel's normal stream: the reference's Rng (jofc_rng.h).
class Normals {
 public:
  explicit Normals(uint64_t seed) : rng_(seed) {}
  double next() { return rng_.normal(); }

 private:
  RefRng rng_;
};

// Host algebra on Mat: the shared routines of host_linalg.h.
inline bool jacobi_eigen(const Mat& a, std::vector<double>& values, Mat& v) {
  values.resize(a.r);
  v = Mat(a.r, a.r);
  return hostla::jacobi_eigh(a.a.data(), a.r, values.data(), v.a.data());
}

inline void fix_sign(std::vector<double>& vec) { hostla::orient(vec.data(), vec.size()); }

inline void orthonormalize(Mat& q) { hostla::orthonormalize_columns(q.a.data(), q.r, q.c); }

inline void svd_small(const Mat& a, Mat& u, Mat& v) {
  u = Mat(a.r, a.r);
  v = Mat(a.r, a.r);
  std::vector<double> sig(a.r);
  hostla::svd_jacobi(a.a.data(), a.r, u.a.data(), sig.data(), v.a.data());
}

inline void center_columns(Mat& x) {
  if (x.r == 0) return;
  std::vector<double> mean(x.c, 0.0);
  for (std::size_t i = 0; i < x.r; ++i)
    for (std::size_t j = 0; j < x.c; ++j) mean[j] += x(i, j);
  for (double& v : mean) v /= static_cast<double>(x.r);
  for (std::size_t i = 0; i < x.r; ++i)
    for (std::size_t j = 0; j < x.c; ++j) x(i, j) -= mean[j];
}

// Upper-triangular Cholesky factor of a symmetric positive definite p x p
// matrix (G = R^T R) and its inverse.  False when a pivot collapses below
// 1e-12 of its diagonal (the panel is too ill-conditioned for Cholesky-QR;
// the caller falls back to Gram-Schmidt).
inline bool cholesky_rinv(const Mat& g, Mat& rinv) {
  const std::size_t p = g.r;
  Mat r(p, p);
  for (std::size_t j = 0; j < p; ++j) {
    double d = g(j, j);
    for (std::size_t k = 0; k < j; ++k) d -= r(k, j) * r(k, j);
    if (!(d > 1e-12 * g(j, j)) || !(g(j, j) > 0.0)) return false;
    r(j, j) = std::sqrt(d);
    for (std::size_t i = j + 1; i < p; ++i) {
      double v = g(j, i);
      for (std::size_t k = 0; k < j; ++k) v -= r(k, j) * r(k, i);
      r(j, i) = v / r(j, j);
    }
  }
  rinv = Mat(p, p);
  for (std::size_t j = 0; j < p; ++j) {  // solve R X = I column by column (back substitution)
    for (std::size_t ii = j + 1; ii-- > 0;) {
      double v = (ii == j) ? 1.0 : 0.0;
      for (std::size_t k = ii + 1; k <= j; ++k) v -= r(ii, k) * rinv(k, j);
      rinv(ii, j) = v / r(ii, ii);
    }
  }
  return true;
}

inline Mat procrustes(const Mat& source, const Mat& target) {
  Mat s = source, t = target;
  center_columns(s);
  center_columns(t);
  const std::size_t d = s.c;
  Mat cross(d, d);
  for (std::size_t i = 0; i < d; ++i)
    for (std::size_t k = 0; k < s.r; ++k) {
      const double v = s(k, i);  // (s^T t)(i, j) accumulated row by row of s^T
      for (std::size_t j = 0; j < d; ++j) cross(i, j) += v * t(k, j);
    }
  Mat u, v;
  svd_small(cross, u, v);
  Mat rot(d, d);
  for (std::size_t i = 0; i < d; ++i)
    for (std::size_t k = 0; k < d; ++k) {
      const double uv = u(i, k);
      for (std::size_t j = 0; j < d; ++j) rot(i, j) += uv * v(j, k);
    }
  Mat out(s.r, d);
  for (std::size_t i = 0; i < s.r; ++i)
    for (std::size_t k = 0; k < d; ++k) {
      const double sv = s(i, k);
      for (std::size_t j = 0; j < d; ++j) out(i, j) += sv * rot(k, j);
    }
  return out;
}

}  // namespace init
}  // namespace jofc_gpu
