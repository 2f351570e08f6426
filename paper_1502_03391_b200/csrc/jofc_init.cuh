// jofc_init.cuh -- GPU initialisation for fjofc_embed.
//
// averaged_procrustes_init (proj/src/init.cpp:57-88): cMDS of the modality
// average, cMDS of every modality, each Procrustes-rotated onto the average.
// cmds (proj/src/init.cpp:21-42) = top-d eigenpairs of the double-centred
// squared dissimilarities S = -1/2 J (Delta o Delta) J.
//
// Device side: S is materialised densely in HBM from the resident packed
// Delta (3.2 GB at n = 20000), its Frobenius norm reduced, and the subspace
// iteration's n x p products S Q run as a bandwidth-bound warp-per-row kernel.
// Host side (p x p and d x d work, O(n p^2)): the reference's shifted
// orthogonal iteration with Rayleigh-Ritz (proj/src/linalg.cpp:167-271) -- same
// start (Rng(0x9e3779b97f4a7c15) normals), same Gram-Schmidt with one
// re-orthogonalisation, same cyclic Jacobi on the Ritz matrix, same stopping
// residual 1e-9 ||S||_F -- and, for n <= 320, the reference's full cyclic
// Jacobi on the whole S; plus its one-sided Jacobi SVD for the d x d
// Procrustes rotation (proj/src/linalg.cpp:333-416).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <numeric>
#include <random>
#include <stdexcept>
#include <vector>

#include "jofc_layout.h"

namespace jofc_gpu {
namespace init {

// ------------------------------------------------------------------- kernels
// Dense D2 (n x n) from the packed blocks: for modality `which`, or the
// modality average when which < 0 (sum in modality order, then / m, as
// proj/src/init.cpp:62-67), squared (proj/src/init.cpp:26-28).  The diagonal
// is left to a prior memset.
__global__ void __launch_bounds__(256) dense_d2_kernel(const double* __restrict__ packed,
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

// Row sums of a dense n x n matrix: one warp per row.
__global__ void __launch_bounds__(256) row_sums_kernel(const double* __restrict__ a, long long n,
                                                       double* __restrict__ out) {
  const long long row = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  double s = 0.0;
  for (long long j = lane; j < n; j += 32) s += a[row * n + j];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[row] = s;
}

// In place: S_ij = -1/2 (D2_ij - rm_i - rm_j + tm) (proj/src/distance.cpp:31-53),
// accumulating sum S_ij^2 for ||S||_F.
__global__ void __launch_bounds__(256) double_center_kernel(double* __restrict__ a, long long n,
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

// Z (n x p) = S (n x n) Q (n x p), row-major; one warp per row of S.
template <int P>
__global__ void __launch_bounds__(256) matvec_kernel(const double* __restrict__ s, long long n,
                                                     const double* __restrict__ q,
                                                     double* __restrict__ z) {
  const long long row = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  double acc[P];
#pragma unroll
  for (int c = 0; c < P; ++c) acc[c] = 0.0;
  const double* sr = s + row * n;
  for (long long j = lane; j < n; j += 32) {
    const double v = __ldcs(sr + j);
#pragma unroll
    for (int c = 0; c < P; ++c) acc[c] = fma(v, __ldg(q + j * P + c), acc[c]);
  }
#pragma unroll
  for (int c = 0; c < P; ++c)
    for (int o = 16; o > 0; o >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < P; ++c) z[row * P + c] = acc[c];
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

// The reference Rng's normal stream (mt19937_64, 53-bit uniforms, Box-Muller
// with cached sine) -- proj/include/jofc/rng.hpp:17-55.
class Normals {
 public:
  explicit Normals(uint64_t seed) : e_(seed) {}
  double next() {
    if (have_) {
      have_ = false;
      return spare_;
    }
    double u1 = uni();
    while (u1 <= 0.0) u1 = uni();
    const double u2 = uni();
    const double rad = std::sqrt(-2.0 * std::log(u1));
    const double th = 2.0 * 3.14159265358979323846 * u2;
    spare_ = rad * std::sin(th);
    have_ = true;
    return rad * std::cos(th);
  }

 private:
  double uni() { return static_cast<double>(e_() >> 11) * 0x1.0p-53; }
  std::mt19937_64 e_;
  double spare_ = 0.0;
  bool have_ = false;
};

// Cyclic Jacobi eigen-decomposition (rotation by rotation as the reference's
// jacobi_decompose, sweep cap 100, off-diagonal tolerance 1e-12 ||A||_F).
inline bool jacobi_eigen(Mat a, std::vector<double>& values, Mat& v) {
  const std::size_t n = a.r;
  v = Mat(n, n);
  for (std::size_t i = 0; i < n; ++i) v(i, i) = 1.0;
  double fro = 0.0;
  for (double x : a.a) fro += x * x;
  const double tol = 1e-12 * std::sqrt(fro);
  auto off = [&]() {
    double s = 0.0;
    for (std::size_t i = 0; i < n; ++i)
      for (std::size_t j = i + 1; j < n; ++j) s += 2.0 * a(i, j) * a(i, j);
    return std::sqrt(s);
  };
  int sweep = 0;
  for (; sweep < 100; ++sweep) {
    if (off() <= tol) break;
    for (std::size_t p = 0; p + 1 < n; ++p)
      for (std::size_t q = p + 1; q < n; ++q) {
        const double apq = a(p, q);
        if (apq == 0.0) continue;
        const double tau = (a(q, q) - a(p, p)) / (2.0 * apq);
        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (std::abs(tau) + std::sqrt(1.0 + tau * tau));
        const double cs = 1.0 / std::sqrt(1.0 + t * t);
        const double sn = t * cs;
        const double app = a(p, p), aqq = a(q, q);
        a(p, p) = app - t * apq;
        a(q, q) = aqq + t * apq;
        a(p, q) = a(q, p) = 0.0;
        for (std::size_t r = 0; r < n; ++r) {
          if (r == p || r == q) continue;
          const double arp = a(r, p), arq = a(r, q);
          a(r, p) = a(p, r) = cs * arp - sn * arq;
          a(r, q) = a(q, r) = sn * arp + cs * arq;
        }
        for (std::size_t r = 0; r < n; ++r) {
          const double vrp = v(r, p), vrq = v(r, q);
          v(r, p) = cs * vrp - sn * vrq;
          v(r, q) = sn * vrp + cs * vrq;
        }
      }
  }
  if (sweep == 100 && off() > tol) return false;
  values.resize(n);
  for (std::size_t i = 0; i < n; ++i) values[i] = a(i, i);
  return true;
}

// Largest-magnitude component made positive (the reference's sign convention).
inline void fix_sign(std::vector<double>& vec) {
  std::size_t arg = 0;
  double best = 0.0;
  for (std::size_t i = 0; i < vec.size(); ++i)
    if (std::abs(vec[i]) > best) {
      best = std::abs(vec[i]);
      arg = i;
    }
  if (!vec.empty() && vec[arg] < 0.0)
    for (double& x : vec) x = -x;
}

// Gram-Schmidt of column j against columns < j, twice (re-orthogonalisation).
inline void project_out(Mat& q, std::size_t j) {
  for (int pass = 0; pass < 2; ++pass)
    for (std::size_t i = 0; i < j; ++i) {
      double dot = 0.0;
      for (std::size_t r = 0; r < q.r; ++r) dot += q(r, i) * q(r, j);
      for (std::size_t r = 0; r < q.r; ++r) q(r, j) -= dot * q(r, i);
    }
}

inline void orthonormalize(Mat& q) {
  for (std::size_t j = 0; j < q.c; ++j) {
    project_out(q, j);
    double nrm = 0.0;
    for (std::size_t r = 0; r < q.r; ++r) nrm += q(r, j) * q(r, j);
    nrm = std::sqrt(nrm);
    if (nrm < 1e-150) {  // vanished column: first coordinate vector outside the span
      for (std::size_t e = 0; e < q.r; ++e) {
        for (std::size_t r = 0; r < q.r; ++r) q(r, j) = (r == e) ? 1.0 : 0.0;
        project_out(q, j);
        double n2 = 0.0;
        for (std::size_t r = 0; r < q.r; ++r) n2 += q(r, j) * q(r, j);
        n2 = std::sqrt(n2);
        if (n2 > 1e-8) {
          nrm = n2;
          break;
        }
      }
    }
    for (std::size_t r = 0; r < q.r; ++r) q(r, j) /= nrm;
  }
}

// One-sided Jacobi SVD of a small square matrix -> (U, V) with the reference's
// ordering and deterministic completion of U (proj/src/linalg.cpp:333-416).
inline void svd_small(const Mat& a, Mat& u, Mat& vout) {
  const std::size_t n = a.r;
  Mat g = a, v(n, n);
  for (std::size_t i = 0; i < n; ++i) v(i, i) = 1.0;
  for (int sweep = 0; sweep < 64; ++sweep) {
    bool rotated = false;
    for (std::size_t p = 0; p + 1 < n; ++p)
      for (std::size_t q = p + 1; q < n; ++q) {
        double al = 0.0, be = 0.0, ga = 0.0;
        for (std::size_t r = 0; r < n; ++r) {
          al += g(r, p) * g(r, p);
          be += g(r, q) * g(r, q);
          ga += g(r, p) * g(r, q);
        }
        if (std::abs(ga) <= 1e-14 * std::sqrt(al * be) || ga == 0.0) continue;
        rotated = true;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / std::sqrt(1.0 + t * t);
        const double sn = cs * t;
        for (std::size_t r = 0; r < n; ++r) {
          const double gp = g(r, p), gq = g(r, q);
          g(r, p) = cs * gp - sn * gq;
          g(r, q) = sn * gp + cs * gq;
          const double vp = v(r, p), vq = v(r, q);
          v(r, p) = cs * vp - sn * vq;
          v(r, q) = sn * vp + cs * vq;
        }
      }
    if (!rotated) break;
  }
  std::vector<double> sig(n);
  for (std::size_t j = 0; j < n; ++j) {
    double nr = 0.0;
    for (std::size_t r = 0; r < n; ++r) nr += g(r, j) * g(r, j);
    sig[j] = std::sqrt(nr);
  }
  std::vector<std::size_t> order(n);
  std::iota(order.begin(), order.end(), std::size_t{0});
  std::stable_sort(order.begin(), order.end(),
                   [&](std::size_t x, std::size_t y) { return sig[x] > sig[y]; });
  u = Mat(n, n);
  vout = Mat(n, n);
  const double rank_tol = 1e-13 * std::max(1.0, n ? sig[order[0]] : 0.0);
  std::size_t filled = 0;
  for (std::size_t j = 0; j < n; ++j) {
    const std::size_t src = order[j];
    for (std::size_t r = 0; r < n; ++r) vout(r, j) = v(r, src);
    if (sig[src] > rank_tol) {
      for (std::size_t r = 0; r < n; ++r) u(r, j) = g(r, src) / sig[src];
      filled = j + 1;
    }
  }
  for (std::size_t j = filled; j < n; ++j)
    for (std::size_t e = 0; e < n; ++e) {
      std::vector<double> cand(n, 0.0);
      cand[e] = 1.0;
      for (std::size_t i = 0; i < j; ++i) {
        double dot = 0.0;
        for (std::size_t r = 0; r < n; ++r) dot += u(r, i) * cand[r];
        for (std::size_t r = 0; r < n; ++r) cand[r] -= dot * u(r, i);
      }
      double nr = 0.0;
      for (double x : cand) nr += x * x;
      nr = std::sqrt(nr);
      if (nr > 1e-6) {
        for (std::size_t r = 0; r < n; ++r) u(r, j) = cand[r] / nr;
        break;
      }
    }
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
