// pairs_probe.cu -- EXPERIMENT (not shipped): how fast can the pass kernel's
// per-pair arithmetic run on one SM as a function of the thread's tile
// (A rows x C columns), the warps per SM and where the row accumulators live?
// Shared-memory Delta / X reads as in the real kernel, no HBM traffic, no
// column reduction.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
//   -shared -Xcompiler -fPIC -o build/libpairs_probe.so scripts/exp/pairs_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

namespace {

__device__ __forceinline__ double rsqrt_nr(double s) {
  double y0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(s));
  const double h = s * y0;
  const double e = fma(-h, y0, 1.0);
  const double p = fma(e, 0.375, 0.5);
  const double q = e * y0;
  return fma(p, q, y0);
}

// RACC: 0 registers, 1 shared memory (per-thread slots, loaded/stored per row)
template <int D, int A, int C, int THREADS, int RACC>
__global__ void __launch_bounds__(THREADS, 1) pairs_kernel(double* out, int blocks) {
  extern __shared__ double sm[];
  double* sd = sm;                      // 128 x 64 "delta" (column-major)
  double* sx = sd + 128 * 64;           // 192 x D x rows of X (block: 128 rows x <= 64 columns)
  double* sr = sx + 192 * (D | 1);      // racc slots [a][cc][thread]
  for (int e = threadIdx.x; e < 128 * 64; e += THREADS) sd[e] = 1.0 + 1e-3 * (e % 97);
  for (int e = threadIdx.x; e < 192 * (D | 1); e += THREADS) sx[e] = 1e-2 * ((e * 37) % 101);
  if (RACC == 1)
    for (int e = threadIdx.x; e < A * D * THREADS; e += THREADS) sr[e] = 0.0;
  __syncthreads();
  constexpr int kW = THREADS / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // tile of this thread: rows r0 + RS*a, columns c0 + CS*b
  constexpr int kRowLanes = 128 / A;       // threads along rows
  const int t = threadIdx.x;
  const int rt = t % kRowLanes, ct = t / kRowLanes;  // ct * C < 64
  double racc[RACC == 0 ? A : 1][D];
  if (RACC == 0)
#pragma unroll
    for (int a = 0; a < A; ++a)
#pragma unroll
      for (int c = 0; c < D; ++c) racc[a][c] = 0.0;
  double fid[C];
#pragma unroll
  for (int b = 0; b < C; ++b) fid[b] = 0.0;
  double tot = 0.0;
  for (int blk = 0; blk < blocks; ++blk) {
    asm volatile("" ::: "memory");  // the real kernel's mbarrier wait
    double xj[C][D], cacc[C][D];
#pragma unroll
    for (int b = 0; b < C; ++b)
#pragma unroll
      for (int c = 0; c < D; ++c) xj[b][c] = sx[(128 + ct * C + b) * (D | 1) + c] + 1e-9 * blk;
#pragma unroll
    for (int a = 0; a < A; ++a) {
      const int il = rt + kRowLanes * a;
      double xi[D], ra[D];
#pragma unroll
      for (int c = 0; c < D; ++c) xi[c] = sx[il * (D | 1) + c];
      if (RACC == 1) {
#pragma unroll
        for (int c = 0; c < D; ++c) ra[c] = sr[(a * D + c) * THREADS + t];
      } else {
#pragma unroll
        for (int c = 0; c < D; ++c) ra[c] = racc[a][c];
      }
#pragma unroll
      for (int b = 0; b < C; ++b) {
        const double dl = sd[(ct * C + b) * 128 + il];
        double diff[D], s;
#pragma unroll
        for (int c = 0; c < D; ++c) diff[c] = xi[c] - xj[b][c];
#pragma unroll
        for (int c = 0; c < D; ++c) s = c == 0 ? fma(diff[c], diff[c], 0x1p-1022) : fma(diff[c], diff[c], s);
        const double y = rsqrt_nr(s);
        const double rr = dl * y;
        const double res = dl - s * y;
        fid[b] = fma(res, res, fid[b]);
#pragma unroll
        for (int c = 0; c < D; ++c) {
          ra[c] = fma(rr, diff[c], ra[c]);
          cacc[b][c] = a == 0 ? -rr * diff[c] : fma(-rr, diff[c], cacc[b][c]);
        }
      }
      if (RACC == 1) {
#pragma unroll
        for (int c = 0; c < D; ++c) sr[(a * D + c) * THREADS + t] = ra[c];
      } else {
#pragma unroll
        for (int c = 0; c < D; ++c) racc[a][c] = ra[c];
      }
    }
#pragma unroll
    for (int b = 0; b < C; ++b)
#pragma unroll
      for (int c = 0; c < D; ++c) tot += cacc[b][c];
  }
#pragma unroll
  for (int b = 0; b < C; ++b) tot += fid[b];
  if (RACC == 0)
#pragma unroll
    for (int a = 0; a < A; ++a)
#pragma unroll
      for (int c = 0; c < D; ++c) tot += racc[a][c];
  else
    for (int e = 0; e < A * D; ++e) tot += sr[e * THREADS + t];
  (void)lane;
  (void)warp;
  (void)kW;
  if (tot == 12345.678) out[threadIdx.x] = tot;
}

template <int D, int A, int C, int THREADS, int RACC>
double run(int sms, double* buf, int* regs, int* spill) {
  auto k = pairs_kernel<D, A, C, THREADS, RACC>;
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, k);
  *regs = fa.numRegs;
  *spill = static_cast<int>(fa.localSizeBytes);
  const int smem = (128 * 64 + 192 * (D | 1) + (RACC ? A * D * THREADS : 0)) * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int blocks = 200;
  for (int w = 0; w < 3; ++w) k<<<sms, THREADS, smem>>>(buf, blocks);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int w = 0; w < 5; ++w) k<<<sms, THREADS, smem>>>(buf, blocks);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  if (cudaGetLastError() != cudaSuccess) return -1.0;
  // pairs per launch: sms x THREADS x blocks x A x C
  const double pairs = 5.0 * sms * THREADS * double(blocks) * A * C;
  return pairs / (ms * 1e-3) / 1e9;  // Gpairs/s
}

}  // namespace

extern "C" int pairs_probe(int device) {
  cudaSetDevice(device);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* buf;
  cudaMalloc(&buf, 4096 * sizeof(double));
  int regs, spill;
#define RUN(D, A, C, T, R)                                                                    \
  {                                                                                           \
    double g = run<D, A, C, T, R>(sms, buf, &regs, &spill);                                   \
    printf("D=%d A=%d C=%d threads=%d racc=%s: %7.1f Gpairs/s  C3-equiv %.3f ms  regs %d spill %d\n", \
           D, A, C, T, R ? "smem" : "regs", g, 4.0e8 / (g * 1e9) * 1e3, regs, spill);         \
    fflush(stdout);                                                                           \
  }
  RUN(5, 8, 4, 256, 0)
  RUN(5, 8, 2, 384, 0)
  RUN(5, 8, 2, 256, 0)
  RUN(5, 4, 4, 384, 0)
  RUN(5, 4, 2, 512, 0)
  RUN(5, 8, 1, 512, 0)
  RUN(5, 4, 4, 256, 0)
  RUN(3, 8, 4, 256, 0)
  RUN(3, 8, 2, 384, 0)
  RUN(3, 4, 4, 512, 0)
  RUN(3, 8, 2, 512, 0)
#undef RUN
  cudaFree(buf);
  return 0;
}
