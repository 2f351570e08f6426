// probe.cu -- FP64 throughput microbenchmarks (libjofc_probe.so).
//
// MEASURED_PEAKS.json carries HBM and bf16 peaks only; the fJOFC roofline
// also needs the FP64 ceiling, so bench.py measures it
// here on the same box: DFMA on the FP64 pipe, DMMA (mma.sync m8n8k4 f64) on
// the tensor pipe, and both interleaved (do they overlap?).
#include <cuda_runtime.h>

#include <cstdint>

namespace {

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) dfma_kernel(double* out, int iters, double b, double c) {
  double a[kChains];
#pragma unroll
  for (int k = 0; k < kChains; ++k) a[k] = 1e-3 * (threadIdx.x + k);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < kChains; ++k) a[k] = fma(a[k], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += a[k];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256) dmma_kernel(double* out, int iters, double b, double c) {
  double d[kChains][2];
  const double a = 1e-3 * threadIdx.x;
#pragma unroll
  for (int k = 0; k < kChains; ++k) d[k][0] = d[k][1] = c * k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < kChains; ++k) dmma(d[k][0], d[k][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += d[k][0] + d[k][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) mixed_kernel(double* out, int iters, double b, double c) {
  double a[kChains], d[4][2];
  const double av = 1e-3 * threadIdx.x;
#pragma unroll
  for (int k = 0; k < kChains; ++k) a[k] = 1e-3 * (threadIdx.x + k);
#pragma unroll
  for (int k = 0; k < 4; ++k) d[k][0] = d[k][1] = c * k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < kChains; ++k) a[k] = fma(a[k], b, c);
#pragma unroll
    for (int k = 0; k < 4; ++k) dmma(d[k][0], d[k][1], av, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += a[k];
#pragma unroll
  for (int k = 0; k < 4; ++k) s += d[k][0] + d[k][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <class K>
float time_kernel(K kern, int blocks, int iters, double* buf) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<blocks, 256>>>(buf, iters, 0.9999999, 1e-9);  // warm-up
  cudaEventRecord(e0);
  kern<<<blocks, 256>>>(buf, iters, 0.9999999, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return ms;
}

}  // namespace

extern "C" int jofc_probe_fp64(int device, double* dfma_tflops, double* dmma_tflops,
                               double* mixed_tflops) {
  if (cudaSetDevice(device) != cudaSuccess) return 3;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int blocks = sms * 8;
  const int iters = 4096;
  double* buf = nullptr;
  if (cudaMalloc(&buf, 256 * sizeof(double)) != cudaSuccess) return 3;
  const double threads = static_cast<double>(blocks) * 256.0;
  float ms = time_kernel(dfma_kernel, blocks, iters, buf);
  *dfma_tflops = 2.0 * kChains * iters * threads / (ms * 1e-3) / 1e12;
  ms = time_kernel(dmma_kernel, blocks, iters / 4, buf);
  // per warp per mma: 8x8x4 FMA = 256 FMA = 512 flop
  *dmma_tflops = 512.0 * kChains * (iters / 4) * (threads / 32.0) / (ms * 1e-3) / 1e12;
  ms = time_kernel(mixed_kernel, blocks, iters / 4, buf);
  *mixed_tflops = (2.0 * kChains * (iters / 4) * threads +
                   512.0 * 4 * (iters / 4) * (threads / 32.0)) /
                  (ms * 1e-3) / 1e12;
  cudaFree(buf);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}
