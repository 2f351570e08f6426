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
  for (int w = 0; w < 20; ++w) kern<<<blocks, 256>>>(buf, iters, 0.9999999, 1e-9);  // warm-up, clocks up
  cudaEventRecord(e0);
  for (int w = 0; w < 5; ++w) kern<<<blocks, 256>>>(buf, iters, 0.9999999, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 5.0f;
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

// ---------------------------------------------------------------- latencies
namespace {

__global__ void lat_kernel(double* out, long long* cycles, int iters, double seed) {
  double a = seed + threadIdx.x, b = 0.9999999, c = 1e-9;
  long long t0, t1;
  // DFMA dependent chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) a = fma(a, b, c);
  t1 = clock64();
  cycles[0] = t1 - t0;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) a = a + c;
  t1 = clock64();
  cycles[1] = t1 - t0;
  // MUFU.RSQ64H + DFMA chain (rsqrt approx feeding back)
  double y = a;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double r;
    asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y));
    y = r + 1.0;
  }
  t1 = clock64();
  cycles[2] = t1 - t0;
  // SHFL.64 chain
  double z = a;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) z = __shfl_xor_sync(0xffffffffu, z, 1) + 1.0;
  t1 = clock64();
  cycles[3] = t1 - t0;
  out[threadIdx.x] = a + y + z;
}

}  // namespace

extern "C" int jofc_probe_latency(int device, double* dfma, double* dadd, double* rsq_plus_dadd,
                                  double* shfl_plus_dadd) {
  if (cudaSetDevice(device) != cudaSuccess) return 3;
  double* out;
  long long* cyc;
  cudaMalloc(&out, 64 * sizeof(double));
  cudaMalloc(&cyc, 8 * sizeof(long long));
  const int iters = 4096;
  lat_kernel<<<1, 32>>>(out, cyc, iters, 1.5);
  lat_kernel<<<1, 32>>>(out, cyc, iters, 1.5);
  long long h[4];
  cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  *dfma = static_cast<double>(h[0]) / iters;
  *dadd = static_cast<double>(h[1]) / iters;
  *rsq_plus_dadd = static_cast<double>(h[2]) / iters;
  *shfl_plus_dadd = static_cast<double>(h[3]) / iters;
  cudaFree(out);
  cudaFree(cyc);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

// ---------------------------------------------------------- occupancy sweep
namespace {

template <int CH>
__global__ void dfma_chains(double* out, int iters, double b, double c) {
  double a[CH];
#pragma unroll
  for (int k = 0; k < CH; ++k) a[k] = 1e-3 * (threadIdx.x + k);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CH; ++k) a[k] = fma(a[k], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < CH; ++k) s += a[k];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int CH>
float run_chains(int blocks, int threads, int iters, double* buf) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 5; ++w) dfma_chains<CH><<<blocks, threads>>>(buf, iters, 0.9999999, 1e-9);
  cudaEventRecord(e0);
  for (int w = 0; w < 5; ++w) dfma_chains<CH><<<blocks, threads>>>(buf, iters, 0.9999999, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double flops = 2.0 * CH * iters * static_cast<double>(blocks) * threads * 5;
  return static_cast<float>(flops / (ms * 1e-3) / 1e12);
}

}  // namespace

// TF/s of pure DFMA chains for (warps per SM, independent chains per thread).
extern "C" int jofc_probe_occupancy(int device, int warps_per_sm, int chains, double* tflops) {
  if (cudaSetDevice(device) != cudaSuccess) return 3;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* buf;
  cudaMalloc(&buf, 1024 * sizeof(double));
  const int threads = warps_per_sm * 32;
  float t = 0.f;
  switch (chains) {
    case 1: t = run_chains<1>(sms, threads, 20000, buf); break;
    case 2: t = run_chains<2>(sms, threads, 10000, buf); break;
    case 4: t = run_chains<4>(sms, threads, 5000, buf); break;
    case 8: t = run_chains<8>(sms, threads, 2500, buf); break;
    default: t = run_chains<16>(sms, threads, 1250, buf); break;
  }
  *tflops = t;
  cudaFree(buf);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

// ------------------------------------------- synthetic pair math (no memory)
namespace {

// FL bit flags: 1 = no column accumulation, 2 = no fidelity, 4 = fp32 MUFU
// seed via integer exponent rebias, 8 = shared-product accumulation
// (t = rr*diff once, +t / -t), 16 = row accumulation only via R/Q form.
template <int D, int G, int FL>
__global__ void __launch_bounds__(256, 1) pair_math_kernel(double* out, int iters) {
  double xi[8][D], xj[4][D], racc[8][D], cacc[4][D];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int c = 0; c < D; ++c) {
      xi[a][c] = 1e-3 * (threadIdx.x + 7 * a + c);
      racc[a][c] = 0.0;
    }
#pragma unroll
  for (int b = 0; b < 4; ++b)
#pragma unroll
    for (int c = 0; c < D; ++c) {
      xj[b][c] = 2e-3 * (threadIdx.x + 3 * b - c);
      cacc[b][c] = 0.0;
    }
  double fid = 0.0, dl = 0.37;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int a = 0; a < 8; ++a) {
#pragma unroll
      for (int b0 = 0; b0 < 4; b0 += G) {
        double diff[G][D], s[G], y0[G], e[G], q[G], inv[G];
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
          for (int c = 0; c < D; ++c) {
            diff[g][c] = xi[a][c] - xj[b0 + g][c];
            s[g] = (c == 0) ? diff[g][c] * diff[g][c] : fma(diff[g][c], diff[g][c], s[g]);
          }
#pragma unroll
        for (int g = 0; g < G; ++g) {
          if (FL & 16) {
            // seed without MUFU: s -> float by exponent rebias, magic-constant
            // rsqrt + 2 FP32 Newton steps (~2^-17.7), float -> double rebias
            const int hi = __double2hiint(s[g]), lo = __double2loint(s[g]);
            const unsigned fb = (static_cast<unsigned>(hi - ((1023 - 127) << 20)) << 3) |
                                (static_cast<unsigned>(lo) >> 29);
            const float sf = __uint_as_float(fb);
            float yf = __uint_as_float(0x5f3759dfu - (fb >> 1));
            const float hs = 0.5f * sf;
            yf = yf * fmaf(-hs * yf, yf, 1.5f);
            yf = yf * fmaf(-hs * yf, yf, 1.5f);
            const unsigned rb = __float_as_uint(yf);
            y0[g] = __hiloint2double(static_cast<int>((rb >> 3) + ((1023 - 127) << 20)),
                                     static_cast<int>(rb << 29));
          } else if (FL & 4) {
            // fp32 seed: double -> float by exponent rebias (s in float range)
            const int hi = __double2hiint(s[g]), lo = __double2loint(s[g]);
            const unsigned fb = (static_cast<unsigned>(hi - ((1023 - 127) << 20)) << 3) |
                                (static_cast<unsigned>(lo) >> 29);
            float rf;
            asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(rf) : "f"(__uint_as_float(fb)));
            const unsigned rb = __float_as_uint(rf);
            y0[g] = __hiloint2double(static_cast<int>((rb >> 3) + ((1023 - 127) << 20)),
                                     static_cast<int>(rb << 29));
          } else {
            asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0[g]) : "d"(s[g]));
          }
        }
#pragma unroll
        for (int g = 0; g < G; ++g) e[g] = fma(-(s[g] * y0[g]), y0[g], 1.0);
#pragma unroll
        for (int g = 0; g < G; ++g) q[g] = e[g] * y0[g];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const double y = fma(fma(e[g], 0.375, 0.5), q[g], y0[g]);
          inv[g] = (__double2hiint(s[g]) >= 0x00100000) ? y : 0.0;
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const double rr = dl * inv[g];
          if (!(FL & 2)) {
            const double res = dl - s[g] * inv[g];
            fid = fma(res, res, fid);
          }
#pragma unroll
          for (int c = 0; c < D; ++c) {
            if (FL & 8) {
              const double t = rr * diff[g][c];
              racc[a][c] += t;
              if (!(FL & 1)) cacc[b0 + g][c] -= t;
            } else {
              racc[a][c] = fma(rr, diff[g][c], racc[a][c]);
              if (!(FL & 1)) cacc[b0 + g][c] = fma(-rr, diff[g][c], cacc[b0 + g][c]);
            }
          }
        }
      }
      xi[a][0] += 1e-12;  // defeat hoisting of the distance math out of `it`
    }
    dl += 1e-9;
  }
  double t = fid;
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int c = 0; c < D; ++c) t += racc[a][c] + xi[a][c];
#pragma unroll
  for (int b = 0; b < 4; ++b)
#pragma unroll
    for (int c = 0; c < D; ++c) t += cacc[b][c];
  if (t == 12345.678) out[threadIdx.x] = t;
}

template <int D, int G, int FL>
void run_pair(int sms, int iters, double* buf, cudaEvent_t e0, cudaEvent_t e1, int* regs) {
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, pair_math_kernel<D, G, FL>);
  *regs = fa.numRegs;
  for (int w = 0; w < 3; ++w) pair_math_kernel<D, G, FL><<<sms, 256>>>(buf, iters);
  cudaEventRecord(e0);
  for (int w = 0; w < 5; ++w) pair_math_kernel<D, G, FL><<<sms, 256>>>(buf, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
}

}  // namespace

// pairs/s per GPU of the pass kernel's per-pair math alone (8 warps/SM).
extern "C" int jofc_probe_pair_math(int device, int d, int group, int flags,
                                    double* gpairs_per_s, int* regs) {
  if (cudaSetDevice(device) != cudaSuccess) return 3;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* buf;
  cudaMalloc(&buf, 1024 * sizeof(double));
  const int iters = 400;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
#define JOFC_PM(DD, GG, FF) \
  if (d == DD && group == GG && flags == FF) run_pair<DD, GG, FF>(sms, iters, buf, e0, e1, regs);
#define JOFC_PM_ALL(FF) JOFC_PM(5, 4, FF) JOFC_PM(5, 1, FF) JOFC_PM(3, 4, FF) JOFC_PM(3, 1, FF)
  JOFC_PM_ALL(0) JOFC_PM_ALL(1) JOFC_PM_ALL(2) JOFC_PM_ALL(3) JOFC_PM_ALL(4) JOFC_PM_ALL(8)
  JOFC_PM_ALL(12) JOFC_PM_ALL(16)
#undef JOFC_PM_ALL
#undef JOFC_PM
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  *gpairs_per_s = 5.0 * iters * 32.0 * sms * 256.0 / (ms * 1e-3) / 1e9;
  cudaFree(buf);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

// ------------------------------------------------ per-instruction throughput
namespace {

template <int OP>
__global__ void __launch_bounds__(256) op_tput_kernel(double* out, int iters) {
  double v[8], w1[8], w2[8];
  float f[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    w1[k] = 0.999 + 1e-4 * (threadIdx.x ^ k);
    w2[k] = 1e-9 * (k + 1) + 1e-12 * threadIdx.x;
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    v[k] = 1.0 + 1e-3 * (threadIdx.x + k);
    f[k] = 1.0f + 1e-3f * (threadIdx.x + k);
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) {  // MUFU.RSQ64H
        double r;
        asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(v[k]));
        v[k] = r;
      } else if (OP == 1) {  // MUFU.RSQ (fp32)
        float r;
        asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f[k]));
        f[k] = r;
      } else if (OP == 2) {
        v[k] = v[k] + 1e-9;
      } else if (OP == 3) {
        v[k] = v[k] * 0.9999999;
      } else if (OP == 4) {  // DFMA, three distinct register operands (independent chains)
        v[k] = fma(w1[k], w2[k], v[k]);
      } else if (OP == 5) {  // DFMA, one register operand + two reused
        v[k] = fma(v[k], 0.9999999, 1e-9);
      } else if (OP == 6) {  // DFMA, shared multiplier (reuse), fresh addend (acc pattern)
        v[k] = fma(w1[0], w2[k], v[k]);
      } else if (OP == 7) {  // DADD, two fresh registers
        v[k] = v[k] + w2[k];
      } else if (OP == 8) {  // 1 RSQ64H per 7 DFMA (pair-loop proportion), independent
        if (k == 0) {
          double r;
          asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(w1[0]));
          w1[0] = r + 1e-300;
        } else {
          v[k] = fma(v[k], 0.9999999, 1e-9);
        }
      } else if (OP == 10) {  // F2F.F32.F64
        f[k] = __double2float_rn(v[k]) + f[k];
        v[k] = v[k] * 1.0000001;
      } else if (OP == 11) {  // 7 DFMA + 1 (F2F.F32.F64, MUFU.RSQ f32, F2F.F64.F32)
        if (k == 0) {
          float t;
          asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(__double2float_rn(w1[0])));
          w1[0] = static_cast<double>(t) + 1e-300;
        } else {
          v[k] = fma(v[k], 0.9999999, 1e-9);
        }
      } else if (OP == 9) {  // 8 DFMA + one 2-FSEL select per 8
        v[k] = fma(v[k], 0.9999999, 1e-9);
        if (k == 7) v[0] = (__double2hiint(v[7]) > 5) ? v[0] : 0.0;
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += v[k] + f[k] + w1[k] + w2[k];
  if (s == 12345.678) out[threadIdx.x] = s;
}

}  // namespace

// Warp-instructions per clock per SM for op: 0 RSQ64H, 1 RSQ f32, 2 DADD, 3 DMUL.
extern "C" int jofc_probe_op(int device, int op, double* per_clk_per_sm) {
  if (cudaSetDevice(device) != cudaSuccess) return 3;
  int sms = 0, khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, device);
  double* buf;
  cudaMalloc(&buf, 1024 * sizeof(double));
  const int iters = 2000, blocks = sms * 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](auto kern) {
    for (int w = 0; w < 3; ++w) kern<<<blocks, 256>>>(buf, iters);
    cudaEventRecord(e0);
    for (int w = 0; w < 3; ++w) kern<<<blocks, 256>>>(buf, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  };
  switch (op) {
    case 0: run(op_tput_kernel<0>); break;
    case 1: run(op_tput_kernel<1>); break;
    case 2: run(op_tput_kernel<2>); break;
    case 3: run(op_tput_kernel<3>); break;
    case 4: run(op_tput_kernel<4>); break;
    case 5: run(op_tput_kernel<5>); break;
    case 6: run(op_tput_kernel<6>); break;
    case 7: run(op_tput_kernel<7>); break;
    case 8: run(op_tput_kernel<8>); break;
    case 9: run(op_tput_kernel<9>); break;
    case 10: run(op_tput_kernel<10>); break;
    default: run(op_tput_kernel<11>); break;
  }
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warp_instrs = 3.0 * iters * 8.0 * blocks * 8.0;
  const double clocks = ms * 1e-3 * khz * 1e3;
  *per_clk_per_sm = warp_instrs / clocks / sms;
  cudaFree(buf);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

// ------------------------------------------------- MUFU.RSQ64H seed accuracy
namespace {
__global__ void rsq_err_kernel(unsigned long long seed, int per_thread, double* out) {
  unsigned long long x = seed ^ (0x9E3779B97F4A7C15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1));
  double worst = 0.0;
  for (int i = 0; i < per_thread; ++i) {
    x ^= x >> 12;
    x ^= x << 25;
    x ^= x >> 27;
    const unsigned long long m = (x * 0x2545F4914F6CDD1Dull) >> 12;  // 52 random mantissa bits
    const int ex = 1023 + static_cast<int>((x >> 5) % 80) - 40;      // s in ~[2^-40, 2^40)
    const double s = __longlong_as_double((static_cast<long long>(ex) << 52) | m);
    double y0;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(s));
    const double e = fabs(fma(-(s * y0), y0, 1.0));
    worst = fmax(worst, e);
  }
  for (int o = 16; o > 0; o >>= 1) worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
  if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<unsigned long long*>(out),
                                         static_cast<unsigned long long>(__double_as_longlong(worst)));
}
}  // namespace

// max |1 - s y0^2| of the MUFU.RSQ64H seed over random s (~2^26 samples)
extern "C" int jofc_probe_rsq_error(int device, double* max_e) {
  if (cudaSetDevice(device) != cudaSuccess) return 3;
  double* d;
  cudaMalloc(&d, sizeof(double));
  cudaMemset(d, 0, sizeof(double));
  rsq_err_kernel<<<1024, 256>>>(12345ull, 256, d);
  cudaMemcpy(max_e, d, sizeof(double), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

// ------------------------------------------------- L2-resident read bandwidth
// The out-of-sample pass re-reads its k x m x n delta rows (80 MB at C5)
// every update: an L2-resident working set, not an HBM stream.  This is the
// roof it is judged against: a buffer of `bytes` read once to warm L2, then
// read `reps` times by a grid-stride kernel of 16-byte loads, summed so the
// loads cannot be elided.
namespace {
__global__ void __launch_bounds__(256) l2_read_kernel(const double2* __restrict__ buf, size_t n2,
                                                      double* out) {
  double acc = 0.0;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n2;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const double2 v = __ldcg(buf + i);
    acc += v.x + v.y;
  }
  if (acc == 12345.678) out[0] = acc;
}
}  // namespace

extern "C" int jofc_probe_l2_read(int device, size_t bytes, double* gbs) {
  if (cudaSetDevice(device) != cudaSuccess) return 3;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double2* buf = nullptr;
  double* out = nullptr;
  if (cudaMalloc(&buf, bytes) != cudaSuccess || cudaMalloc(&out, sizeof(double)) != cudaSuccess)
    return 3;
  cudaMemset(buf, 0, bytes);
  const size_t n2 = bytes / sizeof(double2);
  const int grid = sms * 8;
  for (int w = 0; w < 5; ++w) l2_read_kernel<<<grid, 256>>>(buf, n2, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 50;
  cudaEventRecord(e0);
  for (int w = 0; w < reps; ++w) l2_read_kernel<<<grid, 256>>>(buf, n2, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  *gbs = static_cast<double>(bytes) * reps / (ms * 1e-3) / 1e9;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}
