// Accuracy of rsqrt.approx.ftz.f64 (MUFU.RSQ64H) and of the Newton steps built
// on it, over s in [2^-40, 2^40): max and mean relative error vs 1/sqrt(s)
// computed in long double on the host.  nvcc -arch=sm_100a rsq_probe.cu
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

__global__ void k(const double* s, double* y0, double* y2, double* y3, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = s[i], y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y0[i] = y;
  double h = x * y, e = fma(-h, y, 1.0);
  y2[i] = fma(e * y, 0.5, y);
  y3[i] = fma(fma(e, 0.375, 0.5), e * y, y);
}

int main() {
  const int n = 1 << 22;
  std::vector<double> s(n), a(n), b(n), c(n);
  std::mt19937_64 g(1);
  std::uniform_real_distribution<double> u(-40.0, 40.0);
  for (auto& v : s) v = std::exp2(u(g));
  double *ds, *d0, *d2, *d3;
  cudaMalloc(&ds, n * 8); cudaMalloc(&d0, n * 8); cudaMalloc(&d2, n * 8); cudaMalloc(&d3, n * 8);
  cudaMemcpy(ds, s.data(), n * 8, cudaMemcpyHostToDevice);
  k<<<n / 256, 256>>>(ds, d0, d2, d3, n);
  cudaMemcpy(a.data(), d0, n * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.data(), d2, n * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(c.data(), d3, n * 8, cudaMemcpyDeviceToHost);
  double mx[3] = {0, 0, 0}, mean[3] = {0, 0, 0};
  for (int i = 0; i < n; ++i) {
    long double t = 1.0L / std::sqrt((long double)s[i]);
    double r[3] = {(double)((a[i] - t) / t), (double)((b[i] - t) / t), (double)((c[i] - t) / t)};
    for (int j = 0; j < 3; ++j) { mx[j] = std::fmax(mx[j], std::fabs(r[j])); mean[j] += r[j] / n; }
  }
  std::printf("seed   max rel %.3e (2^%.1f) mean %.3e\n", mx[0], std::log2(mx[0]), mean[0]);
  std::printf("2nd    max rel %.3e (2^%.1f) mean %.3e\n", mx[1], std::log2(mx[1]), mean[1]);
  std::printf("3rd    max rel %.3e (2^%.1f) mean %.3e\n", mx[2], std::log2(mx[2]), mean[2]);
  return 0;
}
