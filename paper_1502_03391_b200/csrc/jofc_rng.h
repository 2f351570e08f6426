// jofc_rng.h -- the reference's random stream (proj/include/jofc/rng.hpp:17-55)
// for the host side of libjofc_gpu.so: the synthetic workloads
// (workloads.cpp) and the subspace iteration's start panel (capi_init.cu).
// std::mt19937_64 (its output sequence is fixed by the C++ standard), 53-bit
// uniforms on [0, 1), and Box-Muller normals that return the cosine variate
// first and keep the sine one for the next call -- the arithmetic the
// reference specifies, so a caller holding the reference regenerates the
// same bits.
#pragma once

#include <cmath>
#include <cstdint>
#include <random>

namespace jofc_gpu {

class RefRng {
 public:
  explicit RefRng(std::uint64_t seed) : engine_(seed) {}

  double uniform() { return static_cast<double>(engine_() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }

  double normal() {
    if (cached_) {
      cached_ = false;
      return spare_;
    }
    double u1;
    do u1 = uniform(); while (u1 <= 0.0);
    const double u2 = uniform();
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 2.0 * 3.14159265358979323846 * u2;
    spare_ = radius * std::sin(angle);
    cached_ = true;
    return radius * std::cos(angle);
  }

 private:
  std::mt19937_64 engine_;
  double spare_ = 0.0;
  bool cached_ = false;
};

}  // namespace jofc_gpu
