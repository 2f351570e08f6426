// Test-only C entry points over csrc/host_linalg.cpp (tests/test_host_linalg.py
// compiles this file together with it; nothing here ships).
#include <cstddef>

#include "host_linalg.h"

namespace la = jofc_gpu::hostla;

extern "C" {
int t_jacobi(const double* a, size_t n, double* w, double* v) { return la::jacobi_eigh(a, n, w, v); }
void t_svd(const double* a, size_t n, double* u, double* s, double* v) { la::svd_jacobi(a, n, u, s, v); }
void t_orth(double* q, size_t r, size_t c) { la::orthonormalize_columns(q, r, c); }
int t_inv(const double* a, size_t n, double* inv) { return la::gauss_jordan_inverse(a, n, inv); }
void t_orient(double* x, size_t n) { la::orient(x, n); }
}
