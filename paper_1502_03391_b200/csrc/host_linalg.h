// host_linalg.h -- the small dense host algebra of libjofc_gpu.so, shared by
// the initialisers (capi_init.cu: the Jacobi route of cmds, the p x p
// Rayleigh-Ritz step of the subspace iteration, Procrustes), the weights
// (jofc_weights.cpp: the general W^-1) and the drop-in API
// (dropin/linalg.cpp).  One implementation of each routine.
//
// All matrices are dense row-major arrays of doubles.  The routines follow
// the reference's CONTRACTS (proj/include/jofc/linalg.hpp): the same
// stopping rules, sweep caps, orderings and sign / completion conventions,
// so that results agree with the reference to rounding; the numerical
// kernels are the textbook ones (cyclic Jacobi with Rutishauser's
// tau-form updates, Hestenes' one-sided Jacobi SVD, classical Gram-Schmidt
// with one re-orthogonalisation pass, partial-pivot Gauss-Jordan).
#pragma once

#include <cstddef>
#include <vector>

namespace jofc_gpu {
namespace hostla {

// Symmetric eigen-decomposition by cyclic Jacobi rotations of the n x n
// matrix a (only read).  Pivots (p, q) sweep row by row; a sweep starts only
// while off(A) = sqrt(sum_{i != j} a_ij^2) exceeds rel_tol * ||a||_F.  On
// return w holds the eigenvalues in diagonal order and the COLUMNS of v the
// eigenvectors.  False when max_sweeps sweeps did not reach the tolerance
// (proj/src/linalg.cpp's cap: 100 sweeps, 1e-12).
bool jacobi_eigh(const double* a, std::size_t n, double* w, double* v, int max_sweeps = 100,
                 double rel_tol = 1e-12);

// Indices of w[0..n) by descending value; equal values keep their order.
std::vector<std::size_t> descending_order(const double* w, std::size_t n);

// Sign convention of the reference's eigenvectors: flip x (n entries,
// stride apart) so that its first largest-magnitude entry is positive.
void orient(double* x, std::size_t n, std::size_t stride = 1);

// Square n x n SVD a = u diag(s) v^T by one-sided Jacobi on the columns
// (at most 64 sweeps; a pair is skipped once |g_p . g_q| <= 1e-14 |g_p||g_q|).
// s descending (stable); columns of u for singular values <= 1e-13
// max(1, s_max) are completed with the coordinate vectors e_0, e_1, ...
// orthogonalised against the columns before them (the reference's
// deterministic completion for rank-deficient inputs).
void svd_jacobi(const double* a, std::size_t n, double* u, double* s, double* v);

// Orthonormalise the columns of q (rows x cols), left to right: classical
// Gram-Schmidt against the earlier columns, applied twice; a column that
// vanishes (norm < 1e-150) is replaced by the first coordinate vector that
// keeps norm > 1e-8 after the same projection.
void orthonormalize_columns(double* q, std::size_t rows, std::size_t cols);

// Inverse of the n x n matrix a by Gauss-Jordan elimination with partial
// (row) pivoting.  False when a pivot falls below pivot_rel * max(1, max|a|)
// (proj/src/linalg.cpp: 1e-13, "singular matrix").
bool gauss_jordan_inverse(const double* a, std::size_t n, double* inv, double pivot_rel = 1e-13);

}  // namespace hostla
}  // namespace jofc_gpu
