// jofc_weights.h -- host-side constants of the Guttman loop (product code).
//
// Restates, for the C ABI, the reference's weight algebra
// (proj/src/weights.cpp:21-135): within weights a_l, cross weights w_ll',
// the m x m system matrix W (diag n a_i + sum_j w_ij, off-diag -w_ij), its
// inverse (closed forms for uniform / product, partial-pivot Gauss-Jordan for
// general, as proj/src/linalg.cpp:296-331) and ScriptW::make's check
// ||W W^-1 - I|| <= 1e-12 max(1, max|W|).  Errors carry the reference's
// messages.
#pragma once

#include <cstddef>
#include <string>
#include <vector>

#include "jofc_gpu.h"

namespace jofc_gpu {

struct HostWeights {
  std::vector<double> within;  // a_l
  std::vector<double> cross;   // m*m, w_ll' (0 on the diagonal)
  std::vector<double> winv;    // m*m
  std::vector<double> coef;    // m*m, winv(j,l) * a_l  (mix coefficients)
};

// Returns JOFC_OK / JOFC_EINVAL / JOFC_ENUMERIC and fills *msg on failure.
int build_weights(const jofc_weights* spec, std::size_t m, std::size_t n, HostWeights* out,
                  std::string* msg);

// Validation only (WeightSpec factories + validate(m)).
int validate_weights(const jofc_weights* spec, std::size_t m, std::string* msg);

}  // namespace jofc_gpu
