// Drop-in for proj/include/jofc/weights.hpp (hot-path subset): the weight
// families and the m x m system W whose inverse mixes the per-modality
// products in the fast Guttman transform.
#pragma once

#include <cstddef>
#include <vector>

#include "jofc/dense_matrix.hpp"

namespace jofc {

//   uniform(w):      a_i = 1,      w_ij = w
//   general(W):      a_i = W_ii,   w_ij = W_ij
//   product(a, c):   a_i = c a_i,  w_ij = a_i a_j
class WeightSpec {
public:
  enum class Kind { uniform, general_symmetric, product };

  static WeightSpec uniform(double w);
  static WeightSpec general(DenseMatrix w);
  static WeightSpec product(std::vector<double> within, double fidelity_scale = 1.0);

  Kind kind() const { return kind_; }
  double within_weight(std::size_t i) const;
  double cross_weight(std::size_t i, std::size_t j) const;
  void validate(std::size_t m) const;

  double uniform_w() const { return uniform_w_; }
  double fidelity_scale() const { return scale_; }
  const DenseMatrix& general_matrix() const { return general_; }
  const std::vector<double>& product_within() const { return product_; }

private:
  WeightSpec() = default;
  Kind kind_ = Kind::uniform;
  double uniform_w_ = 1.0;
  double scale_ = 1.0;
  DenseMatrix general_;
  std::vector<double> product_;
};

DenseMatrix script_w(const WeightSpec& spec, std::size_t m, std::size_t n);
DenseMatrix script_w_inverse(const WeightSpec& spec, std::size_t m, std::size_t n);

struct ScriptW {
  DenseMatrix w;
  DenseMatrix w_inverse;
  static ScriptW make(const WeightSpec& spec, std::size_t m, std::size_t n);
};

}  // namespace jofc
