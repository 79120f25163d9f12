// llsa C++ operator API — B200 build.  Drop-in replacement for the reference
// library's public headers (P/include/llsa/*.hpp): same names, argument
// meaning and typed errors; the work runs on the GPU through include/llsa_cuda.h.
//
// Element type: the GPU path computes in fp32, so `real` is float (the
// reference's LLSA_SINGLE_PRECISION configuration, P/include/llsa/types.hpp:12-16).
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>
#include <vector>

namespace llsa {

using real = float;

// Row-major rows × cols matrix of `real`, one row per token.  Same contract
// as the reference (P/include/llsa/types.hpp:22-59): default/zero-filled
// construction, and a validating factory for external data.
class FeatureMatrix {
 public:
  FeatureMatrix() = default;
  FeatureMatrix(std::size_t rows, std::size_t cols);

  // ShapeMismatch when values.size() != rows*cols, NonFiniteError on NaN/inf.
  static FeatureMatrix from_values(std::size_t rows, std::size_t cols,
                                   std::vector<real> values);

  std::size_t rows() const noexcept { return n_rows_; }
  std::size_t cols() const noexcept { return n_cols_; }
  std::size_t size() const noexcept { return data_.size(); }
  bool empty() const noexcept { return data_.empty(); }
  bool same_shape(const FeatureMatrix& o) const noexcept {
    return n_rows_ == o.n_rows_ && n_cols_ == o.n_cols_;
  }

  real* data() noexcept { return data_.data(); }
  const real* data() const noexcept { return data_.data(); }
  std::span<const real> values() const noexcept { return data_; }

  real* row(std::size_t r) noexcept { return data_.data() + r * n_cols_; }
  const real* row(std::size_t r) const noexcept { return data_.data() + r * n_cols_; }
  real& at(std::size_t r, std::size_t c) noexcept { return data_[r * n_cols_ + c]; }
  real at(std::size_t r, std::size_t c) const noexcept { return data_[r * n_cols_ + c]; }

  bool all_finite() const noexcept;

 private:
  std::size_t n_rows_ = 0;
  std::size_t n_cols_ = 0;
  std::vector<real> data_;
};

// max_i |a_i - b_i|; ShapeMismatch if the shapes differ.
real max_abs_diff(const FeatureMatrix& a, const FeatureMatrix& b);

}  // namespace llsa
