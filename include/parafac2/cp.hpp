// Drop-in replacement for /root/reference/proj/include/parafac2/cp.hpp:
// cp_als_iteration runs on the GPU (p2g_cp_als_iteration); cp_objective uses
// the device mode-3 MTTKRP and Gram.
#pragma once

#include "mttkrp.hpp"

namespace parafac2 {

struct CpFactors {
  Matrix H, V, W;
  Vector lambda;
};

struct CpOptions {
  bool nonneg = true;
  bool normalize_w = false;
  int threads = 1;
};

namespace detail {
inline void check_cp_shapes(const ProjectedSlices& Y, const CpFactors& f) {
  const Index R = Y.rank();
  if (f.H.rows() != R || f.H.cols() != R) throw std::invalid_argument("cp factors: H must be R x R");
  if (f.V.rows() != Y.n_cols() || f.V.cols() != R) throw std::invalid_argument("cp factors: V must be J x R");
  if (f.W.rows() != Y.n_slices() || f.W.cols() != R) throw std::invalid_argument("cp factors: W must be K x R");
}
}  // namespace detail

/// cp.hpp:78-90
inline double cp_objective(const ProjectedSlices& Y, const CpFactors& f, int threads = 1) {
  detail::check_cp_shapes(Y, f);
  if (static_cast<Index>(f.lambda.size()) != Y.rank()) throw std::invalid_argument("cp factors: lambda must have length R");
  Matrix sw = f.W;
  for (Index r = 0; r < sw.cols(); ++r)
    for (Index k = 0; k < sw.rows(); ++k) sw(k, r) *= f.lambda[static_cast<std::size_t>(r)];
  const Matrix m3 = mttkrp_mode3(Y, f.H, f.V, threads);
  const Matrix C = hadamard(gram(f.H), gram(f.V));
  double cross = 0.0, model = 0.0;
  for (Index i = 0; i < sw.size(); ++i) cross += sw.data()[i] * m3.data()[i];
  const Matrix swC = sw * C;
  for (Index i = 0; i < sw.size(); ++i) model += swC.data()[i] * sw.data()[i];
  return Y.frobenius_sq() - 2.0 * cross + model;
}

/// cp.hpp:99-145
inline CpFactors cp_als_iteration(const ProjectedSlices& Y, CpFactors f, const CpOptions& opts = {},
                                  Matrix* mode3_out = nullptr) {
  detail::check_cp_shapes(Y, f);
  std::vector<std::int64_t> ptr;
  std::vector<std::int32_t> cols;
  std::vector<double> data;
  Y.to_c(ptr, cols, data);
  const Index R = Y.rank();
  f.lambda.assign(static_cast<std::size_t>(R), 1.0);
  Matrix m3(Y.n_slices(), R);
  check(p2g_cp_als_iteration(Device::get().ctx(), Y.n_slices(), Y.n_cols(), static_cast<int32_t>(R), ptr.data(),
                             cols.data(), data.data(), f.H.data(), f.V.data(), f.W.data(), opts.nonneg ? 1 : 0,
                             opts.normalize_w ? 1 : 0, f.lambda.data(), m3.data()));
  if (mode3_out) *mode3_out = m3;
  return f;
}

}  // namespace parafac2
