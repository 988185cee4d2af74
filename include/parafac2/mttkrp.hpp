// Drop-in replacement for /root/reference/proj/include/parafac2/mttkrp.hpp:
// the slice-wise MTTKRP on packed projected slices runs on the GPU
// (p2g_mttkrp_packed); shape checks and exception types as mttkrp.hpp:170-181.
#pragma once

#include "kernels.hpp"
#include "slices.hpp"

namespace parafac2 {

namespace detail {
inline Matrix mttkrp_device(const ProjectedSlices& Y, const Matrix& H, const Matrix& V, const Matrix& W, int mode) {
  std::vector<std::int64_t> ptr;
  std::vector<std::int32_t> cols;
  std::vector<double> data;
  Y.to_c(ptr, cols, data);
  const Index rows = mode == 1 ? Y.rank() : (mode == 2 ? Y.n_cols() : Y.n_slices());
  Matrix out(rows, Y.rank());
  check(p2g_mttkrp_packed(Device::get().ctx(), mode, Y.n_slices(), Y.n_cols(), static_cast<int32_t>(Y.rank()),
                          ptr.data(), cols.data(), data.data(), H.data(), V.data(), W.data(), out.data()));
  return out;
}
/// mttkrp.hpp:170-181
inline void check_mttkrp_input(const ProjectedSlices& Y, const Matrix& H, const Matrix& V, const Matrix& W, int mode) {
  if (mode < 1 || mode > 3) throw std::invalid_argument("mttkrp: mode must be 1, 2 or 3");
  const Index R = Y.rank();
  if (H.rows() != R || H.cols() != R) throw std::invalid_argument("mttkrp: H must be R x R");
  if (V.rows() != Y.n_cols() || V.cols() != R) throw std::invalid_argument("mttkrp: V must be J x R");
  if (W.rows() != Y.n_slices() || W.cols() != R) throw std::invalid_argument("mttkrp: W must be K x R");
}
}  // namespace detail

/// mttkrp.hpp:187-196 (`threads` ignored on the GPU path).
inline Matrix mttkrp(const ProjectedSlices& Y, const Matrix& H, const Matrix& V, const Matrix& W, int mode,
                     int /*threads*/ = 1) {
  detail::check_mttkrp_input(Y, H, V, W, mode);
  return detail::mttkrp_device(Y, H, V, W, mode);
}

/// mttkrp.hpp:81-106
inline Matrix mttkrp_mode1(const ProjectedSlices& Y, const Matrix& V, const Matrix& W, int /*threads*/ = 1) {
  if (V.rows() != Y.n_cols() || W.rows() != Y.n_slices() || W.cols() != V.cols())
    throw std::invalid_argument("mttkrp: factor V has mismatched dimensions");
  return detail::mttkrp_device(Y, Matrix::Identity(Y.rank(), Y.rank()), V, W, 1);
}
/// mttkrp.hpp:111-138
inline Matrix mttkrp_mode2(const ProjectedSlices& Y, const Matrix& H, const Matrix& W, int /*threads*/ = 1) {
  if (H.rows() != Y.rank() || W.rows() != Y.n_slices() || W.cols() != H.cols())
    throw std::invalid_argument("mttkrp: factor H has mismatched dimensions");
  return detail::mttkrp_device(Y, H, Matrix(Y.n_cols(), Y.rank()), W, 2);
}
/// mttkrp.hpp:143-166
inline Matrix mttkrp_mode3(const ProjectedSlices& Y, const Matrix& H, const Matrix& V, int /*threads*/ = 1) {
  if (H.rows() != Y.rank() || V.rows() != Y.n_cols() || V.cols() != H.cols())
    throw std::invalid_argument("mttkrp: factor V has mismatched dimensions");
  return detail::mttkrp_device(Y, H, V, Matrix(Y.n_slices(), Y.rank()), 3);
}

/// mttkrp.hpp:241-253
inline std::uint64_t naive_mttkrp_bytes(Index K, Index J, Index R, int mode) {
  const auto k = static_cast<std::uint64_t>(K), j = static_cast<std::uint64_t>(J), r = static_cast<std::uint64_t>(R);
  switch (mode) {
    case 1: return 8 * (r * j * k + k * j * r + r * r);
    case 2: return 8 * (j * r * k + k * r * r + j * r);
    case 3: return 8 * (k * r * j + j * r * r + k * r);
    default: throw std::invalid_argument("mttkrp: mode must be 1, 2 or 3");
  }
}

}  // namespace parafac2
