// Drop-in replacement for /root/reference/proj/include/parafac2/kernels.hpp:
// gram, pinv_small and nnls_rowwise run on the GPU through the C ABI;
// khatri_rao and hadamard (not on the hot path) stay on the host.
#pragma once

#include <algorithm>

#include "common.hpp"

namespace parafac2 {

/// kernels.hpp:34-44 (host; the naive-MTTKRP oracle only).
inline Matrix khatri_rao(const Matrix& A, const Matrix& B) {
  if (A.cols() != B.cols()) throw std::invalid_argument("khatri_rao: operands differ in column count");
  ensure_finite(A, "khatri_rao left operand");
  ensure_finite(B, "khatri_rao right operand");
  Matrix out(A.rows() * B.rows(), A.cols());
  for (Index k = 0; k < A.rows(); ++k)
    for (Index r = 0; r < A.cols(); ++r)
      for (Index i = 0; i < B.rows(); ++i) out(k * B.rows() + i, r) = B(i, r) * A(k, r);
  return out;
}

/// kernels.hpp:47-53 (host, element-wise).
inline Matrix hadamard(const Matrix& A, const Matrix& B) {
  if (A.rows() != B.rows() || A.cols() != B.cols()) throw std::invalid_argument("hadamard: operands differ in shape");
  ensure_finite(A, "hadamard left operand");
  ensure_finite(B, "hadamard right operand");
  Matrix C(A.rows(), A.cols());
  for (Index i = 0; i < A.size(); ++i) C.data()[i] = A.data()[i] * B.data()[i];
  return C;
}

/// kernels.hpp:57-63 -> p2g_gram (device, exactly symmetric).
inline Matrix gram(const Matrix& A) {
  Matrix G(A.cols(), A.cols());
  check(p2g_gram(Device::get().ctx(), A.data(), A.rows(), static_cast<int32_t>(A.cols()), G.data()));
  return G;
}

/// kernels.hpp:68-87 -> p2g_pinv_small (device).
inline Matrix pinv_small(const Matrix& G) {
  if (G.rows() != G.cols()) throw std::invalid_argument("pinv_small: matrix must be square");
  Matrix out(G.rows(), G.cols());
  check(p2g_pinv_small(Device::get().ctx(), G.data(), static_cast<int32_t>(G.rows()), out.data()));
  return out;
}

/// kernels.hpp:89-93.
struct EconomySvd {
  Matrix P;      // left singular vectors, m x rho
  Vector sigma;  // singular values, non-increasing, length rho
  Matrix Z;      // right singular vectors, n x rho
};

/// kernels.hpp:95-107 -> p2g_economy_svd (device, one-sided Jacobi): thin SVD
/// M = P diag(sigma) Z^T, rho = min(m, n); a zero matrix yields zero singular
/// values and identity-block factors; non-finite entries: NumericalError.
inline EconomySvd economy_svd(const Matrix& M) {
  const Index rho = std::min(M.rows(), M.cols());
  EconomySvd out{Matrix(M.rows(), rho), Vector(static_cast<std::size_t>(rho)), Matrix(M.cols(), rho)};
  check(p2g_economy_svd(Device::get().ctx(), M.data(), M.rows(), M.cols(), out.P.data(), out.sigma.data(),
                        out.Z.data()));
  return out;
}

/// kernels.hpp:194-211 -> p2g_nnls_rowwise (device; `threads` is host-only
/// in the reference and ignored here).
inline Matrix nnls_rowwise(const Matrix& G, const Matrix& B, int /*threads*/ = 1, int max_iter = 0) {
  if (G.rows() != G.cols()) throw std::invalid_argument("nnls_rowwise: G must be square");
  if (B.cols() != G.rows()) throw std::invalid_argument("nnls_rowwise: B column count must match G");
  Matrix X(B.rows(), B.cols());
  check(p2g_nnls_rowwise(Device::get().ctx(), G.data(), B.data(), B.rows(), static_cast<int32_t>(G.rows()), max_iter,
                         X.data()));
  return X;
}

}  // namespace parafac2
