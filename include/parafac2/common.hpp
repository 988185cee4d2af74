// Drop-in replacement for /root/reference/proj/include/parafac2/common.hpp on
// top of the libp2g C ABI (include/p2g.h).  Same namespace, type names and
// exception types as the reference; Matrix/Vector are a self-owned
// column-major type with the memory layout of Eigen::MatrixXd (decision D9:
// Eigen is not a dependency).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <initializer_list>
#include <limits>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../p2g.h"

namespace parafac2 {

using Index = std::ptrdiff_t;

/// common.hpp:37-39 — CLI exit code 2.
struct DataError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
/// common.hpp:43-45 — CLI exit code 3.
struct NumericalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
/// CUDA / NCCL failure or no usable device (the GPU path has no CPU fallback).
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

/// Maps a C-ABI status onto the reference's exception types.
inline void check(int status) {
  if (status == P2G_OK) return;
  const std::string msg = p2g_last_error();
  switch (status) {
    case P2G_EINVAL: throw std::invalid_argument(msg);
    case P2G_EDATA: throw DataError(msg);
    case P2G_ENUM: throw NumericalError(msg);
    default: throw DeviceError(msg);
  }
}

/// Column-major dense matrix (Eigen::MatrixXd layout).
class Matrix {
 public:
  Matrix() = default;
  Matrix(Index r, Index c) : r_(r), c_(c), d_(static_cast<std::size_t>(r * c), 0.0) {}
  static Matrix Zero(Index r, Index c) { return Matrix(r, c); }
  static Matrix Ones(Index r, Index c) { return Constant(r, c, 1.0); }
  static Matrix Constant(Index r, Index c, double v) {
    Matrix m(r, c);
    std::fill(m.d_.begin(), m.d_.end(), v);
    return m;
  }
  static Matrix Identity(Index r, Index c) {
    Matrix m(r, c);
    for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
    return m;
  }
  /// Row-major initializer, e.g. Matrix::FromRows(2, 2, {1, 2, 3, 4}).
  static Matrix FromRows(Index r, Index c, std::initializer_list<double> v) {
    Matrix m(r, c);
    Index k = 0;
    for (double x : v) {
      m(k / c, k % c) = x;
      ++k;
    }
    return m;
  }
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  double& operator()(Index i, Index j) { return d_[static_cast<std::size_t>(i + j * r_)]; }
  double operator()(Index i, Index j) const { return d_[static_cast<std::size_t>(i + j * r_)]; }
  void resize(Index r, Index c) {
    r_ = r;
    c_ = c;
    d_.assign(static_cast<std::size_t>(r * c), 0.0);
  }
  Matrix transpose() const {
    Matrix t(c_, r_);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) t(j, i) = (*this)(i, j);
    return t;
  }
  double squaredNorm() const {
    double a = 0.0;
    for (double v : d_) a += v * v;
    return a;
  }
  double norm() const { return std::sqrt(squaredNorm()); }
  bool allFinite() const {
    for (double v : d_)
      if (!std::isfinite(v)) return false;
    return true;
  }
  bool operator==(const Matrix& o) const { return r_ == o.r_ && c_ == o.c_ && d_ == o.d_; }
  bool operator!=(const Matrix& o) const { return !(*this == o); }
  Matrix operator-(const Matrix& o) const {
    Matrix m = *this;
    for (Index i = 0; i < size(); ++i) m.d_[static_cast<std::size_t>(i)] -= o.d_[static_cast<std::size_t>(i)];
    return m;
  }
  Matrix operator*(const Matrix& o) const {
    if (c_ != o.r_) throw std::invalid_argument("matrix product: shape mismatch");
    Matrix m(r_, o.c_);
    for (Index j = 0; j < o.c_; ++j)
      for (Index k = 0; k < c_; ++k) {
        const double b = o(k, j);
        for (Index i = 0; i < r_; ++i) m(i, j) += (*this)(i, k) * b;
      }
    return m;
  }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> d_;
};

using Vector = std::vector<double>;

/// common.hpp:50-53
inline void ensure_finite(const Matrix& m, const char* what) {
  if (!m.allFinite()) throw NumericalError(std::string(what) + ": non-finite entries");
}

/// common.hpp:65-76
inline std::uint64_t splitmix64(std::uint64_t& state) {
  std::uint64_t z = (state += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
inline std::uint64_t substream_seed(std::uint64_t seed, std::uint64_t idx) {
  std::uint64_t state = seed + idx * 0x9E3779B97F4A7C15ULL;
  return splitmix64(state);
}

/// common.hpp:78-121 — pinned PRNG (bit-exact: std::mt19937_64 is standard).
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : gen_(seed) {}
  std::uint64_t next_u64() { return gen_(); }
  double uniform() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  double normal() {
    if (have_spare_) {
      have_spare_ = false;
      return spare_;
    }
    const double u1 = 1.0 - uniform();
    const double u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 2.0 * M_PI * u2;
    spare_ = r * std::sin(a);
    have_spare_ = true;
    return r * std::cos(a);
  }
  std::uint64_t below(std::uint64_t n) {
    const std::uint64_t mx = std::numeric_limits<std::uint64_t>::max();
    const std::uint64_t limit = mx - mx % n;
    std::uint64_t x;
    do {
      x = gen_();
    } while (x >= limit);
    return x % n;
  }

 private:
  std::mt19937_64 gen_;
  double spare_ = 0.0;
  bool have_spare_ = false;
};

/// The process-wide device context used by the drop-in API (CUDA device 0
/// unless P2G_DEVICE is set).  The reference has no device state; this is the
/// one piece of state the GPU port needs.  Not thread-safe (like a solver).
class Device {
 public:
  static Device& get() {
    static Device d;
    return d;
  }
  p2g_ctx* ctx() {
    if (!ctx_) {
      const char* env = std::getenv("P2G_DEVICE");
      check(p2g_create(env ? std::atoi(env) : 0, 0, 1, nullptr, &ctx_));
    }
    return ctx_;
  }
  ~Device() {
    if (ctx_) p2g_destroy(ctx_);
  }

 private:
  p2g_ctx* ctx_ = nullptr;
};

}  // namespace parafac2
