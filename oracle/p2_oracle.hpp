// ============================================================================
// p2_oracle.hpp — CPU fp64 ORACLE for the SPARTan PARAFAC2-ALS hot path.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may build, import or run
// anything under oracle/.  The product path (paper_1703_04219_b200 + the
// C ABI in include/p2g.h) never links or calls this code.
//
// What it is: a restatement, without Eigen, of the reference library
// /root/reference/proj/include/parafac2 (the reference cannot be compiled in
// this container: Eigen 3.3+, Catch2 and CLI11 are absent — SURVEY.md F2).
// Each function cites the reference file:line whose behaviour it restates.
// Eigen primitives are replaced by:
//   * a column-major Mat (same layout as Eigen::MatrixXd),
//   * a cyclic Jacobi symmetric eigensolver sorted ascending
//     (replaces Eigen::SelfAdjointEigenSolver, kernels.hpp:75),
//   * a one-sided (Hestenes) Jacobi thin SVD sorted descending
//     (replaces Eigen::JacobiSVD, kernels.hpp:105),
//   * Householder QR with the sign fix of generator.hpp:44-45.
//
// Parity pinning: the reference ships no golden data files; its pins are the
// known-answer tests and property tests in proj/tests/*.cpp, which
// tests/test_oracle_*.py re-run against this oracle verbatim (same seeds —
// the Rng below is bit-exact with common.hpp:78-121 because std::mt19937_64
// is standardised).  The Jacobi eig/SVD are cross-checked against LAPACK
// (numpy/scipy) in tests.  The one place the reference is NOT reproducible
// without Eigen is the null-space completion of a rank-deficient Procrustes
// target: there this oracle and the GPU path both implement
// the canonical rule D5 documented at canonical_polar() below.
// ============================================================================
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <mutex>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

namespace p2o {

using Index = std::ptrdiff_t;

// ---------------------------------------------------------------------------
// Errors — common.hpp:37-45 (DataError → exit 2, NumericalError → exit 3).
// ---------------------------------------------------------------------------
struct DataError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------------------
// Column-major dense matrix (layout of Eigen::MatrixXd, common.hpp:30).
// ---------------------------------------------------------------------------
class Mat {
 public:
  Mat() = default;
  Mat(Index r, Index c, double fill = 0.0)
      : r_(r), c_(c), d_(static_cast<std::size_t>(r * c), fill) {}
  static Mat zeros(Index r, Index c) { return Mat(r, c, 0.0); }
  static Mat ones(Index r, Index c) { return Mat(r, c, 1.0); }
  static Mat identity(Index r, Index c) {
    Mat m(r, c, 0.0);
    for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
    return m;
  }
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  double& operator()(Index i, Index j) { return d_[static_cast<std::size_t>(i + j * r_)]; }
  double operator()(Index i, Index j) const { return d_[static_cast<std::size_t>(i + j * r_)]; }
  double* col(Index j) { return d_.data() + j * r_; }
  const double* col(Index j) const { return d_.data() + j * r_; }
  bool all_finite() const {
    for (double v : d_)
      if (!std::isfinite(v)) return false;
    return true;
  }
  bool is_zero() const {
    for (double v : d_)
      if (v != 0.0) return false;
    return true;
  }
  double squared_norm() const {
    double a = 0.0;
    for (double v : d_) a += v * v;
    return a;
  }
  double norm() const { return std::sqrt(squared_norm()); }
  Mat transpose() const {
    Mat t(c_, r_);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) t(j, i) = (*this)(i, j);
    return t;
  }
  bool operator==(const Mat& o) const { return r_ == o.r_ && c_ == o.c_ && d_ == o.d_; }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> d_;
};

using Vec = std::vector<double>;

inline Mat matmul(const Mat& A, const Mat& B) {
  if (A.cols() != B.rows()) throw std::invalid_argument("matmul: shape mismatch");
  Mat C(A.rows(), B.cols());
  for (Index j = 0; j < B.cols(); ++j)
    for (Index k = 0; k < A.cols(); ++k) {
      const double b = B(k, j);
      if (b == 0.0) continue;
      const double* a = A.col(k);
      double* c = C.col(j);
      for (Index i = 0; i < A.rows(); ++i) c[i] += a[i] * b;
    }
  return C;
}

/// A^T B without forming the transpose.
inline Mat matmul_tn(const Mat& A, const Mat& B) {
  if (A.rows() != B.rows()) throw std::invalid_argument("matmul_tn: shape mismatch");
  Mat C(A.cols(), B.cols());
  for (Index j = 0; j < B.cols(); ++j)
    for (Index i = 0; i < A.cols(); ++i) {
      double acc = 0.0;
      const double* a = A.col(i);
      const double* b = B.col(j);
      for (Index k = 0; k < A.rows(); ++k) acc += a[k] * b[k];
      C(i, j) = acc;
    }
  return C;
}

/// common.hpp:50-53
inline void ensure_finite(const Mat& m, const char* what) {
  if (!m.all_finite()) throw NumericalError(std::string(what) + ": non-finite entries");
}

// ---------------------------------------------------------------------------
// Pinned PRNG — common.hpp:65-121 (bit-exact: std::mt19937_64 is standard).
// ---------------------------------------------------------------------------
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

// ---------------------------------------------------------------------------
// Deterministic chunking — parallel.hpp:34-124.
// ---------------------------------------------------------------------------
using Ranges = std::vector<std::pair<Index, Index>>;

/// parallel.hpp:34-45
inline Ranges partition_even(Index n, int n_chunks) {
  const Index chunks = std::max<Index>(1, std::min<Index>(n_chunks, std::max<Index>(n, 1)));
  Ranges out;
  for (Index c = 0; c < chunks; ++c) out.emplace_back(n * c / chunks, n * (c + 1) / chunks);
  return out;
}

/// parallel.hpp:51-79 — contiguous ranges of ~equal cumulative weight; at least
/// one element per range and one left for every later range.
inline Ranges partition_weighted(const std::vector<std::uint64_t>& weights, int n_chunks) {
  const Index n = static_cast<Index>(weights.size());
  const Index chunks = std::max<Index>(1, std::min<Index>(n_chunks, std::max<Index>(n, 1)));
  std::uint64_t total = 0;
  for (std::uint64_t w : weights) total += w;
  if (total == 0) return partition_even(n, static_cast<int>(chunks));
  Ranges out;
  Index begin = 0;
  std::uint64_t cum = 0;
  for (Index c = 0; c < chunks; ++c) {
    const std::uint64_t target =
        total * static_cast<std::uint64_t>(c + 1) / static_cast<std::uint64_t>(chunks);
    Index end = begin;
    while (end < n && (cum < target || end == begin) && n - end > chunks - c - 1) {
      cum += weights[static_cast<std::size_t>(end)];
      ++end;
    }
    if (c + 1 == chunks) end = n;
    out.emplace_back(begin, end);
    begin = end;
  }
  return out;
}

/// parallel.hpp:86-108 — chunk 0 inline, one std::thread per other chunk,
/// first exception rethrown on the caller.
template <typename Fn>
void run_chunks(const Ranges& chunks, Fn&& fn) {
  if (chunks.size() == 1) {
    fn(std::size_t{0}, chunks[0].first, chunks[0].second);
    return;
  }
  std::exception_ptr first_error;
  std::mutex mu;
  auto guarded = [&](std::size_t c) {
    try {
      fn(c, chunks[c].first, chunks[c].second);
    } catch (...) {
      std::lock_guard<std::mutex> lock(mu);
      if (!first_error) first_error = std::current_exception();
    }
  };
  std::vector<std::thread> workers;
  for (std::size_t c = 1; c < chunks.size(); ++c) workers.emplace_back(guarded, c);
  guarded(0);
  for (auto& t : workers) t.join();
  if (first_error) std::rethrow_exception(first_error);
}

/// parallel.hpp:115-124 — fixed pairwise tree.
template <typename T, typename Merge>
T merge_tree(std::vector<T> parts, Merge&& merge) {
  while (parts.size() > 1) {
    std::size_t out = 0;
    for (std::size_t i = 0; i + 1 < parts.size(); i += 2)
      parts[out++] = merge(std::move(parts[i]), std::move(parts[i + 1]));
    if (parts.size() % 2 == 1) parts[out++] = std::move(parts.back());
    parts.resize(out);
  }
  return std::move(parts.front());
}

// ---------------------------------------------------------------------------
// Sparse slices — sparse.hpp:40-223.
// ---------------------------------------------------------------------------
struct Triplet {
  Index row;
  Index col;
  double value;
};

class SparseSlice {
 public:
  SparseSlice() = default;

  /// sparse.hpp:47-86: sort by (col,row), sum duplicates, drop exact zeros.
  static SparseSlice from_triplets(Index n_rows, Index n_cols, std::vector<Triplet> e) {
    if (n_rows < 0 || n_cols < 0) throw std::invalid_argument("slice dimensions must be non-negative");
    for (const Triplet& t : e) {
      if (t.row < 0 || t.row >= n_rows) throw std::invalid_argument("slice row index out of range");
      if (t.col < 0 || t.col >= n_cols) throw std::invalid_argument("slice column index out of range");
    }
    std::sort(e.begin(), e.end(), [](const Triplet& a, const Triplet& b) {
      return a.col != b.col ? a.col < b.col : a.row < b.row;
    });
    SparseSlice s;
    s.n_rows_ = n_rows;
    s.n_cols_ = n_cols;
    std::size_t i = 0;
    while (i < e.size()) {
      std::size_t j = i + 1;
      double v = e[i].value;
      while (j < e.size() && e[j].col == e[i].col && e[j].row == e[i].row) v += e[j++].value;
      if (v != 0.0) {
        if (s.nnz_cols_.empty() || s.nnz_cols_.back() != e[i].col) {
          s.nnz_cols_.push_back(e[i].col);
          s.col_start_.push_back(static_cast<Index>(s.row_idx_.size()));
        }
        s.row_idx_.push_back(e[i].row);
        s.values_.push_back(v);
      }
      i = j;
    }
    s.col_start_.push_back(static_cast<Index>(s.row_idx_.size()));
    return s;
  }

  Index n_rows() const { return n_rows_; }
  Index n_cols() const { return n_cols_; }
  Index nnz() const { return static_cast<Index>(values_.size()); }
  Index n_nnz_cols() const { return static_cast<Index>(nnz_cols_.size()); }
  const std::vector<Index>& nnz_cols() const { return nnz_cols_; }
  Index col(Index c) const { return nnz_cols_[static_cast<std::size_t>(c)]; }
  std::pair<Index, Index> col_range(Index c) const {
    return {col_start_[static_cast<std::size_t>(c)], col_start_[static_cast<std::size_t>(c) + 1]};
  }
  Index entry_row(Index p) const { return row_idx_[static_cast<std::size_t>(p)]; }
  double entry_value(Index p) const { return values_[static_cast<std::size_t>(p)]; }

  /// sparse.hpp:111-115 (storage order).
  double frobenius_sq() const {
    double acc = 0.0;
    for (double v : values_) acc += v * v;
    return acc;
  }
  Mat dense() const {
    Mat d(n_rows_, n_cols_);
    for (Index c = 0; c < n_nnz_cols(); ++c) {
      auto [p0, p1] = col_range(c);
      for (Index p = p0; p < p1; ++p) d(entry_row(p), col(c)) = entry_value(p);
    }
    return d;
  }
  std::vector<Triplet> triplets() const {
    std::vector<Triplet> out;
    for (Index c = 0; c < n_nnz_cols(); ++c) {
      auto [p0, p1] = col_range(c);
      for (Index p = p0; p < p1; ++p) out.push_back({entry_row(p), col(c), entry_value(p)});
    }
    return out;
  }

 private:
  Index n_rows_ = 0, n_cols_ = 0;
  std::vector<Index> nnz_cols_, col_start_, row_idx_;
  std::vector<double> values_;
};

/// sparse.hpp:155-172
inline std::pair<SparseSlice, std::vector<Index>> filter_zero_rows(const SparseSlice& s) {
  if (s.nnz() == 0) throw DataError("empty slice: no non-zero entries");
  std::vector<Triplet> e = s.triplets();
  std::vector<Index> row_map;
  for (const Triplet& t : e) row_map.push_back(t.row);
  std::sort(row_map.begin(), row_map.end());
  row_map.erase(std::unique(row_map.begin(), row_map.end()), row_map.end());
  for (Triplet& t : e)
    t.row = static_cast<Index>(std::lower_bound(row_map.begin(), row_map.end(), t.row) - row_map.begin());
  SparseSlice f = SparseSlice::from_triplets(static_cast<Index>(row_map.size()), s.n_cols(), std::move(e));
  return {std::move(f), std::move(row_map)};
}

/// sparse.hpp:176-215
class IrregularTensor {
 public:
  static IrregularTensor from_slices(Index n_cols, std::vector<SparseSlice> slices) {
    if (n_cols <= 0) throw DataError("tensor must have at least one column");
    if (slices.empty()) throw DataError("tensor must have at least one slice");
    IrregularTensor t;
    t.n_cols_ = n_cols;
    for (std::size_t k = 0; k < slices.size(); ++k) {
      if (slices[k].n_cols() != n_cols)
        throw DataError("slice " + std::to_string(k) + " column count differs from tensor column count");
      t.total_nnz_ += static_cast<std::uint64_t>(slices[k].nnz());
    }
    t.slices_ = std::move(slices);
    return t;
  }
  Index n_cols() const { return n_cols_; }
  Index n_slices() const { return static_cast<Index>(slices_.size()); }
  std::uint64_t total_nnz() const { return total_nnz_; }
  const SparseSlice& slice(Index k) const { return slices_[static_cast<std::size_t>(k)]; }
  Index max_rows() const {
    Index m = 0;
    for (const auto& s : slices_) m = std::max(m, s.n_rows());
    return m;
  }

 private:
  Index n_cols_ = 0;
  std::vector<SparseSlice> slices_;
  std::uint64_t total_nnz_ = 0;
};

/// sparse.hpp:219-223
inline double frobenius_sq(const IrregularTensor& t) {
  double acc = 0.0;
  for (Index k = 0; k < t.n_slices(); ++k) acc += t.slice(k).frobenius_sq();
  return acc;
}

// ---------------------------------------------------------------------------
// Projected slices Y_k — slices.hpp:37-129.
// ---------------------------------------------------------------------------
class ProjectedSlices {
 public:
  /// slices.hpp:43-67
  static ProjectedSlices from_packed(Index rank, Index n_cols, std::vector<Mat> packed,
                                     std::vector<std::vector<Index>> cols) {
    if (rank <= 0) throw std::invalid_argument("slice rank must be positive");
    if (packed.size() != cols.size()) throw std::invalid_argument("packed blocks and column lists differ in count");
    for (std::size_t k = 0; k < packed.size(); ++k) {
      if (packed[k].rows() != rank) throw std::invalid_argument("packed block row count differs from rank");
      if (packed[k].cols() != static_cast<Index>(cols[k].size()))
        throw std::invalid_argument("packed block width differs from column list");
      for (std::size_t c = 0; c < cols[k].size(); ++c) {
        if (cols[k][c] < 0 || cols[k][c] >= n_cols) throw std::invalid_argument("packed column index out of range");
        if (c > 0 && cols[k][c] <= cols[k][c - 1])
          throw std::invalid_argument("packed column indices must be ascending");
      }
    }
    ProjectedSlices y;
    y.rank_ = rank;
    y.n_cols_ = n_cols;
    y.packed_ = std::move(packed);
    y.cols_ = std::move(cols);
    return y;
  }
  /// slices.hpp:71-86
  static ProjectedSlices from_dense(Index n_cols, const std::vector<Mat>& dense) {
    std::vector<Mat> packed(dense.size());
    std::vector<std::vector<Index>> cols(dense.size());
    Index rank = dense.empty() ? 0 : dense.front().rows();
    for (std::size_t k = 0; k < dense.size(); ++k) {
      if (dense[k].cols() != n_cols) throw std::invalid_argument("dense slice column count mismatch");
      for (Index j = 0; j < n_cols; ++j) {
        bool nz = false;
        for (Index i = 0; i < dense[k].rows(); ++i) nz |= dense[k](i, j) != 0.0;
        if (nz) cols[k].push_back(j);
      }
      packed[k] = Mat(dense[k].rows(), static_cast<Index>(cols[k].size()));
      for (std::size_t c = 0; c < cols[k].size(); ++c)
        for (Index i = 0; i < dense[k].rows(); ++i) packed[k](i, static_cast<Index>(c)) = dense[k](i, cols[k][c]);
    }
    return from_packed(rank, n_cols, std::move(packed), std::move(cols));
  }
  Index rank() const { return rank_; }
  Index n_cols() const { return n_cols_; }
  Index n_slices() const { return static_cast<Index>(packed_.size()); }
  const Mat& packed(Index k) const { return packed_[static_cast<std::size_t>(k)]; }
  const std::vector<Index>& cols(Index k) const { return cols_[static_cast<std::size_t>(k)]; }
  Index n_nnz_cols(Index k) const { return static_cast<Index>(cols_[static_cast<std::size_t>(k)].size()); }
  Mat dense(Index k) const {
    Mat d(rank_, n_cols_);
    const auto& c = cols(k);
    const Mat& p = packed(k);
    for (std::size_t i = 0; i < c.size(); ++i)
      for (Index r = 0; r < rank_; ++r) d(r, c[i]) = p(r, static_cast<Index>(i));
    return d;
  }
  double frobenius_sq() const {
    double acc = 0.0;
    for (const Mat& p : packed_) acc += p.squared_norm();
    return acc;
  }

 private:
  Index rank_ = 0, n_cols_ = 0;
  std::vector<Mat> packed_;
  std::vector<std::vector<Index>> cols_;
};

// ---------------------------------------------------------------------------
// Dense kernels — kernels.hpp:34-211.
// ---------------------------------------------------------------------------

/// kernels.hpp:34-44
inline Mat khatri_rao(const Mat& A, const Mat& B) {
  if (A.cols() != B.cols()) throw std::invalid_argument("khatri_rao: operands differ in column count");
  ensure_finite(A, "khatri_rao left operand");
  ensure_finite(B, "khatri_rao right operand");
  Mat out(A.rows() * B.rows(), A.cols());
  for (Index k = 0; k < A.rows(); ++k)
    for (Index r = 0; r < A.cols(); ++r)
      for (Index i = 0; i < B.rows(); ++i) out(k * B.rows() + i, r) = B(i, r) * A(k, r);
  return out;
}

/// kernels.hpp:47-53
inline Mat hadamard(const Mat& A, const Mat& B) {
  if (A.rows() != B.rows() || A.cols() != B.cols()) throw std::invalid_argument("hadamard: operands differ in shape");
  ensure_finite(A, "hadamard left operand");
  ensure_finite(B, "hadamard right operand");
  Mat C(A.rows(), A.cols());
  for (Index i = 0; i < A.size(); ++i) C.data()[i] = A.data()[i] * B.data()[i];
  return C;
}

/// kernels.hpp:57-63 — A^T A, exactly symmetric (lower computed, mirrored).
inline Mat gram(const Mat& A) {
  ensure_finite(A, "gram operand");
  const Index n = A.cols();
  Mat G(n, n);
  for (Index j = 0; j < n; ++j)
    for (Index i = j; i < n; ++i) {
      double acc = 0.0;
      const double* a = A.col(i);
      const double* b = A.col(j);
      for (Index k = 0; k < A.rows(); ++k) acc += a[k] * b[k];
      G(i, j) = acc;
      G(j, i) = acc;
    }
  return G;
}

/// Cyclic Jacobi eigensolver for a symmetric matrix; eigenvalues ascending
/// with matching eigenvector columns (the contract of Eigen's
/// SelfAdjointEigenSolver used at kernels.hpp:75 and solver.hpp:160).
struct SymEig {
  Vec values;
  Mat vectors;
};

inline SymEig sym_eig(const Mat& S) {
  const Index n = S.rows();
  Mat a = S;
  Mat v = Mat::identity(n, n);
  // Scale for robustness (eigenvectors are scale invariant).
  double amax = 0.0;
  for (Index i = 0; i < a.size(); ++i) amax = std::max(amax, std::abs(a.data()[i]));
  const double scale = amax > 0.0 ? amax : 1.0;
  for (Index i = 0; i < a.size(); ++i) a.data()[i] /= scale;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (Index j = 0; j < n; ++j) {
      diag += a(j, j) * a(j, j);
      for (Index i = j + 1; i < n; ++i) off += a(i, j) * a(i, j);
    }
    if (off <= 1e-34 * std::max(diag, 1e-300) || off == 0.0) break;
    for (Index p = 0; p < n - 1; ++p)
      for (Index q = p + 1; q < n; ++q) {
        const double apq = a(p, q);
        if (apq == 0.0) continue;
        const double app = a(p, p), aqq = a(q, q);
        if (std::abs(apq) <= 1e-300) continue;
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0);
        const double s = t * c;
        for (Index k = 0; k < n; ++k) {  // columns p,q
          const double akp = a(k, p), akq = a(k, q);
          a(k, p) = c * akp - s * akq;
          a(k, q) = s * akp + c * akq;
        }
        for (Index k = 0; k < n; ++k) {  // rows p,q
          const double apk = a(p, k), aqk = a(q, k);
          a(p, k) = c * apk - s * aqk;
          a(q, k) = s * apk + c * aqk;
        }
        a(p, q) = 0.0;
        a(q, p) = 0.0;
        for (Index k = 0; k < n; ++k) {
          const double vkp = v(k, p), vkq = v(k, q);
          v(k, p) = c * vkp - s * vkq;
          v(k, q) = s * vkp + c * vkq;
        }
      }
  }
  std::vector<Index> order(static_cast<std::size_t>(n));
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](Index x, Index y) { return a(x, x) < a(y, y); });
  SymEig out;
  out.values.resize(static_cast<std::size_t>(n));
  out.vectors = Mat(n, n);
  for (Index c = 0; c < n; ++c) {
    const Index src = order[static_cast<std::size_t>(c)];
    out.values[static_cast<std::size_t>(c)] = a(src, src) * scale;
    for (Index k = 0; k < n; ++k) out.vectors(k, c) = v(k, src);
  }
  return out;
}

/// kernels.hpp:68-87 — symmetrize, eig, drop eigenvalues <= 1e-12*max|ev|.
inline Mat pinv_small(const Mat& G) {
  if (G.rows() != G.cols()) throw std::invalid_argument("pinv_small: matrix must be square");
  ensure_finite(G, "pseudoinverse operand");
  const Index n = G.rows();
  Mat S(n, n);
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < n; ++i) S(i, j) = 0.5 * (G(i, j) + G(j, i));
  const SymEig e = sym_eig(S);
  double amax = 0.0;
  for (double x : e.values) amax = std::max(amax, std::abs(x));
  const double cutoff = 1e-12 * std::max(amax, 0.0);
  Mat out(n, n);
  for (Index i = 0; i < n; ++i) {
    const double ev = e.values[static_cast<std::size_t>(i)];
    if (ev > cutoff && ev > 0.0) {
      const double* v = e.vectors.col(i);
      for (Index c = 0; c < n; ++c)
        for (Index r = c; r < n; ++r) out(r, c) += v[r] * v[c] / ev;
    }
  }
  for (Index c = 0; c < n; ++c)
    for (Index r = c + 1; r < n; ++r) out(c, r) = out(r, c);
  return out;
}

/// One-sided (Hestenes) Jacobi SVD of a tall matrix A (m x n, m >= n):
/// A = U diag(sigma) V^T with sigma descending, V n x n orthogonal, U m x n
/// (columns for zero singular values are left zero; callers complete them).
struct Svd {
  Mat U;
  Vec sigma;
  Mat V;
};

inline Svd one_sided_jacobi(const Mat& A0) {
  const Index m = A0.rows(), n = A0.cols();
  Mat A = A0;
  double amax = 0.0;
  for (Index i = 0; i < A.size(); ++i) amax = std::max(amax, std::abs(A.data()[i]));
  const double scale = amax > 0.0 ? amax : 1.0;
  for (Index i = 0; i < A.size(); ++i) A.data()[i] /= scale;
  Mat V = Mat::identity(n, n);
  const double tol = 1e-15;
  for (int sweep = 0; sweep < 80; ++sweep) {
    bool rotated = false;
    for (Index p = 0; p < n - 1; ++p)
      for (Index q = p + 1; q < n; ++q) {
        double alpha = 0.0, beta = 0.0, gamma = 0.0;
        const double* ap = A.col(p);
        const double* aq = A.col(q);
        for (Index i = 0; i < m; ++i) {
          alpha += ap[i] * ap[i];
          beta += aq[i] * aq[i];
          gamma += ap[i] * aq[i];
        }
        if (gamma == 0.0 || std::abs(gamma) <= tol * std::sqrt(alpha * beta)) continue;
        rotated = true;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t);
        const double s = c * t;
        double* xp = A.col(p);
        double* xq = A.col(q);
        for (Index i = 0; i < m; ++i) {
          const double u = xp[i], w = xq[i];
          xp[i] = c * u - s * w;
          xq[i] = s * u + c * w;
        }
        double* vp = V.col(p);
        double* vq = V.col(q);
        for (Index i = 0; i < n; ++i) {
          const double u = vp[i], w = vq[i];
          vp[i] = c * u - s * w;
          vq[i] = s * u + c * w;
        }
      }
    if (!rotated) break;
  }
  Vec sig(static_cast<std::size_t>(n));
  for (Index j = 0; j < n; ++j) {
    double acc = 0.0;
    for (Index i = 0; i < m; ++i) acc += A(i, j) * A(i, j);
    sig[static_cast<std::size_t>(j)] = std::sqrt(acc);
  }
  std::vector<Index> order(static_cast<std::size_t>(n));
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](Index x, Index y) { return sig[static_cast<std::size_t>(x)] > sig[static_cast<std::size_t>(y)]; });
  Svd out;
  out.U = Mat(m, n);
  out.V = Mat(n, n);
  out.sigma.resize(static_cast<std::size_t>(n));
  for (Index c = 0; c < n; ++c) {
    const Index src = order[static_cast<std::size_t>(c)];
    const double s = sig[static_cast<std::size_t>(src)];
    out.sigma[static_cast<std::size_t>(c)] = s * scale;
    for (Index k = 0; k < n; ++k) out.V(k, c) = V(k, src);
    if (s > 0.0)
      for (Index i = 0; i < m; ++i) out.U(i, c) = A(i, src) / s;
  }
  return out;
}

/// Completes the zero columns of a matrix with orthonormal columns (Gram-
/// Schmidt over unit vectors, twice) so the result is column-orthonormal.
inline void complete_orthonormal(Mat& U, Index from_col) {
  const Index m = U.rows();
  Index cand = 0;
  for (Index c = from_col; c < U.cols(); ++c) {
    while (cand < m) {
      Vec x(static_cast<std::size_t>(m), 0.0);
      x[static_cast<std::size_t>(cand++)] = 1.0;
      for (int pass = 0; pass < 2; ++pass)
        for (Index j = 0; j < c; ++j) {
          double d = 0.0;
          for (Index i = 0; i < m; ++i) d += U(i, j) * x[static_cast<std::size_t>(i)];
          for (Index i = 0; i < m; ++i) x[static_cast<std::size_t>(i)] -= d * U(i, j);
        }
      double nn = 0.0;
      for (double xi : x) nn += xi * xi;
      nn = std::sqrt(nn);
      if (nn > 0.5) {
        for (Index i = 0; i < m; ++i) U(i, c) = x[static_cast<std::size_t>(i)] / nn;
        break;
      }
    }
  }
}

/// kernels.hpp:92-107 — thin SVD M = P diag(sigma) Z^T, rho = min(m, n);
/// exact-zero M yields identity blocks (kernels.hpp:101-104).
struct EconomySvd {
  Mat P;
  Vec sigma;
  Mat Z;
};

inline EconomySvd economy_svd(const Mat& M) {
  ensure_finite(M, "svd operand");
  const Index m = M.rows(), n = M.cols(), rho = std::min(m, n);
  if (M.is_zero())
    return {Mat::identity(m, rho), Vec(static_cast<std::size_t>(rho), 0.0), Mat::identity(n, rho)};
  EconomySvd out;
  if (m >= n) {
    Svd s = one_sided_jacobi(M);
    Index nz = 0;
    while (nz < n && s.sigma[static_cast<std::size_t>(nz)] > 0.0) ++nz;
    complete_orthonormal(s.U, nz);
    out = {s.U, s.sigma, s.V};
  } else {
    Svd s = one_sided_jacobi(M.transpose());
    Index nz = 0;
    while (nz < m && s.sigma[static_cast<std::size_t>(nz)] > 0.0) ++nz;
    complete_orthonormal(s.U, nz);
    out = {s.V, s.sigma, s.U};
  }
  return out;
}

namespace detail {

/// kernels.hpp:115-185 — active-set NNLS for one right-hand side on the
/// normal equations; passive solves via pinv_small; cap -> NumericalError.
inline Vec nnls_single(const Mat& G, const Vec& b, int max_iter) {
  const Index n = G.rows();
  const double kkt_tol = 1e-10;
  std::vector<char> passive(static_cast<std::size_t>(n), 0);
  std::vector<Index> pset;
  Vec x(static_cast<std::size_t>(n), 0.0), w = b, s(static_cast<std::size_t>(n), 0.0);
  int iters = 0;
  while (true) {
    Index enter = -1;
    double best = kkt_tol;
    for (Index j = 0; j < n; ++j)
      if (!passive[static_cast<std::size_t>(j)] && w[static_cast<std::size_t>(j)] > best) {
        best = w[static_cast<std::size_t>(j)];
        enter = j;
      }
    if (enter < 0) break;
    passive[static_cast<std::size_t>(enter)] = 1;
    while (true) {
      if (++iters > max_iter) throw NumericalError("NNLS did not converge");
      pset.clear();
      for (Index j = 0; j < n; ++j)
        if (passive[static_cast<std::size_t>(j)]) pset.push_back(j);
      const Index np = static_cast<Index>(pset.size());
      Mat Gpp(np, np);
      Vec bp(static_cast<std::size_t>(np));
      for (Index a = 0; a < np; ++a) {
        bp[static_cast<std::size_t>(a)] = b[static_cast<std::size_t>(pset[static_cast<std::size_t>(a)])];
        for (Index c = 0; c < np; ++c)
          Gpp(a, c) = G(pset[static_cast<std::size_t>(a)], pset[static_cast<std::size_t>(c)]);
      }
      const Mat P = pinv_small(Gpp);
      Vec sp(static_cast<std::size_t>(np), 0.0);
      for (Index a = 0; a < np; ++a) {
        double acc = 0.0;
        for (Index c = 0; c < np; ++c) acc += P(a, c) * bp[static_cast<std::size_t>(c)];
        sp[static_cast<std::size_t>(a)] = acc;
      }
      bool all_pos = true;
      for (double v : sp) all_pos &= v > 0.0;
      if (all_pos) {
        std::fill(x.begin(), x.end(), 0.0);
        for (Index a = 0; a < np; ++a) x[static_cast<std::size_t>(pset[static_cast<std::size_t>(a)])] = sp[static_cast<std::size_t>(a)];
        break;
      }
      std::fill(s.begin(), s.end(), 0.0);
      for (Index a = 0; a < np; ++a) s[static_cast<std::size_t>(pset[static_cast<std::size_t>(a)])] = sp[static_cast<std::size_t>(a)];
      double alpha = std::numeric_limits<double>::infinity();
      for (Index a = 0; a < np; ++a) {
        const std::size_t j = static_cast<std::size_t>(pset[static_cast<std::size_t>(a)]);
        if (sp[static_cast<std::size_t>(a)] <= 0.0) {
          const double denom = x[j] - s[j];
          const double step = denom > 0.0 ? x[j] / denom : 0.0;
          alpha = std::min(alpha, step);
        }
      }
      for (Index a = 0; a < np; ++a) {
        const std::size_t j = static_cast<std::size_t>(pset[static_cast<std::size_t>(a)]);
        x[j] += alpha * (s[j] - x[j]);
      }
      double xmax = 0.0;
      for (double v : x) xmax = std::max(xmax, std::abs(v));
      const double drop_tol = 1e-14 * std::max(1.0, xmax);
      for (Index a = 0; a < np; ++a) {
        const std::size_t j = static_cast<std::size_t>(pset[static_cast<std::size_t>(a)]);
        if (x[j] <= drop_tol) {
          x[j] = 0.0;
          passive[j] = 0;
        }
      }
    }
    for (Index j = 0; j < n; ++j) {
      double acc = 0.0;
      for (Index c = 0; c < n; ++c) acc += G(j, c) * x[static_cast<std::size_t>(c)];
      w[static_cast<std::size_t>(j)] = b[static_cast<std::size_t>(j)] - acc;
    }
  }
  return x;
}

}  // namespace detail

/// kernels.hpp:194-211
inline Mat nnls_rowwise(const Mat& G, const Mat& B, int threads = 1, int max_iter = 0) {
  if (G.rows() != G.cols()) throw std::invalid_argument("nnls_rowwise: G must be square");
  if (B.cols() != G.rows()) throw std::invalid_argument("nnls_rowwise: B column count must match G");
  ensure_finite(G, "nonnegative solve normal matrix");
  ensure_finite(B, "nonnegative solve right-hand side");
  const int cap = max_iter > 0 ? max_iter : 30 * static_cast<int>(G.rows());
  Mat X(B.rows(), B.cols());
  run_chunks(partition_even(B.rows(), threads > 0 ? threads : 1), [&](std::size_t, Index b0, Index b1) {
    Vec row(static_cast<std::size_t>(B.cols()));
    for (Index j = b0; j < b1; ++j) {
      for (Index c = 0; c < B.cols(); ++c) row[static_cast<std::size_t>(c)] = B(j, c);
      const Vec x = detail::nnls_single(G, row, cap);
      for (Index c = 0; c < B.cols(); ++c) X(j, c) = x[static_cast<std::size_t>(c)];
    }
  });
  return X;
}

// ---------------------------------------------------------------------------
// Slice-wise MTTKRP — mttkrp.hpp:47-253.
// ---------------------------------------------------------------------------
namespace detail {
inline void check_factor(const Mat& F, Index rows, Index cols, const char* name) {
  if (F.rows() != rows || F.cols() != cols)
    throw std::invalid_argument(std::string("mttkrp: factor ") + name + " has mismatched dimensions");
}
/// mttkrp.hpp:58-64
inline std::vector<std::uint64_t> slice_weights(const ProjectedSlices& Y) {
  std::vector<std::uint64_t> w(static_cast<std::size_t>(Y.n_slices()));
  for (Index k = 0; k < Y.n_slices(); ++k) w[static_cast<std::size_t>(k)] = static_cast<std::uint64_t>(Y.n_nnz_cols(k));
  return w;
}
/// Y_k * V(cols_k, :) without reading V rows outside cols_k (mttkrp.hpp:69-75,99-100).
inline Mat packed_times_gathered(const Mat& Yk, const std::vector<Index>& cols, const Mat& V) {
  const Index R = Yk.rows(), F = V.cols();
  Mat prod(R, F);
  for (Index f = 0; f < F; ++f)
    for (std::size_t c = 0; c < cols.size(); ++c) {
      const double v = V(cols[c], f);
      const double* y = Yk.col(static_cast<Index>(c));
      double* p = prod.col(f);
      for (Index r = 0; r < R; ++r) p[r] += y[r] * v;
    }
  return prod;
}
}  // namespace detail

/// mttkrp.hpp:81-106
inline Mat mttkrp_mode1(const ProjectedSlices& Y, const Mat& V, const Mat& W, int threads = 1) {
  const Index R = Y.rank();
  detail::check_factor(V, Y.n_cols(), V.cols(), "V");
  detail::check_factor(W, Y.n_slices(), V.cols(), "W");
  const Index F = V.cols();
  const Ranges chunks = partition_weighted(detail::slice_weights(Y), threads);
  std::vector<Mat> parts(chunks.size(), Mat(R, F));
  run_chunks(chunks, [&](std::size_t c, Index b, Index e) {
    Mat& acc = parts[c];
    for (Index k = b; k < e; ++k) {
      if (Y.n_nnz_cols(k) == 0) continue;
      const Mat prod = detail::packed_times_gathered(Y.packed(k), Y.cols(k), V);
      for (Index f = 0; f < F; ++f)
        for (Index r = 0; r < R; ++r) acc(r, f) += prod(r, f) * W(k, f);
    }
  });
  return merge_tree(std::move(parts), [](Mat a, const Mat& b) {
    for (Index i = 0; i < a.size(); ++i) a.data()[i] += b.data()[i];
    return a;
  });
}

/// mttkrp.hpp:111-138
inline Mat mttkrp_mode2(const ProjectedSlices& Y, const Mat& H, const Mat& W, int threads = 1) {
  const Index R = Y.rank();
  detail::check_factor(H, R, H.cols(), "H");
  detail::check_factor(W, Y.n_slices(), H.cols(), "W");
  const Index F = H.cols();
  const Ranges chunks = partition_weighted(detail::slice_weights(Y), threads);
  std::vector<Mat> parts(chunks.size(), Mat(Y.n_cols(), F));
  run_chunks(chunks, [&](std::size_t c, Index b, Index e) {
    Mat& acc = parts[c];
    for (Index k = b; k < e; ++k) {
      const Index ck = Y.n_nnz_cols(k);
      if (ck == 0) continue;
      const Mat& Yk = Y.packed(k);
      const auto& cols = Y.cols(k);
      for (Index i = 0; i < ck; ++i)
        for (Index f = 0; f < F; ++f) {
          double t = 0.0;  // (Y_k^T H)(i, f)
          for (Index r = 0; r < R; ++r) t += Yk(r, i) * H(r, f);
          acc(cols[static_cast<std::size_t>(i)], f) += t * W(k, f);
        }
    }
  });
  return merge_tree(std::move(parts), [](Mat a, const Mat& b) {
    for (Index i = 0; i < a.size(); ++i) a.data()[i] += b.data()[i];
    return a;
  });
}

/// mttkrp.hpp:143-166
inline Mat mttkrp_mode3(const ProjectedSlices& Y, const Mat& H, const Mat& V, int threads = 1) {
  const Index R = Y.rank();
  detail::check_factor(H, R, H.cols(), "H");
  detail::check_factor(V, Y.n_cols(), H.cols(), "V");
  const Index F = H.cols();
  Mat M(Y.n_slices(), F);
  run_chunks(partition_weighted(detail::slice_weights(Y), threads), [&](std::size_t, Index b, Index e) {
    for (Index k = b; k < e; ++k) {
      if (Y.n_nnz_cols(k) == 0) continue;
      const Mat prod = detail::packed_times_gathered(Y.packed(k), Y.cols(k), V);
      for (Index f = 0; f < F; ++f) {
        double acc = 0.0;
        for (Index r = 0; r < R; ++r) acc += H(r, f) * prod(r, f);
        M(k, f) = acc;
      }
    }
  });
  return M;
}

/// mttkrp.hpp:170-181
inline void check_mttkrp_input(const ProjectedSlices& Y, const Mat& H, const Mat& V, const Mat& W, int mode) {
  if (mode < 1 || mode > 3) throw std::invalid_argument("mttkrp: mode must be 1, 2 or 3");
  const Index R = Y.rank();
  if (H.rows() != R || H.cols() != R) throw std::invalid_argument("mttkrp: H must be R x R");
  if (V.rows() != Y.n_cols() || V.cols() != R) throw std::invalid_argument("mttkrp: V must be J x R");
  if (W.rows() != Y.n_slices() || W.cols() != R) throw std::invalid_argument("mttkrp: W must be K x R");
}

/// mttkrp.hpp:187-196
inline Mat mttkrp(const ProjectedSlices& Y, const Mat& H, const Mat& V, const Mat& W, int mode, int threads = 1) {
  check_mttkrp_input(Y, H, V, W, mode);
  switch (mode) {
    case 1: return mttkrp_mode1(Y, V, W, threads);
    case 2: return mttkrp_mode2(Y, H, W, threads);
    default: return mttkrp_mode3(Y, H, V, threads);
  }
}

/// mttkrp.hpp:208-235 — materialized unfolding times Khatri-Rao (test oracle).
inline Mat naive_mttkrp(const ProjectedSlices& Y, const Mat& H, const Mat& V, const Mat& W, int mode) {
  check_mttkrp_input(Y, H, V, W, mode);
  const Index R = Y.rank(), J = Y.n_cols(), K = Y.n_slices();
  switch (mode) {
    case 1: {
      Mat unf(R, J * K);
      for (Index k = 0; k < K; ++k) {
        const Mat d = Y.dense(k);
        for (Index j = 0; j < J; ++j)
          for (Index r = 0; r < R; ++r) unf(r, k * J + j) = d(r, j);
      }
      return matmul(unf, khatri_rao(W, V));
    }
    case 2: {
      Mat unf(J, R * K);
      for (Index k = 0; k < K; ++k) {
        const Mat d = Y.dense(k);
        for (Index r = 0; r < R; ++r)
          for (Index j = 0; j < J; ++j) unf(j, k * R + r) = d(r, j);
      }
      return matmul(unf, khatri_rao(W, H));
    }
    default: {
      Mat unf(K, R * J);
      for (Index k = 0; k < K; ++k) {
        const Mat d = Y.dense(k);
        for (Index i = 0; i < R * J; ++i) unf(k, i) = d.data()[i];
      }
      return matmul(unf, khatri_rao(V, H));
    }
  }
}

/// mttkrp.hpp:241-253
inline std::uint64_t naive_mttkrp_bytes(Index K, Index J, Index R, int mode) {
  const auto k = static_cast<std::uint64_t>(K), j = static_cast<std::uint64_t>(J), r = static_cast<std::uint64_t>(R);
  std::uint64_t unf = 0, krp = 0, res = 0;
  switch (mode) {
    case 1: unf = r * j * k; krp = k * j * r; res = r * r; break;
    case 2: unf = j * r * k; krp = k * r * r; res = j * r; break;
    case 3: unf = k * r * j; krp = j * r * r; res = k * r; break;
    default: throw std::invalid_argument("mttkrp: mode must be 1, 2 or 3");
  }
  return 8 * (unf + krp + res);
}

// ---------------------------------------------------------------------------
// CP-ALS step — cp.hpp:34-145.
// ---------------------------------------------------------------------------
struct CpFactors {
  Mat H, V, W;
  Vec lambda;
};
struct CpOptions {
  bool nonneg = true;
  bool normalize_w = false;
  int threads = 1;
};

namespace detail {
/// cp.hpp:49-57
inline void check_cp_shapes(const ProjectedSlices& Y, const CpFactors& f) {
  const Index R = Y.rank();
  if (f.H.rows() != R || f.H.cols() != R) throw std::invalid_argument("cp factors: H must be R x R");
  if (f.V.rows() != Y.n_cols() || f.V.cols() != R) throw std::invalid_argument("cp factors: V must be J x R");
  if (f.W.rows() != Y.n_slices() || f.W.cols() != R) throw std::invalid_argument("cp factors: W must be K x R");
}
/// cp.hpp:62-70 — unit columns of A, norms absorbed into B; zero columns skipped.
inline Vec normalize_columns_into(Mat& A, Mat& B) {
  Vec norms(static_cast<std::size_t>(A.cols()), 1.0);
  for (Index r = 0; r < A.cols(); ++r) {
    double s = 0.0;
    for (Index i = 0; i < A.rows(); ++i) s += A(i, r) * A(i, r);
    const double nrm = std::sqrt(s);
    if (nrm > 0.0) {
      for (Index i = 0; i < A.rows(); ++i) A(i, r) /= nrm;
      for (Index i = 0; i < B.rows(); ++i) B(i, r) *= nrm;
      norms[static_cast<std::size_t>(r)] = nrm;
    }
  }
  return norms;
}
}  // namespace detail

/// cp.hpp:78-90
inline double cp_objective(const ProjectedSlices& Y, const CpFactors& f, int threads = 1) {
  detail::check_cp_shapes(Y, f);
  if (static_cast<Index>(f.lambda.size()) != Y.rank()) throw std::invalid_argument("cp factors: lambda must have length R");
  Mat sw = f.W;
  for (Index r = 0; r < sw.cols(); ++r)
    for (Index k = 0; k < sw.rows(); ++k) sw(k, r) *= f.lambda[static_cast<std::size_t>(r)];
  const Mat m3 = mttkrp_mode3(Y, f.H, f.V, threads);
  const Mat C = hadamard(gram(f.H), gram(f.V));
  double cross = 0.0;
  for (Index i = 0; i < sw.size(); ++i) cross += sw.data()[i] * m3.data()[i];
  const Mat swC = matmul(sw, C);
  double model = 0.0;
  for (Index i = 0; i < sw.size(); ++i) model += swC.data()[i] * sw.data()[i];
  return Y.frobenius_sq() - 2.0 * cross + model;
}

/// Per-step intermediates of one CP-ALS iteration (parity dumps).
struct CpStepDump {
  Mat m1, m2, m3;
  Vec norm_h, norm_v;
};

inline double ms_since(std::chrono::steady_clock::time_point t0);

/// cp.hpp:99-145 — H, V, W in fixed order.
/// (Oracle-only diagnostic `ms_v_update`: wall time of the V solve, the
/// step whose cost scales with J rather than with the number of subjects;
/// bench.py uses it to extrapolate a subject-prefix sample to the full
/// workload.)
inline CpFactors cp_als_iteration(const ProjectedSlices& Y, CpFactors f, const CpOptions& opts = {},
                                  Mat* mode3_out = nullptr, CpStepDump* dump = nullptr,
                                  double* ms_v_update = nullptr) {
  detail::check_cp_shapes(Y, f);
  const Index R = Y.rank();
  {
    const Mat m1 = mttkrp_mode1(Y, f.V, f.W, opts.threads);
    const Mat G = hadamard(gram(f.W), gram(f.V));
    f.H = matmul(m1, pinv_small(G));
    const Vec nh = detail::normalize_columns_into(f.H, f.W);
    if (dump) {
      dump->m1 = m1;
      dump->norm_h = nh;
    }
  }
  {
    const Mat m2 = mttkrp_mode2(Y, f.H, f.W, opts.threads);
    const Mat G = hadamard(gram(f.W), gram(f.H));
    const auto tv = std::chrono::steady_clock::now();
    f.V = opts.nonneg ? nnls_rowwise(G, m2, opts.threads) : matmul(m2, pinv_small(G));
    if (ms_v_update) *ms_v_update = ms_since(tv);
    const Vec nv = detail::normalize_columns_into(f.V, f.W);
    if (dump) {
      dump->m2 = m2;
      dump->norm_v = nv;
    }
  }
  {
    const Mat m3 = mttkrp_mode3(Y, f.H, f.V, opts.threads);
    const Mat G = hadamard(gram(f.V), gram(f.H));
    f.W = opts.nonneg ? nnls_rowwise(G, m3, opts.threads) : matmul(m3, pinv_small(G));
    if (mode3_out) *mode3_out = m3;
    if (dump) dump->m3 = m3;
  }
  f.lambda.assign(static_cast<std::size_t>(R), 1.0);
  if (opts.normalize_w) {
    for (Index r = 0; r < R; ++r) {
      double s = 0.0;
      for (Index k = 0; k < f.W.rows(); ++k) s += f.W(k, r) * f.W(k, r);
      const double nrm = std::sqrt(s);
      f.lambda[static_cast<std::size_t>(r)] = nrm;
      if (nrm > 0.0)
        for (Index k = 0; k < f.W.rows(); ++k) f.W(k, r) /= nrm;
    }
  }
  return f;
}

// ---------------------------------------------------------------------------
// PARAFAC2 solver — solver.hpp:48-321.
// ---------------------------------------------------------------------------
struct SolverConfig {
  enum class Init { random, eye };
  Index rank = 1;
  int max_iters = 200;
  double tol = 1e-8;
  bool nonneg = true;
  Init init = Init::random;
  std::uint64_t seed = 0;
  int threads = 1;
};

struct Parafac2Factors {
  std::vector<Mat> Q;
  Mat H, S, V;
  Index rank = 0;
};

struct IterationStats {
  int iter = 0;
  double residual_sq = 0;
  double fit = 0;
  double ms_procrustes = 0, ms_project = 0, ms_cp = 0;
  double ms_v_update = 0;  // oracle-only: the J-row V solve inside ms_cp
  // Oracle-only diagnostics: rank-deficient Procrustes targets (D5 rule).
  std::int64_t n_deficient = 0;
  std::int64_t n_degenerate = 0;
  double min_lambda_ratio = 1.0;  // min_k lambda_min/lambda_max of A_k^T A_k
};

struct FitTrace {
  std::vector<IterationStats> iterations;
  double total_ms = 0;
  bool converged = false;
};

using IterationObserver = std::function<void(const Parafac2Factors&, const IterationStats&)>;

inline double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

/// solver.hpp:104-166 — validation, H = I, S = ones, V random (r-outer,
/// j-inner) or |leading eigenvectors| of sum_k X_k^T X_k.
inline Parafac2Factors initialize(const IrregularTensor& X, const SolverConfig& cfg) {
  const Index R = cfg.rank;
  if (R < 1) throw std::invalid_argument("rank must be at least 1");
  if (!(cfg.tol > 0.0)) throw std::invalid_argument("convergence tolerance must be positive");
  if (cfg.max_iters < 1) throw std::invalid_argument("iteration limit must be at least 1");
  if (X.n_cols() < R)
    throw DataError("rank exceeds variables: J = " + std::to_string(X.n_cols()) + " < rank " + std::to_string(R));
  for (Index k = 0; k < X.n_slices(); ++k)
    if (X.slice(k).n_rows() < R)
      throw DataError("rank exceeds observations for subject " + std::to_string(k) + ": I_k = " +
                      std::to_string(X.slice(k).n_rows()) + " < rank " + std::to_string(R));
  Parafac2Factors f;
  f.rank = R;
  f.H = Mat::identity(R, R);
  f.S = Mat::ones(X.n_slices(), R);
  if (cfg.init == SolverConfig::Init::random) {
    Rng rng(cfg.seed);
    f.V = Mat(X.n_cols(), R);
    for (Index r = 0; r < R; ++r)
      for (Index j = 0; j < X.n_cols(); ++j) f.V(j, r) = rng.uniform();
  } else {
    const Index J = X.n_cols();
    Mat C(J, J);
    for (Index k = 0; k < X.n_slices(); ++k) {
      const SparseSlice& s = X.slice(k);
      for (Index a = 0; a < s.n_nnz_cols(); ++a) {
        auto [a0, a1] = s.col_range(a);
        for (Index b = a; b < s.n_nnz_cols(); ++b) {
          auto [b0, b1] = s.col_range(b);
          double dot = 0.0;
          for (Index p = a0, q = b0; p < a1 && q < b1;) {
            if (s.entry_row(p) == s.entry_row(q)) {
              dot += s.entry_value(p) * s.entry_value(q);
              ++p, ++q;
            } else if (s.entry_row(p) < s.entry_row(q)) {
              ++p;
            } else {
              ++q;
            }
          }
          C(s.col(a), s.col(b)) += dot;
          if (a != b) C(s.col(b), s.col(a)) += dot;
        }
      }
    }
    const SymEig e = sym_eig(C);
    f.V = Mat(J, R);
    for (Index r = 0; r < R; ++r)
      for (Index j = 0; j < J; ++j) f.V(j, r) = std::abs(e.vectors(j, J - 1 - r));
  }
  return f;
}

// Canonical Procrustes rule D5.
//
// The reference returns Q_k = Z P^T from Eigen's JacobiSVD of
// M = H diag(s) (X_k V)^T (solver.hpp:189-192), i.e. the polar factor of
// A = M^T = X_k V diag(s) H^T.  For rank(A) = R that factor is unique and
// this function returns it (one-sided Jacobi SVD, backward stable like
// JacobiSVD).  For rank(A) = rho < R the reference's completion is whatever
// Eigen produces (unpinned); both this oracle and the GPU use:
//   * eigen-directions of A^T A with lambda_i <= kNullRatio * lambda_max are
//     null (E_perp); the rest give U_rho = A E_rho Lambda_rho^{-1/2};
//   * N = (I - U_rho U_rho^T) L E_perp with L = I(I_k, R) (the identity
//     block the reference itself uses for M == 0, kernels.hpp:101-104);
//   * Q = U_rho E_rho^T + polar(N) E_perp^T.
// Q is column-orthonormal, independent of the basis chosen for E_perp, and
// reduces to the reference exactly when M == 0 (Q = I(I_k, R)).
// On lambda = sigma^2: a direction is null only at round-off level
// (sigma <= 1e-13 sigma_max), so genuinely small singular values are kept
// exactly as Eigen's JacobiSVD keeps them (kernels.hpp:105).
constexpr double kNullRatio = 1e-26;

enum ProcrustesFlag : int { kFullRank = 0, kDeficient = 1, kDegenerate = 3 };

struct PolarInfo {
  int flag = kFullRank;
  int rho = 0;
  double lambda_ratio = 1.0;  // lambda_min / lambda_max of A^T A (1 if A==0)
};

inline Mat canonical_polar(const Mat& A, PolarInfo* info = nullptr) {
  const Index m = A.rows(), R = A.cols();
  PolarInfo pi;
  if (A.is_zero()) {
    pi.flag = kDeficient;
    pi.rho = 0;
    if (info) *info = pi;
    return Mat::identity(m, R);
  }
  const Svd s = one_sided_jacobi(A);
  const double smax = s.sigma[0];
  Index rho = 0;
  while (rho < R && s.sigma[static_cast<std::size_t>(rho)] * s.sigma[static_cast<std::size_t>(rho)] >
                        kNullRatio * smax * smax)
    ++rho;
  pi.rho = static_cast<int>(rho);
  const double smin = s.sigma[static_cast<std::size_t>(R - 1)];
  pi.lambda_ratio = (smin * smin) / (smax * smax);
  Mat Q(m, R);
  for (Index c = 0; c < rho; ++c)
    for (Index j = 0; j < R; ++j) {
      const double v = s.V(j, c);
      for (Index i = 0; i < m; ++i) Q(i, j) += s.U(i, c) * v;
    }
  if (rho < R) {
    pi.flag = kDeficient;
    const Index nn = R - rho;
    // N = L E_perp - U_rho (U_rho^T L E_perp); L E_perp = E_perp in rows 0..R-1.
    Mat N(m, nn);
    for (Index c = 0; c < nn; ++c)
      for (Index i = 0; i < R; ++i) N(i, c) = s.V(i, rho + c);
    for (Index c = 0; c < nn; ++c)
      for (Index a = 0; a < rho; ++a) {
        double d = 0.0;
        for (Index i = 0; i < R; ++i) d += s.U(i, a) * s.V(i, rho + c);
        for (Index i = 0; i < m; ++i) N(i, c) -= d * s.U(i, a);
      }
    const Svd sn = one_sided_jacobi(N);
    const double nmin = sn.sigma[static_cast<std::size_t>(nn - 1)];
    if (!(nmin * nmin > 1e-8)) pi.flag = kDegenerate;
    // polar(N) = U_N V_N^T ; Q += polar(N) E_perp^T
    Mat PN(m, nn);
    for (Index c = 0; c < nn; ++c)
      for (Index b = 0; b < nn; ++b) {
        const double v = sn.V(c, b);
        for (Index i = 0; i < m; ++i) PN(i, c) += sn.U(i, b) * v;
      }
    for (Index c = 0; c < nn; ++c)
      for (Index j = 0; j < R; ++j) {
        const double e = s.V(j, rho + c);
        for (Index i = 0; i < m; ++i) Q(i, j) += PN(i, c) * e;
      }
  }
  if (info) *info = pi;
  return Q;
}

/// X_k V (solver.hpp:182-188): CSC walk, column ascending, rows ascending.
inline Mat slice_times(const SparseSlice& Xk, const Mat& V) {
  const Index R = V.cols();
  Mat XV(Xk.n_rows(), R);
  for (Index c = 0; c < Xk.n_nnz_cols(); ++c) {
    const Index j = Xk.col(c);
    auto [p0, p1] = Xk.col_range(c);
    for (Index p = p0; p < p1; ++p) {
      const Index i = Xk.entry_row(p);
      const double v = Xk.entry_value(p);
      for (Index r = 0; r < R; ++r) XV(i, r) += v * V(j, r);
    }
  }
  return XV;
}

/// solver.hpp:173-193 (SVD replaced by the canonical polar rule above).
inline Mat procrustes_update(const SparseSlice& Xk, const Mat& H, const Vec& s, const Mat& V,
                             PolarInfo* info = nullptr) {
  const Index R = H.rows();
  if (H.cols() != R) throw std::invalid_argument("H must be square");
  if (static_cast<Index>(s.size()) != R || V.cols() != R || V.rows() != Xk.n_cols())
    throw std::invalid_argument("procrustes factors have mismatched shapes");
  if (Xk.n_rows() < R) throw std::invalid_argument("rank exceeds observations in procrustes step");
  const Mat XV = slice_times(Xk, V);
  // M = (H diag(s)) XV^T ; A = M^T = XV diag(s) H^T  (I_k x R)
  Mat A(Xk.n_rows(), R);
  for (Index a = 0; a < R; ++a)
    for (Index r = 0; r < R; ++r) {
      const double hs = H(a, r) * s[static_cast<std::size_t>(r)];
      if (hs == 0.0) continue;
      for (Index i = 0; i < Xk.n_rows(); ++i) A(i, a) += XV(i, r) * hs;
    }
  ensure_finite(A, "svd operand");
  return canonical_polar(A, info);
}

/// solver.hpp:197-208
inline Mat project_slice(const SparseSlice& Xk, const Mat& Qk) {
  if (Qk.rows() != Xk.n_rows()) throw std::invalid_argument("projection: Q_k row count mismatch");
  Mat packed(Qk.cols(), Xk.n_nnz_cols());
  for (Index c = 0; c < Xk.n_nnz_cols(); ++c) {
    auto [p0, p1] = Xk.col_range(c);
    for (Index p = p0; p < p1; ++p) {
      const double v = Xk.entry_value(p);
      const Index i = Xk.entry_row(p);
      for (Index r = 0; r < Qk.cols(); ++r) packed(r, c) += v * Qk(i, r);
    }
  }
  return packed;
}

/// solver.hpp:212-235
inline ProjectedSlices project_slices(const IrregularTensor& X, const std::vector<Mat>& Q, int threads = 1) {
  if (static_cast<Index>(Q.size()) != X.n_slices()) throw std::invalid_argument("projection: one Q_k per slice required");
  const Index K = X.n_slices();
  const Index R = Q.empty() ? 0 : Q.front().cols();
  std::vector<Mat> packed(static_cast<std::size_t>(K));
  std::vector<std::vector<Index>> cols(static_cast<std::size_t>(K));
  std::vector<std::uint64_t> w(static_cast<std::size_t>(K));
  for (Index k = 0; k < K; ++k) w[static_cast<std::size_t>(k)] = static_cast<std::uint64_t>(X.slice(k).nnz());
  run_chunks(partition_weighted(w, threads), [&](std::size_t, Index b, Index e) {
    for (Index k = b; k < e; ++k) {
      packed[static_cast<std::size_t>(k)] = project_slice(X.slice(k), Q[static_cast<std::size_t>(k)]);
      cols[static_cast<std::size_t>(k)] = X.slice(k).nnz_cols();
    }
  });
  return ProjectedSlices::from_packed(R, X.n_cols(), std::move(packed), std::move(cols));
}

/// solver.hpp:238-243
inline std::vector<Mat> assemble_U(const Parafac2Factors& f) {
  std::vector<Mat> U;
  for (const Mat& Qk : f.Q) U.push_back(matmul(Qk, f.H));
  return U;
}

/// Optional explicit starting factors: the reference has no
/// such entry point (solver.hpp:251-253); BASELINE configs need it.
struct InitialFactors {
  Mat H, V, W;
};

/// Per-iteration state dumps for teacher-forced parity gates.
struct IterationDump {
  Mat H_in, V_in, W_in;  // factors entering the iteration
  std::vector<Mat> Q;
  std::vector<int> flags;
  CpStepDump cp;
  Mat H, V, W;  // factors leaving the iteration
  double fit = 0, residual_sq = 0;
};

/// solver.hpp:251-321 — the full PARAFAC2-ALS loop.
inline std::pair<Parafac2Factors, FitTrace> fit_parafac2(const IrregularTensor& X, const SolverConfig& cfg,
                                                         const IterationObserver& observer = nullptr,
                                                         const InitialFactors* init = nullptr,
                                                         std::vector<IterationDump>* dumps = nullptr) {
  const auto t_start = std::chrono::steady_clock::now();
  Parafac2Factors state = initialize(X, cfg);
  const Index K = X.n_slices();
  const Index R = cfg.rank;
  if (init) {
    if (init->H.rows() != R || init->H.cols() != R || init->V.rows() != X.n_cols() || init->V.cols() != R ||
        init->W.rows() != K || init->W.cols() != R)
      throw std::invalid_argument("initial factors have mismatched shapes");
    state.H = init->H;
    state.V = init->V;
    state.S = init->W;
  }
  const double norm_x = frobenius_sq(X);
  if (!(norm_x > 0.0)) throw DataError("tensor has no non-zero entries");
  state.Q.assign(static_cast<std::size_t>(K), Mat());
  std::vector<std::uint64_t> weights(static_cast<std::size_t>(K));
  for (Index k = 0; k < K; ++k)
    weights[static_cast<std::size_t>(k)] =
        static_cast<std::uint64_t>(X.slice(k).nnz()) + static_cast<std::uint64_t>(X.slice(k).n_rows());
  CpFactors cp{state.H, state.V, state.S, Vec(static_cast<std::size_t>(R), 1.0)};
  CpOptions opts{cfg.nonneg, false, cfg.threads};
  FitTrace trace;
  double prev_fit = 0.0;
  std::vector<PolarInfo> infos(static_cast<std::size_t>(K));
  for (int iter = 1; iter <= cfg.max_iters; ++iter) {
    IterationStats st;
    st.iter = iter;
    IterationDump dump;
    if (dumps) {
      dump.H_in = cp.H;
      dump.V_in = cp.V;
      dump.W_in = cp.W;
    }
    auto t0 = std::chrono::steady_clock::now();
    run_chunks(partition_weighted(weights, cfg.threads), [&](std::size_t, Index b, Index e) {
      Vec s(static_cast<std::size_t>(R));
      for (Index k = b; k < e; ++k) {
        for (Index r = 0; r < R; ++r) s[static_cast<std::size_t>(r)] = cp.W(k, r);
        state.Q[static_cast<std::size_t>(k)] =
            procrustes_update(X.slice(k), cp.H, s, cp.V, &infos[static_cast<std::size_t>(k)]);
      }
    });
    st.ms_procrustes = ms_since(t0);
    for (const PolarInfo& pi : infos) {
      st.n_deficient += pi.flag != kFullRank;
      st.n_degenerate += pi.flag == kDegenerate;
      st.min_lambda_ratio = std::min(st.min_lambda_ratio, pi.lambda_ratio);
    }
    t0 = std::chrono::steady_clock::now();
    const ProjectedSlices Y = project_slices(X, state.Q, cfg.threads);
    st.ms_project = ms_since(t0);
    t0 = std::chrono::steady_clock::now();
    Mat m3;
    cp = cp_als_iteration(Y, std::move(cp), opts, &m3, dumps ? &dump.cp : nullptr, &st.ms_v_update);
    state.H = cp.H;
    state.V = cp.V;
    state.S = cp.W;
    st.ms_cp = ms_since(t0);
    double cross = 0.0;
    for (Index i = 0; i < cp.W.size(); ++i) cross += cp.W.data()[i] * m3.data()[i];
    const Mat C = hadamard(gram(cp.H), gram(cp.V));
    const Mat WC = matmul(cp.W, C);
    double model = 0.0;
    for (Index i = 0; i < cp.W.size(); ++i) model += WC.data()[i] * cp.W.data()[i];
    st.residual_sq = std::max(0.0, norm_x - 2.0 * cross + model);
    st.fit = 1.0 - st.residual_sq / norm_x;
    if (!std::isfinite(st.fit) || !std::isfinite(st.residual_sq))
      throw NumericalError("numerical divergence at iteration " + std::to_string(iter));
    trace.iterations.push_back(st);
    if (dumps) {
      dump.Q = state.Q;
      dump.flags.resize(static_cast<std::size_t>(K));
      for (Index k = 0; k < K; ++k) dump.flags[static_cast<std::size_t>(k)] = infos[static_cast<std::size_t>(k)].flag;
      dump.H = cp.H;
      dump.V = cp.V;
      dump.W = cp.W;
      dump.fit = st.fit;
      dump.residual_sq = st.residual_sq;
      dumps->push_back(std::move(dump));
    }
    if (observer) observer(state, st);
    const double change = std::abs(st.fit - prev_fit) / std::max(prev_fit, std::numeric_limits<double>::epsilon());
    prev_fit = st.fit;
    if (change < cfg.tol) {
      trace.converged = true;
      break;
    }
  }
  trace.total_ms = ms_since(t_start);
  return {std::move(state), std::move(trace)};
}

// ---------------------------------------------------------------------------
// Generator pieces — generator.hpp:36-162 (reference test inputs).
// ---------------------------------------------------------------------------

/// generator.hpp:36-47 — Householder QR of a Gaussian matrix, sign-fixed so
/// diag(R) >= 0.
inline Mat random_orthonormal(Rng& rng, Index rows, Index cols) {
  if (rows < cols) throw std::invalid_argument("orthonormal factor needs rows >= cols");
  Mat A(rows, cols);
  for (Index c = 0; c < cols; ++c)
    for (Index r = 0; r < rows; ++r) A(r, c) = rng.normal();
  // Householder QR (LAPACK dgeqrf convention: v(0)=1, beta = -sign(alpha)*norm).
  std::vector<Vec> vs;
  Vec taus;
  Vec rdiag(static_cast<std::size_t>(cols));
  for (Index c = 0; c < cols; ++c) {
    double sig = 0.0;
    for (Index r = c + 1; r < rows; ++r) sig += A(r, c) * A(r, c);
    const double alpha = A(c, c);
    Vec v(static_cast<std::size_t>(rows), 0.0);
    double tau = 0.0, beta = alpha;
    if (sig != 0.0) {
      beta = -std::copysign(std::sqrt(alpha * alpha + sig), alpha);
      tau = (beta - alpha) / beta;
      const double inv = 1.0 / (alpha - beta);
      v[static_cast<std::size_t>(c)] = 1.0;
      for (Index r = c + 1; r < rows; ++r) v[static_cast<std::size_t>(r)] = A(r, c) * inv;
      // apply H = I - tau v v^T to remaining columns
      for (Index j = c + 1; j < cols; ++j) {
        double d = A(c, j);
        for (Index r = c + 1; r < rows; ++r) d += v[static_cast<std::size_t>(r)] * A(r, j);
        d *= tau;
        A(c, j) -= d;
        for (Index r = c + 1; r < rows; ++r) A(r, j) -= d * v[static_cast<std::size_t>(r)];
      }
    } else {
      v[static_cast<std::size_t>(c)] = 1.0;
    }
    A(c, c) = beta;
    rdiag[static_cast<std::size_t>(c)] = beta;
    vs.push_back(std::move(v));
    taus.push_back(tau);
  }
  Mat Q = Mat::identity(rows, cols);
  for (Index c = cols - 1; c >= 0; --c) {
    const Vec& v = vs[static_cast<std::size_t>(c)];
    const double tau = taus[static_cast<std::size_t>(c)];
    if (tau == 0.0) continue;
    for (Index j = 0; j < cols; ++j) {
      double d = 0.0;
      for (Index r = c; r < rows; ++r) d += v[static_cast<std::size_t>(r)] * Q(r, j);
      d *= tau;
      for (Index r = c; r < rows; ++r) Q(r, j) -= d * v[static_cast<std::size_t>(r)];
    }
  }
  for (Index c = 0; c < cols; ++c)
    if (rdiag[static_cast<std::size_t>(c)] < 0.0)
      for (Index r = 0; r < rows; ++r) Q(r, c) = -Q(r, c);
  return Q;
}

/// generator.hpp:50-56
inline Mat random_uniform(Rng& rng, Index rows, Index cols, double lo, double hi) {
  Mat A(rows, cols);
  for (Index c = 0; c < cols; ++c)
    for (Index r = 0; r < rows; ++r) A(r, c) = rng.uniform(lo, hi);
  return A;
}

struct GeneratorSpec {
  Index subjects = 1, cols = 1, max_rows = 1, rank = 1;
  double density = 1.0;
  std::uint64_t seed = 0;
  bool nonneg_factors = true;
};

struct GeneratedTensor {
  IrregularTensor tensor;
  Index dropped_subjects = 0;
};

/// generator.hpp:89-162 — planted rank-R model with geometric-gap
/// sparsification and zero-row filtering.
inline GeneratedTensor generate_synthetic(const GeneratorSpec& spec) {
  if (spec.subjects < 1) throw std::invalid_argument("generator: subjects must be at least 1");
  if (spec.cols < 1) throw std::invalid_argument("generator: cols must be at least 1");
  if (spec.max_rows < 1) throw std::invalid_argument("generator: max_rows must be at least 1");
  if (spec.rank < 1 || spec.rank > std::min(spec.max_rows, spec.cols))
    throw std::invalid_argument("generator: rank must satisfy 1 <= rank <= min(max_rows, cols)");
  if (!(spec.density > 0.0) || spec.density > 1.0) throw std::invalid_argument("generator: density must be in (0, 1]");
  const Index K = spec.subjects, J = spec.cols, I = spec.max_rows, R = spec.rank;
  const double lo = spec.nonneg_factors ? 0.0 : -1.0;
  Rng master(spec.seed);
  const Mat H = random_uniform(master, R, R, lo, 1.0);
  const Mat V = random_uniform(master, J, R, lo, 1.0);
  const Mat S = random_uniform(master, K, R, lo, 1.0);
  GeneratedTensor out;
  std::vector<SparseSlice> slices;
  std::vector<Triplet> kept;
  for (Index k = 0; k < K; ++k) {
    Rng rk(substream_seed(spec.seed, static_cast<std::uint64_t>(k) + 1));
    const Mat Q = random_orthonormal(rk, I, R);
    Mat HS(R, R);
    for (Index c = 0; c < R; ++c)
      for (Index r = 0; r < R; ++r) HS(r, c) = H(r, c) * S(k, c);
    const Mat A = matmul(Q, HS);
    auto value = [&](Index i, Index j) {
      double acc = 0.0;
      for (Index r = 0; r < R; ++r) acc += A(i, r) * V(j, r);
      return acc;
    };
    kept.clear();
    const std::uint64_t total = static_cast<std::uint64_t>(I) * static_cast<std::uint64_t>(J);
    if (spec.density >= 1.0) {
      for (Index i = 0; i < I; ++i)
        for (Index j = 0; j < J; ++j) kept.push_back({i, j, value(i, j)});
    } else {
      const double log_q = std::log1p(-spec.density);
      std::uint64_t pos = 0;
      while (true) {
        const double u = 1.0 - rk.uniform();
        const double gap = std::floor(std::log(u) / log_q);
        if (gap >= static_cast<double>(total)) break;
        pos += static_cast<std::uint64_t>(gap);
        if (pos >= total) break;
        const Index i = static_cast<Index>(pos / static_cast<std::uint64_t>(J));
        const Index j = static_cast<Index>(pos % static_cast<std::uint64_t>(J));
        kept.push_back({i, j, value(i, j)});
        ++pos;
      }
    }
    if (kept.empty()) {
      ++out.dropped_subjects;
      continue;
    }
    SparseSlice full = SparseSlice::from_triplets(I, J, kept);
    if (full.nnz() == 0) {
      ++out.dropped_subjects;
      continue;
    }
    slices.push_back(filter_zero_rows(full).first);
  }
  if (slices.empty()) throw DataError("generator: every subject sparsified to empty");
  out.tensor = IrregularTensor::from_slices(J, std::move(slices));
  return out;
}

// ---------------------------------------------------------------------------
// Test fixtures — tests/support/helpers.hpp:52-141 (seeded instance builders
// and dense evaluation oracles), restated so the reference's property tests
// can be re-run on bit-identical inputs.
// ---------------------------------------------------------------------------
namespace fixtures {

inline double rel_frob(const Mat& a, const Mat& ref) {
  double d = 0.0;
  for (Index i = 0; i < a.size(); ++i) {
    const double x = a.data()[i] - ref.data()[i];
    d += x * x;
  }
  return std::sqrt(d) / std::max(1.0, ref.norm());
}

/// helpers.hpp:52-58
inline Mat random_matrix(Rng& rng, Index rows, Index cols, double lo = -1.0, double hi = 1.0) {
  Mat m(rows, cols);
  for (Index c = 0; c < cols; ++c)
    for (Index r = 0; r < rows; ++r) m(r, c) = rng.uniform(lo, hi);
  return m;
}

/// helpers.hpp:62-76
inline SparseSlice random_slice(Rng& rng, Index rows, Index cols, double density, double lo = -1.0, double hi = 1.0) {
  std::vector<Triplet> e;
  for (Index i = 0; i < rows; ++i)
    for (Index j = 0; j < cols; ++j)
      if (rng.uniform() < density) e.push_back({i, j, rng.uniform(lo, hi)});
  if (e.empty()) {
    const Index i = static_cast<Index>(rng.below(static_cast<std::uint64_t>(rows)));
    const Index j = static_cast<Index>(rng.below(static_cast<std::uint64_t>(cols)));
    e.push_back({i, j, rng.uniform(0.5, 1.5)});
  }
  return SparseSlice::from_triplets(rows, cols, e);
}

/// helpers.hpp:78-93
inline IrregularTensor random_tensor(Rng& rng, Index n_slices, Index n_cols, Index min_rows, Index max_rows,
                                     double density, double lo = -1.0, double hi = 1.0) {
  std::vector<SparseSlice> slices;
  for (Index k = 0; k < n_slices; ++k) {
    Index rows = min_rows;
    if (max_rows > min_rows) rows += static_cast<Index>(rng.below(static_cast<std::uint64_t>(max_rows - min_rows + 1)));
    slices.push_back(random_slice(rng, rows, n_cols, density, lo, hi));
  }
  return IrregularTensor::from_slices(n_cols, std::move(slices));
}

/// helpers.hpp:97-115
inline ProjectedSlices random_projected(Rng& rng, Index rank, Index n_cols, Index n_slices, double density,
                                        double lo = -1.0, double hi = 1.0) {
  std::vector<Mat> packed;
  std::vector<std::vector<Index>> cols;
  for (Index k = 0; k < n_slices; ++k) {
    std::vector<Index> c;
    for (Index j = 0; j < n_cols; ++j)
      if (rng.uniform() < density) c.push_back(j);
    if (c.empty()) c.push_back(static_cast<Index>(rng.below(static_cast<std::uint64_t>(n_cols))));
    packed.push_back(random_matrix(rng, rank, static_cast<Index>(c.size()), lo, hi));
    cols.push_back(std::move(c));
  }
  return ProjectedSlices::from_packed(rank, n_cols, std::move(packed), std::move(cols));
}

/// helpers.hpp:119-128
inline double dense_cp_objective(const ProjectedSlices& y, const CpFactors& f) {
  double total = 0.0;
  for (Index k = 0; k < y.n_slices(); ++k) {
    Mat HW(f.H.rows(), f.H.cols());
    for (Index c = 0; c < f.H.cols(); ++c)
      for (Index r = 0; r < f.H.rows(); ++r) HW(r, c) = f.H(r, c) * f.W(k, c) * f.lambda[static_cast<std::size_t>(c)];
    const Mat model = matmul(HW, f.V.transpose());
    const Mat d = y.dense(k);
    for (Index i = 0; i < d.size(); ++i) {
      const double x = d.data()[i] - model.data()[i];
      total += x * x;
    }
  }
  return total;
}

/// helpers.hpp:132-141
inline double dense_residual(const IrregularTensor& x, const Parafac2Factors& f) {
  double total = 0.0;
  for (Index k = 0; k < x.n_slices(); ++k) {
    const Mat QH = matmul(f.Q[static_cast<std::size_t>(k)], f.H);
    Mat QHS = QH;
    for (Index c = 0; c < QH.cols(); ++c)
      for (Index r = 0; r < QH.rows(); ++r) QHS(r, c) *= f.S(k, c);
    const Mat model = matmul(QHS, f.V.transpose());
    const Mat d = x.slice(k).dense();
    for (Index i = 0; i < d.size(); ++i) {
      const double e = d.data()[i] - model.data()[i];
      total += e * e;
    }
  }
  return total;
}

}  // namespace fixtures

}  // namespace p2o
