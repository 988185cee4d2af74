// Drop-in replacement for /root/reference/proj/include/parafac2/io.hpp on top
// of the libp2g C ABI (include/p2g.h, ingest/export section).  Same names,
// formats, messages and exception types.  Parsing runs in libp2g on all host
// threads; writers produce the reference's canonical bytes.
//
// Difference: write_factors takes the metadata as a JSON text string
// (nlohmann::json is not a dependency), embedded verbatim as "config".
#pragma once

#include <cstdio>
#include <fstream>
#include <istream>
#include <iterator>
#include <ostream>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include "common.hpp"
#include "solver.hpp"
#include "sparse.hpp"

namespace parafac2 {

/// io.hpp:55-60: 17 significant digits, round-trips a double exactly.
inline std::string format_value(double v) {
  char buf[32];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

struct ParsedTensor {
  IrregularTensor tensor;
  Index filtered_rows = 0;  // all-zero rows removed across all subjects
};

namespace detail {

/// Owned p2g_csr -> IrregularTensor (per-subject CSC via from_triplets).
inline ParsedTensor take_parsed(p2g_csr* h) {
  struct Free {
    p2g_csr* h;
    ~Free() { p2g_csr_free(h); }
  } guard{h};
  int64_t K = 0, J = 0, NR = 0, nnz = 0, filtered = 0;
  check(p2g_csr_info(h, &K, &J, &NR, &nnz, &filtered));
  std::vector<int64_t> srp(static_cast<std::size_t>(K + 1)), rp(static_cast<std::size_t>(NR + 1));
  std::vector<int32_t> ci(static_cast<std::size_t>(nnz));
  std::vector<double> val(static_cast<std::size_t>(nnz));
  check(p2g_csr_copy(h, srp.data(), rp.data(), ci.data(), val.data()));
  std::vector<SparseSlice> slices;
  slices.reserve(static_cast<std::size_t>(K));
  for (int64_t k = 0; k < K; ++k) {
    std::vector<Triplet> t;
    const int64_t r0 = srp[static_cast<std::size_t>(k)], r1 = srp[static_cast<std::size_t>(k + 1)];
    for (int64_t r = r0; r < r1; ++r)
      for (int64_t p = rp[static_cast<std::size_t>(r)]; p < rp[static_cast<std::size_t>(r + 1)]; ++p)
        t.push_back({static_cast<Index>(r - r0), ci[static_cast<std::size_t>(p)], val[static_cast<std::size_t>(p)]});
    slices.push_back(SparseSlice::from_triplets(static_cast<Index>(r1 - r0), static_cast<Index>(J), std::move(t)));
  }
  ParsedTensor out;
  out.tensor = IrregularTensor::from_slices(static_cast<Index>(J), std::move(slices));
  out.filtered_rows = static_cast<Index>(filtered);
  return out;
}

}  // namespace detail

/// io.hpp:100-171.
inline ParsedTensor parse_coordinate_stream(std::istream& in) {
  const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  p2g_csr* h = nullptr;
  check(p2g_coo_parse(text.data(), static_cast<int64_t>(text.size()), 0, &h));
  return detail::take_parsed(h);
}

/// io.hpp:173-177.
inline ParsedTensor parse_coordinate_file(const std::string& path) {
  p2g_csr* h = nullptr;
  check(p2g_coo_read(path.c_str(), 0, &h));
  return detail::take_parsed(h);
}

/// io.hpp:179-195: comment lines, "K J", entries by subject, column, row.
inline void write_coordinate_stream(std::ostream& out, const IrregularTensor& t,
                                    const std::vector<std::string>& comments = {}) {
  for (const std::string& c : comments) out << "# " << c << '\n';
  out << t.n_slices() << ' ' << t.n_cols() << '\n';
  for (Index k = 0; k < t.n_slices(); ++k)
    for (const Triplet& e : t.slice(k).triplets())  // CSC order: column, then row
      out << k << ' ' << e.row << ' ' << e.col << ' ' << format_value(e.value) << '\n';
}

inline void write_coordinate_file(const std::string& path, const IrregularTensor& t,
                                  const std::vector<std::string>& comments = {}) {
  std::ofstream out(path);
  if (!out) throw DataError("cannot open output file: " + path);
  write_coordinate_stream(out, t, comments);
  if (!out) throw DataError("failed writing output file: " + path);
}

/// io.hpp:206-216.
inline void write_matrix_stream(std::ostream& out, const Matrix& M, const std::string& title) {
  out << "# " << title << '\n' << M.rows() << ' ' << M.cols() << '\n';
  for (Index r = 0; r < M.rows(); ++r) {
    for (Index c = 0; c < M.cols(); ++c) {
      if (c) out << ' ';
      out << format_value(M(r, c));
    }
    out << '\n';
  }
}

/// io.hpp:218-254.
inline Matrix read_matrix_stream(std::istream& in) {
  const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  int64_t rows = 0, cols = 0;
  check(p2g_matrix_parse(text.data(), static_cast<int64_t>(text.size()), &rows, &cols, nullptr, 0));
  Matrix M(static_cast<Index>(rows), static_cast<Index>(cols));
  check(p2g_matrix_parse(text.data(), static_cast<int64_t>(text.size()), &rows, &cols, M.data(), rows * cols));
  return M;
}

inline Matrix read_matrix_file(const std::string& path) {
  int64_t rows = 0, cols = 0;
  check(p2g_matrix_read(path.c_str(), &rows, &cols, nullptr, 0));
  Matrix M(static_cast<Index>(rows), static_cast<Index>(cols));
  check(p2g_matrix_read(path.c_str(), &rows, &cols, M.data(), rows * cols));
  return M;
}

inline void write_matrix_file(const std::string& path, const Matrix& M, const std::string& title) {
  check(p2g_matrix_write(path.c_str(), M.rows(), M.cols(), M.data(), title.c_str()));
}

/// io.hpp:270-305: V.txt, S.txt, H.txt, U_<k>.txt (U_k = Q_k H), manifest.json.
inline void write_factors(const Parafac2Factors& f, const std::string& out_dir, const std::string& metadata_json = "{}") {
  const Index K = static_cast<Index>(f.Q.size()), R = f.rank;
  std::vector<int64_t> srp(static_cast<std::size_t>(K + 1), 0);
  for (Index k = 0; k < K; ++k) srp[static_cast<std::size_t>(k + 1)] = srp[static_cast<std::size_t>(k)] + f.Q[static_cast<std::size_t>(k)].rows();
  std::vector<double> q(static_cast<std::size_t>(srp.back() * R));  // packed row-major
  for (Index k = 0; k < K; ++k) {
    const Matrix& Qk = f.Q[static_cast<std::size_t>(k)];
    for (Index i = 0; i < Qk.rows(); ++i)
      for (Index c = 0; c < R; ++c) q[static_cast<std::size_t>((srp[static_cast<std::size_t>(k)] + i) * R + c)] = Qk(i, c);
  }
  check(p2g_write_factors(out_dir.c_str(), K, f.V.rows(), static_cast<int32_t>(R), srp.data(), f.H.data(), f.V.data(),
                          f.S.data(), q.data(), metadata_json.c_str()));
}

/// io.hpp:307-315: deterministic fields only.
inline void write_trace_tsv(std::ostream& out, const FitTrace& trace) {
  out << "iter\tresidual_sq\tfit\n";
  for (const IterationStats& s : trace.iterations)
    out << s.iter << '\t' << format_value(s.residual_sq) << '\t' << format_value(s.fit) << '\n';
}

/// io.hpp:317-333.
inline std::vector<std::pair<Index, double>> rank_components(const Matrix& S, Index subject, Index top_n) {
  if (subject < 0 || subject >= S.rows()) throw DataError("subject index out of range: " + std::to_string(subject));
  if (top_n < 0 || top_n > S.cols()) throw std::invalid_argument("top_n must be between 0 and the rank");
  std::vector<std::pair<Index, double>> order;
  for (Index r = 0; r < S.cols(); ++r) order.emplace_back(r, S(subject, r));
  std::stable_sort(order.begin(), order.end(), [](const auto& a, const auto& b) { return a.second > b.second; });
  order.resize(static_cast<std::size_t>(top_n));
  return order;
}

}  // namespace parafac2
