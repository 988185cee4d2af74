// Host-side ingest and export for the path:
// the coordinate text format, a binary CSR cache, matrix files, the factor
// directory and the trace, with the semantics of io.hpp (reference
// proj/include/parafac2/io.hpp:38-315) and the slice normalisation of
// sparse.hpp (SparseSlice::from_triplets :47-86, filter_zero_rows :155-172).
//
// The device path consumes a flattened CSR.  At the north-star sizes
// (500M entries) parsing text dominates the end-to-end time, so the parser
// splits the file at line boundaries over host threads; the first error in
// file order is reported with its exact line number, and subjects are then
// normalised in parallel.  Duplicates are summed in the order std::sort
// leaves equal (column, row) keys, as the reference does, so sums are
// bit-identical to the reference built with the same standard library.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "p2g_common.hpp"

struct p2g_csr {
  std::int64_t K = 0, J = 0, filtered_rows = 0;
  std::vector<std::int64_t> srp, rp;
  std::vector<std::int32_t> ci;
  std::vector<double> val;
};

namespace p2g {
namespace {

struct Entry {
  std::int64_t k, i, j;
  double v;
};

[[noreturn]] void parse_fail(const std::string& what, long long line_no) {
  throw DataError(what + " at line " + std::to_string(line_no));
}

/// Splits on blanks/tabs (io.hpp split_fields semantics); at most `cap` fields
/// are stored, the count is returned (so "too many fields" is detectable).
int split_fields(std::string_view line, std::string_view* out, int cap) {
  int n = 0;
  std::size_t i = 0;
  while (i < line.size()) {
    while (i < line.size() && (line[i] == ' ' || line[i] == '\t')) ++i;
    const std::size_t b = i;
    while (i < line.size() && line[i] != ' ' && line[i] != '\t') ++i;
    if (i > b) {
      if (n < cap) out[n] = line.substr(b, i - b);
      ++n;
    }
  }
  return n;
}

bool parse_int(std::string_view t, std::int64_t& v) {
  long long x = 0;
  const auto r = std::from_chars(t.data(), t.data() + t.size(), x);
  if (r.ec != std::errc() || r.ptr != t.data() + t.size()) return false;
  v = static_cast<std::int64_t>(x);
  return true;
}

bool parse_double(std::string_view t, double& v) {
  const auto r = std::from_chars(t.data(), t.data() + t.size(), v);
  return r.ec == std::errc() && r.ptr == t.data() + t.size();
}

/// One text line without its terminator ('\n', then a trailing '\r').
std::string_view line_at(const char* p, const char* end, const char** next) {
  const char* e = static_cast<const char*>(std::memchr(p, '\n', static_cast<std::size_t>(end - p)));
  const char* le = e ? e : end;
  *next = e ? e + 1 : end;
  std::string_view sv(p, static_cast<std::size_t>(le - p));
  if (!sv.empty() && sv.back() == '\r') sv.remove_suffix(1);
  return sv;
}

bool skip_line(std::string_view sv) {  // blank or comment
  const std::size_t f = sv.find_first_not_of(" \t");
  return f == std::string_view::npos || sv[f] == '#';
}

struct ChunkResult {
  std::vector<Entry> entries;
  long long lines = 0;       // lines in the chunk
  long long err_line = -1;   // local line of the first error (1-based), or -1
  std::string err_what;
};

void parse_chunk(const char* p, const char* end, std::int64_t K, std::int64_t J, ChunkResult& out) {
  long long ln = 0;
  while (p < end) {
    const char* next;
    const std::string_view sv = line_at(p, end, &next);
    p = next;
    ++ln;
    if (skip_line(sv)) continue;
    std::string_view f[4];
    const int nf = split_fields(sv, f, 4);
    std::int64_t k, i, j;
    double v;
    const char* what = nullptr;
    if (nf != 4 || !parse_int(f[0], k) || !parse_int(f[1], i) || !parse_int(f[2], j) || !parse_double(f[3], v))
      what = "malformed entry (expected 'k i j v')";
    else if (k < 0 || k >= K)
      what = "subject index out of range";
    else if (i < 0)
      what = "row index out of range";
    else if (j < 0 || j >= J)
      what = "column index out of range";
    else if (!std::isfinite(v))
      what = "non-finite value";
    if (what) {
      out.err_line = ln;
      out.err_what = what;
      break;
    }
    out.entries.push_back({k, i, j, v});
  }
  // count the remaining lines only when no error stopped the chunk
  out.lines = ln;
}

/// One subject: sort by (column, row) with std::sort and sum equal keys in
/// that order, drop zeros (from_triplets), drop all-zero rows (filter_zero_rows).
struct Slice {
  std::vector<std::int64_t> rows_kept;  // original row ids, ascending
  std::vector<Entry> entries;           // (col, row)-sorted, new row ids in .i
};

void normalise_subject(std::int64_t k, std::vector<Entry>& e, Slice& out) {
  if (e.empty()) throw DataError("subject " + std::to_string(k) + " has no entries (empty slices are rejected)");
  std::sort(e.begin(), e.end(), [](const Entry& a, const Entry& b) { return a.j != b.j ? a.j < b.j : a.i < b.i; });
  std::vector<Entry> s;
  s.reserve(e.size());
  for (std::size_t a = 0; a < e.size();) {
    std::size_t b = a + 1;
    double v = e[a].v;
    while (b < e.size() && e[b].j == e[a].j && e[b].i == e[a].i) v += e[b++].v;
    if (v != 0.0) s.push_back({k, e[a].i, e[a].j, v});
    a = b;
  }
  if (s.empty()) throw DataError("subject " + std::to_string(k) + " has no entries after summing duplicates");
  std::vector<std::int64_t>& rows = out.rows_kept;
  rows.reserve(s.size());
  for (const Entry& x : s) rows.push_back(x.i);
  std::sort(rows.begin(), rows.end());
  rows.erase(std::unique(rows.begin(), rows.end()), rows.end());
  for (Entry& x : s) x.i = std::lower_bound(rows.begin(), rows.end(), x.i) - rows.begin();
  out.entries = std::move(s);
}

int pick_threads(int threads, std::size_t work) {
  int t = threads > 0 ? threads : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  const std::size_t by_work = std::max<std::size_t>(1, work / (1u << 20));
  return static_cast<int>(std::max<std::size_t>(1, std::min<std::size_t>(static_cast<std::size_t>(t), by_work)));
}

template <typename Fn>
void run_parallel(int n, Fn&& fn) {
  std::vector<std::thread> ts;
  std::vector<std::exception_ptr> errs(static_cast<std::size_t>(n));
  for (int t = 0; t < n; ++t)
    ts.emplace_back([&, t] {
      try {
        fn(t);
      } catch (...) {
        errs[static_cast<std::size_t>(t)] = std::current_exception();
      }
    });
  for (auto& th : ts) th.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);  // lowest thread index = earliest subjects
}

std::unique_ptr<p2g_csr> parse_buffer(const char* data, std::size_t len, int threads) {
  const char* p = data;
  const char* end = data + len;
  long long ln = 0;
  std::int64_t K = 0, J = 0;
  bool header = false;
  while (p < end && !header) {  // header: the first data line
    const char* next;
    const std::string_view sv = line_at(p, end, &next);
    p = next;
    ++ln;
    if (skip_line(sv)) continue;
    std::string_view f[2];
    const int nf = split_fields(sv, f, 2);
    if (nf != 2 || !parse_int(f[0], K) || !parse_int(f[1], J)) parse_fail("malformed header (expected 'K J')", ln);
    if (K <= 0) parse_fail("subject count must be positive", ln);
    if (J <= 0) parse_fail("column count must be positive", ln);
    header = true;
  }
  if (!header) throw DataError("empty file: no 'K J' header found");
  // chunks at line boundaries
  const int nt = pick_threads(threads, static_cast<std::size_t>(end - p));
  std::vector<const char*> cut(static_cast<std::size_t>(nt) + 1);
  cut[0] = p;
  cut[static_cast<std::size_t>(nt)] = end;
  for (int t = 1; t < nt; ++t) {
    const char* q = p + (end - p) * t / nt;
    q = std::max(q, cut[static_cast<std::size_t>(t) - 1]);
    const char* nl = q < end ? static_cast<const char*>(std::memchr(q, '\n', static_cast<std::size_t>(end - q))) : nullptr;
    cut[static_cast<std::size_t>(t)] = nl ? nl + 1 : end;
  }
  std::vector<ChunkResult> res(static_cast<std::size_t>(nt));
  run_parallel(nt, [&](int t) {
    parse_chunk(cut[static_cast<std::size_t>(t)], cut[static_cast<std::size_t>(t) + 1], K, J,
                res[static_cast<std::size_t>(t)]);
  });
  long long base = ln;
  for (const ChunkResult& r : res) {  // the first error in file order
    if (r.err_line >= 0) parse_fail(r.err_what, base + r.err_line);
    base += r.lines;
  }
  // group by subject in file order (counting sort over chunks)
  std::vector<std::int64_t> cnt(static_cast<std::size_t>(K) + 1, 0);
  for (const ChunkResult& r : res)
    for (const Entry& e : r.entries) ++cnt[static_cast<std::size_t>(e.k) + 1];
  for (std::int64_t k = 0; k < K; ++k) cnt[static_cast<std::size_t>(k) + 1] += cnt[static_cast<std::size_t>(k)];
  std::vector<Entry> all(static_cast<std::size_t>(cnt[static_cast<std::size_t>(K)]));
  {
    std::vector<std::int64_t> pos(cnt.begin(), cnt.end() - 1);
    for (ChunkResult& r : res) {
      for (const Entry& e : r.entries) all[static_cast<std::size_t>(pos[static_cast<std::size_t>(e.k)]++)] = e;
      std::vector<Entry>().swap(r.entries);
    }
  }
  // normalise subjects in parallel (contiguous subject ranges)
  std::vector<Slice> slices(static_cast<std::size_t>(K));
  const int ns = pick_threads(threads, static_cast<std::size_t>(all.size()) * 16);
  run_parallel(ns, [&](int t) {
    const std::int64_t k0 = K * t / ns, k1 = K * (t + 1) / ns;
    for (std::int64_t k = k0; k < k1; ++k) {
      std::vector<Entry> e(all.begin() + cnt[static_cast<std::size_t>(k)], all.begin() + cnt[static_cast<std::size_t>(k) + 1]);
      normalise_subject(k, e, slices[static_cast<std::size_t>(k)]);
    }
  });
  // flattened CSR: rows in kept order, columns ascending within a row
  auto out = std::make_unique<p2g_csr>();
  out->K = K;
  out->J = J;
  std::int64_t NR = 0, nnz = 0;
  out->srp.resize(static_cast<std::size_t>(K) + 1);
  for (std::int64_t k = 0; k < K; ++k) {
    const Slice& s = slices[static_cast<std::size_t>(k)];
    out->srp[static_cast<std::size_t>(k)] = NR;
    NR += static_cast<std::int64_t>(s.rows_kept.size());
    nnz += static_cast<std::int64_t>(s.entries.size());
  }
  out->srp[static_cast<std::size_t>(K)] = NR;
  out->rp.assign(static_cast<std::size_t>(NR) + 1, 0);
  out->ci.resize(static_cast<std::size_t>(nnz));
  out->val.resize(static_cast<std::size_t>(nnz));
  for (std::int64_t k = 0; k < K; ++k) {
    const Slice& s = slices[static_cast<std::size_t>(k)];
    const std::int64_t r0 = out->srp[static_cast<std::size_t>(k)];
    for (const Entry& e : s.entries) ++out->rp[static_cast<std::size_t>(r0 + e.i) + 1];
  }
  for (std::int64_t r = 0; r < NR; ++r) out->rp[static_cast<std::size_t>(r) + 1] += out->rp[static_cast<std::size_t>(r)];
  {
    std::vector<std::int64_t> fill(out->rp.begin(), out->rp.end() - 1);
    for (std::int64_t k = 0; k < K; ++k) {
      const Slice& s = slices[static_cast<std::size_t>(k)];
      const std::int64_t r0 = out->srp[static_cast<std::size_t>(k)];
      for (const Entry& e : s.entries) {  // (column, row) order: columns ascend within each row
        const std::int64_t q = fill[static_cast<std::size_t>(r0 + e.i)]++;
        out->ci[static_cast<std::size_t>(q)] = static_cast<std::int32_t>(e.j);
        out->val[static_cast<std::size_t>(q)] = e.v;
      }
    }
  }
  // all-zero rows dropped: each subject spanned (max original row + 1) rows
  for (std::int64_t k = 0; k < K; ++k) {
    std::int64_t maxrow = -1;
    for (std::int64_t q = cnt[static_cast<std::size_t>(k)]; q < cnt[static_cast<std::size_t>(k) + 1]; ++q)
      maxrow = std::max(maxrow, all[static_cast<std::size_t>(q)].i);
    out->filtered_rows += (maxrow + 1) - static_cast<std::int64_t>(slices[static_cast<std::size_t>(k)].rows_kept.size());
  }
  return out;
}

std::string format_value(double v) {
  char buf[32];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

void check_csr(std::int64_t K, std::int64_t J, const std::int64_t* srp, const std::int64_t* rp, const std::int32_t* ci,
               const double* val) {
  if (K <= 0 || J <= 0 || !srp || !rp) throw InvalidArgument("invalid CSR tensor");
  if (srp[K] > 0 && rp[srp[K]] > 0 && (!ci || !val)) throw InvalidArgument("invalid CSR tensor");
}

/// Canonical text of subjects [k0, k1) (io.hpp:179-195): subject ascending,
/// then column, then row; values at 17 significant digits.
void format_subjects(std::int64_t k0, std::int64_t k1, const std::int64_t* srp, const std::int64_t* rp,
                     const std::int32_t* ci, const double* val, std::string& out) {
  std::vector<std::int64_t> order, row_of;
  char buf[96];
  for (std::int64_t k = k0; k < k1; ++k) {
    const std::int64_t r0 = srp[k], r1 = srp[k + 1], q0 = rp[r0];
    order.clear();
    row_of.assign(static_cast<std::size_t>(rp[r1] - q0), 0);
    for (std::int64_t r = r0; r < r1; ++r)
      for (std::int64_t q = rp[r]; q < rp[r + 1]; ++q) {
        order.push_back(q);
        row_of[static_cast<std::size_t>(q - q0)] = r - r0;
      }
    // rows ascend in CSR order, so a stable sort by column yields (column, row)
    std::stable_sort(order.begin(), order.end(), [&](std::int64_t a, std::int64_t b) { return ci[a] < ci[b]; });
    for (std::int64_t q : order) {
      const int n = std::snprintf(buf, sizeof(buf), "%lld %lld %d %.17g\n", static_cast<long long>(k),
                                  static_cast<long long>(row_of[static_cast<std::size_t>(q - q0)]), ci[q], val[q]);
      out.append(buf, static_cast<std::size_t>(n));
    }
  }
}

void write_coordinate(std::FILE* f, std::int64_t K, std::int64_t J, const std::int64_t* srp, const std::int64_t* rp,
                      const std::int32_t* ci, const double* val, const std::vector<std::string>& comments) {
  std::string head;
  for (const std::string& c : comments) head += "# " + c + "\n";
  head += std::to_string(K) + " " + std::to_string(J) + "\n";
  std::fwrite(head.data(), 1, head.size(), f);
  // formatted in parallel by subject ranges, written in order
  const int nt = pick_threads(0, static_cast<std::size_t>(rp[srp[K]]) * 24);
  const std::int64_t step = std::max<std::int64_t>(1, std::min<std::int64_t>(K, 4096));
  for (std::int64_t kb = 0; kb < K; kb += step * nt) {
    std::vector<std::string> parts(static_cast<std::size_t>(nt));
    run_parallel(nt, [&](int t) {
      const std::int64_t a = std::min(K, kb + step * t), b = std::min(K, a + step);
      format_subjects(a, b, srp, rp, ci, val, parts[static_cast<std::size_t>(t)]);
    });
    for (const std::string& p : parts) std::fwrite(p.data(), 1, p.size(), f);
  }
}

constexpr char kCacheMagic[8] = {'P', '2', 'G', 'C', 'S', 'R', '0', '1'};

void write_matrix(std::ostream& out, std::int64_t rows, std::int64_t cols, const double* colmajor,
                  const std::string& title) {
  out << "# " << title << '\n' << rows << ' ' << cols << '\n';
  for (std::int64_t r = 0; r < rows; ++r) {
    for (std::int64_t c = 0; c < cols; ++c) {
      if (c) out << ' ';
      out << format_value(colmajor[c * rows + r]);
    }
    out << '\n';
  }
}

void write_matrix_file(const std::filesystem::path& path, std::int64_t rows, std::int64_t cols, const double* colmajor,
                       const std::string& title) {
  std::ofstream out(path);
  if (!out) throw DataError("cannot open output file: " + path.string());
  write_matrix(out, rows, cols, colmajor, title);
  if (!out) throw DataError("failed writing output file: " + path.string());
}

/// read_matrix_stream (io.hpp:218-254); col-major result.
std::vector<double> read_matrix(std::istream& in, std::int64_t& rows, std::int64_t& cols) {
  std::string line;
  long long ln = 0;
  rows = -1;
  cols = -1;
  std::vector<double> m;
  std::int64_t r = 0;
  while (std::getline(in, line)) {
    ++ln;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    const std::string_view sv(line);
    if (skip_line(sv)) continue;
    if (rows < 0) {
      std::string_view f[2];
      const int nf = split_fields(sv, f, 2);
      if (nf != 2 || !parse_int(f[0], rows) || !parse_int(f[1], cols) || rows < 0 || cols < 0)
        parse_fail("malformed matrix header (expected 'rows cols')", ln);
      m.assign(static_cast<std::size_t>(rows * cols), 0.0);
      continue;
    }
    if (r >= rows) parse_fail("unexpected extra matrix row", ln);
    std::vector<std::string_view> f(static_cast<std::size_t>(cols) + 1);
    const int nf = split_fields(sv, f.data(), static_cast<int>(cols) + 1);
    if (nf != cols) parse_fail("wrong number of values in matrix row", ln);
    for (std::int64_t c = 0; c < cols; ++c) {
      double v;
      if (!parse_double(f[static_cast<std::size_t>(c)], v)) parse_fail("malformed matrix value", ln);
      m[static_cast<std::size_t>(c * rows + r)] = v;
    }
    ++r;
  }
  if (rows < 0) throw DataError("empty matrix file");
  if (r != rows) throw DataError("matrix file ended before all rows were read");
  return m;
}

std::string json_escape(const std::string& s) {
  std::string o;
  for (char ch : s) {
    if (ch == '"' || ch == '\\') {
      o += '\\';
      o += ch;
    } else if (ch == '\n') {
      o += "\\n";
    } else {
      o += ch;
    }
  }
  return o;
}

}  // namespace
}  // namespace p2g

using namespace p2g;

extern "C" int p2g_coo_parse(const char* text, int64_t len, int32_t threads, p2g_csr** out) {
  return guarded([&] {
    if (!out || (!text && len > 0) || len < 0) throw InvalidArgument("null argument");
    *out = parse_buffer(text, static_cast<std::size_t>(len), threads).release();
  });
}

extern "C" int p2g_coo_read(const char* path, int32_t threads, p2g_csr** out) {
  return guarded([&] {
    if (!path || !out) throw InvalidArgument("null argument");
    std::FILE* f = std::fopen(path, "rb");
    if (!f) throw DataError(std::string("cannot open input file: ") + path);
    std::vector<char> data;
    std::fseek(f, 0, SEEK_END);
    const long n = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    data.resize(static_cast<std::size_t>(std::max(n, 0L)));
    const std::size_t got = n > 0 ? std::fread(data.data(), 1, data.size(), f) : 0;
    std::fclose(f);
    if (got != data.size()) throw DataError(std::string("failed reading input file: ") + path);
    *out = parse_buffer(data.data(), data.size(), threads).release();
  });
}

extern "C" int p2g_csr_info(const p2g_csr* t, int64_t* K, int64_t* J, int64_t* n_rows, int64_t* nnz,
                            int64_t* filtered_rows) {
  return guarded([&] {
    if (!t) throw InvalidArgument("null tensor");
    if (K) *K = t->K;
    if (J) *J = t->J;
    if (n_rows) *n_rows = t->srp.empty() ? 0 : t->srp.back();
    if (nnz) *nnz = static_cast<int64_t>(t->val.size());
    if (filtered_rows) *filtered_rows = t->filtered_rows;
  });
}

extern "C" int p2g_csr_copy(const p2g_csr* t, int64_t* subj_row_ptr, int64_t* row_ptr, int32_t* col_idx, double* val) {
  return guarded([&] {
    if (!t || !subj_row_ptr || !row_ptr || !col_idx || !val) throw InvalidArgument("null argument");
    std::copy(t->srp.begin(), t->srp.end(), subj_row_ptr);
    std::copy(t->rp.begin(), t->rp.end(), row_ptr);
    std::copy(t->ci.begin(), t->ci.end(), col_idx);
    std::copy(t->val.begin(), t->val.end(), val);
  });
}

extern "C" void p2g_csr_free(p2g_csr* t) { delete t; }

extern "C" int p2g_coo_write(const char* path, int64_t K, int64_t J, const int64_t* srp, const int64_t* rp,
                             const int32_t* ci, const double* val, const char* const* comments, int32_t n_comments) {
  return guarded([&] {
    if (!path) throw InvalidArgument("null path");
    check_csr(K, J, srp, rp, ci, val);
    std::vector<std::string> cm;
    for (int32_t c = 0; c < n_comments; ++c) cm.emplace_back(comments[c]);
    std::FILE* f = std::fopen(path, "wb");
    if (!f) throw DataError(std::string("cannot open output file: ") + path);
    write_coordinate(f, K, J, srp, rp, ci, val, cm);
    const bool bad = std::ferror(f) != 0;
    if (std::fclose(f) != 0 || bad) throw DataError(std::string("failed writing output file: ") + path);
  });
}

extern "C" int p2g_csr_cache_write(const char* path, int64_t K, int64_t J, const int64_t* srp, const int64_t* rp,
                                   const int32_t* ci, const double* val) {
  return guarded([&] {
    if (!path) throw InvalidArgument("null path");
    check_csr(K, J, srp, rp, ci, val);
    const int64_t NR = srp[K], nnz = rp[NR];
    std::ofstream out(path, std::ios::binary);
    if (!out) throw DataError(std::string("cannot open output file: ") + path);
    const int64_t hdr[4] = {K, J, NR, nnz};
    out.write(kCacheMagic, 8);
    out.write(reinterpret_cast<const char*>(hdr), sizeof(hdr));
    out.write(reinterpret_cast<const char*>(srp), static_cast<std::streamsize>(sizeof(int64_t) * (K + 1)));
    out.write(reinterpret_cast<const char*>(rp), static_cast<std::streamsize>(sizeof(int64_t) * (NR + 1)));
    out.write(reinterpret_cast<const char*>(ci), static_cast<std::streamsize>(sizeof(int32_t) * nnz));
    out.write(reinterpret_cast<const char*>(val), static_cast<std::streamsize>(sizeof(double) * nnz));
    if (!out) throw DataError(std::string("failed writing output file: ") + path);
  });
}

extern "C" int p2g_csr_cache_read(const char* path, p2g_csr** out) {
  return guarded([&] {
    if (!path || !out) throw InvalidArgument("null argument");
    std::ifstream in(path, std::ios::binary);
    if (!in) throw DataError(std::string("cannot open input file: ") + path);
    char magic[8];
    int64_t hdr[4];
    in.read(magic, 8);
    in.read(reinterpret_cast<char*>(hdr), sizeof(hdr));
    if (!in || std::memcmp(magic, kCacheMagic, 8) != 0) throw DataError(std::string("not a CSR cache file: ") + path);
    const int64_t K = hdr[0], J = hdr[1], NR = hdr[2], nnz = hdr[3];
    if (K <= 0 || J <= 0 || NR < 0 || nnz < 0) throw DataError("corrupt CSR cache header");
    auto t = std::make_unique<p2g_csr>();
    t->K = K;
    t->J = J;
    t->srp.resize(static_cast<std::size_t>(K) + 1);
    t->rp.resize(static_cast<std::size_t>(NR) + 1);
    t->ci.resize(static_cast<std::size_t>(nnz));
    t->val.resize(static_cast<std::size_t>(nnz));
    in.read(reinterpret_cast<char*>(t->srp.data()), static_cast<std::streamsize>(sizeof(int64_t) * (K + 1)));
    in.read(reinterpret_cast<char*>(t->rp.data()), static_cast<std::streamsize>(sizeof(int64_t) * (NR + 1)));
    in.read(reinterpret_cast<char*>(t->ci.data()), static_cast<std::streamsize>(sizeof(int32_t) * nnz));
    in.read(reinterpret_cast<char*>(t->val.data()), static_cast<std::streamsize>(sizeof(double) * nnz));
    if (!in) throw DataError("truncated CSR cache file");
    if (t->srp[0] != 0 || t->srp[static_cast<std::size_t>(K)] != NR || t->rp[0] != 0 ||
        t->rp[static_cast<std::size_t>(NR)] != nnz)
      throw DataError("corrupt CSR cache offsets");
    *out = t.release();
  });
}

extern "C" int p2g_matrix_write(const char* path, int64_t rows, int64_t cols, const double* colmajor,
                                const char* title) {
  return guarded([&] {
    if (!path || rows < 0 || cols < 0 || (!colmajor && rows * cols > 0)) throw InvalidArgument("invalid matrix");
    write_matrix_file(path, rows, cols, colmajor, title ? title : "");
  });
}

extern "C" int p2g_matrix_read(const char* path, int64_t* rows, int64_t* cols, double* colmajor, int64_t capacity) {
  return guarded([&] {
    if (!path || !rows || !cols) throw InvalidArgument("null argument");
    std::ifstream in(path);
    if (!in) throw DataError(std::string("cannot open matrix file: ") + path);
    const std::vector<double> m = read_matrix(in, *rows, *cols);
    if (colmajor) {
      if (capacity < static_cast<int64_t>(m.size())) throw InvalidArgument("matrix buffer too small");
      std::copy(m.begin(), m.end(), colmajor);
    }
  });
}

extern "C" int p2g_matrix_parse(const char* text, int64_t len, int64_t* rows, int64_t* cols, double* colmajor,
                                int64_t capacity) {
  return guarded([&] {
    if ((!text && len > 0) || !rows || !cols) throw InvalidArgument("null argument");
    std::istringstream in(std::string(text ? text : "", static_cast<std::size_t>(len)));
    const std::vector<double> m = read_matrix(in, *rows, *cols);
    if (colmajor) {
      if (capacity < static_cast<int64_t>(m.size())) throw InvalidArgument("matrix buffer too small");
      std::copy(m.begin(), m.end(), colmajor);
    }
  });
}

extern "C" int p2g_write_factors(const char* dir, int64_t K, int64_t J, int32_t R, const int64_t* subj_row_ptr,
                                 const double* H, const double* V, const double* S, const double* Q,
                                 const char* metadata_json) {
  return guarded([&] {
    namespace fs = std::filesystem;
    if (!dir || K < 0 || J < 0 || R < 1 || !H || !V || !S || (K > 0 && (!subj_row_ptr || !Q)))
      throw InvalidArgument("invalid factor set");
    fs::create_directories(dir);
    const fs::path d(dir);
    write_matrix_file(d / "V.txt", J, R, V, "column factor V (J x R)");
    write_matrix_file(d / "S.txt", K, R, S, "subject scales S (K x R; row k = diag(S_k))");
    write_matrix_file(d / "H.txt", R, R, H, "shared factor H (R x R)");
    // U_k = Q_k H (assemble_U, solver.hpp:238-243); Q packed row-major
    std::vector<double> u;
    for (int64_t k = 0; k < K; ++k) {
      const int64_t r0 = subj_row_ptr[k], I = subj_row_ptr[k + 1] - r0;
      u.assign(static_cast<std::size_t>(I * R), 0.0);
      for (int64_t i = 0; i < I; ++i)
        for (int32_t c = 0; c < R; ++c) {
          double acc = 0.0;
          for (int32_t a = 0; a < R; ++a) acc += Q[(r0 + i) * R + a] * H[c * R + a];
          u[static_cast<std::size_t>(c * I + i)] = acc;
        }
      const std::string name = "U_" + std::to_string(k) + ".txt";
      write_matrix_file(d / name, I, R, u.data(), "subject factor U_" + std::to_string(k) + " (I_k x R)");
    }
    std::ofstream m(d / "manifest.json");
    if (!m) throw DataError("cannot open output file: manifest.json");
    m << "{\n  \"rank\": " << R << ",\n  \"subjects\": " << K << ",\n  \"columns\": " << J
      << ",\n  \"files\": {\n    \"V\": \"V.txt\",\n    \"S\": \"S.txt\",\n    \"H\": \"H.txt\",\n    \"U\": [";
    for (int64_t k = 0; k < K; ++k) m << (k ? ", " : "") << "\"U_" << k << ".txt\"";
    m << "]\n  },\n  \"prng\": \""
      << json_escape("mt19937_64; uniforms = (x >> 11) * 2^-53; normals via Box-Muller; per-subject substreams via "
                     "splitmix64")
      << "\"";
    if (metadata_json && std::strlen(metadata_json) > 0 && std::string(metadata_json) != "{}")
      m << ",\n  \"config\": " << metadata_json;
    m << "\n}\n";
    if (!m) throw DataError("failed writing manifest.json");
  });
}

extern "C" int p2g_write_trace(const char* path, int32_t n, const int32_t* iters, const double* residual_sq,
                               const double* fit) {
  return guarded([&] {
    if (!path || n < 0 || (n > 0 && (!iters || !residual_sq || !fit))) throw InvalidArgument("invalid trace");
    std::ofstream out(path);
    if (!out) throw DataError(std::string("cannot open output file: ") + path);
    out << "iter\tresidual_sq\tfit\n";  // deterministic fields only (io.hpp:307-315)
    for (int32_t i = 0; i < n; ++i)
      out << iters[i] << '\t' << format_value(residual_sq[i]) << '\t' << format_value(fit[i]) << '\n';
    if (!out) throw DataError(std::string("failed writing output file: ") + path);
  });
}
