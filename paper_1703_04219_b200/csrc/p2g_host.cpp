// Host-side (CPU-only) part of the C ABI: error plumbing, the bit-exact
// partition_weighted, the BASELINE synthetic-workload generator and the
// initial factors.  No CUDA here, so these entry points work on a box
// without a GPU.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <thread>
#include <vector>

#include "p2g_common.hpp"

namespace p2g {

namespace {
// Trivially destructible on purpose: a static object's destructor (e.g. the
// drop-in headers' Device) may call into the ABI after the main thread's
// thread_local objects have been destroyed at exit.
thread_local char g_last_error[1024];
}

void set_last_error(const std::string& msg) {
  const std::size_t n = std::min(msg.size(), sizeof(g_last_error) - 1);
  std::memcpy(g_last_error, msg.data(), n);
  g_last_error[n] = '\0';
}

/// parallel.hpp:51-79 (and partition_even :34-45 for zero total weight).
void partition_weighted(const std::uint64_t* w, std::int64_t n, std::int32_t n_chunks,
                        std::vector<std::pair<std::int64_t, std::int64_t>>& out) {
  out.clear();
  const std::int64_t chunks =
      std::max<std::int64_t>(1, std::min<std::int64_t>(n_chunks, std::max<std::int64_t>(n, 1)));
  std::uint64_t total = 0;
  for (std::int64_t i = 0; i < n; ++i) total += w[i];
  if (total == 0) {
    for (std::int64_t c = 0; c < chunks; ++c) out.emplace_back(n * c / chunks, n * (c + 1) / chunks);
    return;
  }
  std::int64_t begin = 0;
  std::uint64_t cum = 0;
  for (std::int64_t c = 0; c < chunks; ++c) {
    const std::uint64_t target = total * static_cast<std::uint64_t>(c + 1) / static_cast<std::uint64_t>(chunks);
    std::int64_t end = begin;
    while (end < n && (cum < target || end == begin) && n - end > chunks - c - 1) cum += w[end++];
    if (c + 1 == chunks) end = n;
    out.emplace_back(begin, end);
    begin = end;
  }
}

}  // namespace p2g

using namespace p2g;

extern "C" const char* p2g_last_error(void) { return g_last_error; }

extern "C" const char* p2g_version(void) { return "p2g 0.1 (sm_100a, fp64)"; }

extern "C" int p2g_partition_weighted(const uint64_t* weights, int64_t n, int32_t n_chunks, int64_t* begin_end,
                                      int32_t* n_out) {
  return guarded([&] {
    if (n < 0 || (n > 0 && !weights) || !begin_end || !n_out) throw InvalidArgument("partition_weighted: bad arguments");
    std::vector<std::pair<std::int64_t, std::int64_t>> r;
    partition_weighted(weights, n, n_chunks, r);
    for (std::size_t i = 0; i < r.size(); ++i) {
      begin_end[2 * i] = r[i].first;
      begin_end[2 * i + 1] = r[i].second;
    }
    *n_out = static_cast<int32_t>(r.size());
  });
}

// ---------------------------------------------------------------------------
// BASELINE synthetic generator.
// ---------------------------------------------------------------------------
struct p2g_gen {
  std::int64_t K = 0, J = 0;
  std::vector<std::int64_t> subj_row_ptr;  // K+1
  // Per-thread chunks, concatenated on export.
  struct Chunk {
    std::vector<std::int64_t> row_nnz;
    std::vector<std::int32_t> cols;
    std::vector<double> vals;
  };
  std::vector<Chunk> chunks;
  std::int64_t n_rows = 0, nnz = 0;
};

namespace {

std::int64_t poisson_inversion(double lambda, double u) {
  // Inversion on one pinned uniform (D11).
  std::int64_t k = 0;
  double p = std::exp(-lambda);
  double F = p;
  while (u > F && k < 100000) {
    ++k;
    p *= lambda / static_cast<double>(k);
    F += p;
  }
  return k;
}

void validate_spec(const p2g_gen_spec& s) {
  if (s.K < 1) throw InvalidArgument("generator: K must be at least 1");
  if (s.J < 1 || s.J > (1ll << 31) - 1) throw InvalidArgument("generator: J out of range");
  if (s.rows_lo < 1 || s.rows_hi < s.rows_lo) throw InvalidArgument("generator: bad row range");
  if (s.rows_dist == 1 && !(s.rows_mean >= 1.0)) throw InvalidArgument("generator: geometric mean must be >= 1");
  if (s.nnz_dist == 0 && (s.nnz_lo < 1 || s.nnz_hi < s.nnz_lo)) throw InvalidArgument("generator: bad nnz range");
  if (s.nnz_dist == 1 && !(s.nnz_lambda >= 0.0)) throw InvalidArgument("generator: lambda must be >= 0");
  if (s.col_dist == 1 && !(s.zipf_s > 0.0)) throw InvalidArgument("generator: zipf exponent must be > 0");
}

}  // namespace

extern "C" int p2g_gen_baseline_spec(int32_t config_id, int32_t R, p2g_gen_spec* spec) {
  return guarded([&] {
    if (!spec) throw InvalidArgument("null spec");
    if (R < 1) throw InvalidArgument("rank must be at least 1");
    p2g_gen_spec s{};
    s.min_rows = R;
    s.threads = 0;
    s.rows_dist = 0;
    s.col_dist = 0;
    s.val_dist = 0;
    switch (config_id) {
      case 1:  // tiny CPU-oracle run
        s.K = 1000; s.J = 500; s.rows_lo = 1; s.rows_hi = 50;
        s.nnz_dist = 0; s.nnz_lo = 1; s.nnz_hi = 10; s.seed = 101;
        break;
      case 2:  // paper-scale R=10, ~63M nnz
        s.K = 1000000; s.J = 5000; s.rows_lo = 1; s.rows_hi = 100;
        s.nnz_dist = 1; s.nnz_lambda = 0.235; s.seed = 102;
        break;
      case 3:  // paper-scale R=40, ~250M nnz
        s.K = 1000000; s.J = 5000; s.rows_lo = 1; s.rows_hi = 100;
        s.nnz_dist = 1; s.nnz_lambda = 3.29; s.seed = 103;
        break;
      case 4:  // largest paper-scale, ~500M nnz
        s.K = 1000000; s.J = 5000; s.rows_lo = 1; s.rows_hi = 100;
        s.nnz_dist = 1; s.nnz_lambda = 7.58; s.seed = 104;
        break;
      case 5:  // EHR-shaped skew
        s.K = 500000; s.J = 1500; s.rows_dist = 1; s.rows_lo = 1; s.rows_hi = 500; s.rows_mean = 30.0;
        s.nnz_dist = 1; s.nnz_lambda = 4.0; s.col_dist = 1; s.zipf_s = 1.1; s.val_dist = 1; s.seed = 105;
        break;
      default:
        throw InvalidArgument("config_id must be 1..5");
    }
    *spec = s;
  });
}

extern "C" int p2g_gen_create(const p2g_gen_spec* spec_in, p2g_gen** out, int64_t* n_rows, int64_t* nnz) {
  return guarded([&] {
    if (!spec_in || !out) throw InvalidArgument("null argument");
    const p2g_gen_spec s = *spec_in;
    validate_spec(s);
    auto g = std::make_unique<p2g_gen>();
    g->K = s.K;
    g->J = s.J;
    // Zipf CDF over column ids (popularity rank = column id).
    std::vector<double> zcdf;
    if (s.col_dist == 1) {
      zcdf.resize(static_cast<std::size_t>(s.J));
      double acc = 0.0;
      for (std::int64_t j = 0; j < s.J; ++j) {
        acc += 1.0 / std::pow(static_cast<double>(j + 1), s.zipf_s);
        zcdf[static_cast<std::size_t>(j)] = acc;
      }
    }
    int nt = s.threads > 0 ? s.threads : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    nt = static_cast<int>(std::min<std::int64_t>(nt, s.K));
    g->chunks.resize(static_cast<std::size_t>(nt));
    std::vector<std::int64_t> rows_of(static_cast<std::size_t>(s.K));
    auto work = [&](int t) {
      const std::int64_t k0 = s.K * t / nt, k1 = s.K * (t + 1) / nt;
      p2g_gen::Chunk& ch = g->chunks[static_cast<std::size_t>(t)];
      std::vector<std::int32_t> rowcols;
      std::vector<char> used(static_cast<std::size_t>(s.J), 0);
      for (std::int64_t k = k0; k < k1; ++k) {
        Rng rng(substream_seed(s.seed, static_cast<std::uint64_t>(k) + 1));
        std::int64_t I;
        if (s.rows_dist == 0) {
          I = s.rows_lo + static_cast<std::int64_t>(rng.below(static_cast<std::uint64_t>(s.rows_hi - s.rows_lo + 1)));
        } else {
          const double p = 1.0 / s.rows_mean;
          const double u = rng.uniform();
          const double gsz = std::floor(std::log1p(-u) / std::log1p(-p));
          I = 1 + static_cast<std::int64_t>(std::min(gsz, 1e15));
          if (I > s.rows_hi) I = s.rows_hi;
        }
        I = std::max(I, s.min_rows);
        rows_of[static_cast<std::size_t>(k)] = I;
        for (std::int64_t i = 0; i < I; ++i) {
          std::int64_t n;
          if (s.nnz_dist == 0)
            n = s.nnz_lo + static_cast<std::int64_t>(rng.below(static_cast<std::uint64_t>(s.nnz_hi - s.nnz_lo + 1)));
          else
            n = 1 + poisson_inversion(s.nnz_lambda, rng.uniform());
          n = std::min(n, s.J);
          rowcols.clear();
          while (static_cast<std::int64_t>(rowcols.size()) < n) {
            std::int64_t c;
            if (s.col_dist == 0) {
              c = static_cast<std::int64_t>(rng.below(static_cast<std::uint64_t>(s.J)));
            } else {
              const double u = rng.uniform() * zcdf.back();
              c = static_cast<std::int64_t>(std::upper_bound(zcdf.begin(), zcdf.end(), u) - zcdf.begin());
              if (c >= s.J) c = s.J - 1;
            }
            if (used[static_cast<std::size_t>(c)]) continue;  // distinct per row, by rejection
            used[static_cast<std::size_t>(c)] = 1;
            rowcols.push_back(static_cast<std::int32_t>(c));
          }
          std::sort(rowcols.begin(), rowcols.end());
          for (std::int32_t c : rowcols) {
            used[static_cast<std::size_t>(c)] = 0;
            const double v = s.val_dist == 0 ? 1.0 - rng.uniform() : 1.0 + static_cast<double>(rng.below(5));
            ch.cols.push_back(c);
            ch.vals.push_back(v);
          }
          ch.row_nnz.push_back(n);
        }
      }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nt; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    g->subj_row_ptr.resize(static_cast<std::size_t>(s.K + 1));
    g->subj_row_ptr[0] = 0;
    for (std::int64_t k = 0; k < s.K; ++k)
      g->subj_row_ptr[static_cast<std::size_t>(k + 1)] = g->subj_row_ptr[static_cast<std::size_t>(k)] + rows_of[static_cast<std::size_t>(k)];
    g->n_rows = g->subj_row_ptr.back();
    g->nnz = 0;
    for (const auto& ch : g->chunks) g->nnz += static_cast<std::int64_t>(ch.vals.size());
    if (n_rows) *n_rows = g->n_rows;
    if (nnz) *nnz = g->nnz;
    *out = g.release();
  });
}

extern "C" int p2g_gen_export(const p2g_gen* g, int64_t* subj_row_ptr, int64_t* row_ptr, int32_t* col_idx,
                              double* val) {
  return guarded([&] {
    if (!g) throw InvalidArgument("null generator");
    if (subj_row_ptr) std::memcpy(subj_row_ptr, g->subj_row_ptr.data(), g->subj_row_ptr.size() * sizeof(int64_t));
    // Concatenate chunks (threads over chunks).
    std::vector<std::int64_t> row_off(g->chunks.size() + 1, 0), nz_off(g->chunks.size() + 1, 0);
    for (std::size_t c = 0; c < g->chunks.size(); ++c) {
      row_off[c + 1] = row_off[c] + static_cast<std::int64_t>(g->chunks[c].row_nnz.size());
      nz_off[c + 1] = nz_off[c] + static_cast<std::int64_t>(g->chunks[c].vals.size());
    }
    auto work = [&](std::size_t c) {
      const auto& ch = g->chunks[c];
      if (row_ptr) {
        std::int64_t p = nz_off[c];
        for (std::size_t r = 0; r < ch.row_nnz.size(); ++r) {
          row_ptr[row_off[c] + static_cast<std::int64_t>(r)] = p;
          p += ch.row_nnz[r];
        }
      }
      if (col_idx) std::memcpy(col_idx + nz_off[c], ch.cols.data(), ch.cols.size() * sizeof(int32_t));
      if (val) std::memcpy(val + nz_off[c], ch.vals.data(), ch.vals.size() * sizeof(double));
    };
    std::vector<std::thread> th;
    for (std::size_t c = 1; c < g->chunks.size(); ++c) th.emplace_back(work, c);
    if (!g->chunks.empty()) work(0);
    for (auto& x : th) x.join();
    if (row_ptr) row_ptr[g->n_rows] = g->nnz;
  });
}

extern "C" void p2g_gen_free(p2g_gen* g) { delete g; }

extern "C" int p2g_init_factors(uint64_t seed, int64_t K, int64_t J, int32_t R, double* H, double* V, double* W) {
  return guarded([&] {
    if (K < 1 || J < 1 || R < 1) throw InvalidArgument("init_factors: bad shape");
    if (H)
      for (int32_t c = 0; c < R; ++c)
        for (int32_t r = 0; r < R; ++r) H[r + static_cast<int64_t>(c) * R] = r == c ? 1.0 : 0.0;
    Rng rng(seed);
    for (int32_t r = 0; r < R; ++r)
      for (int64_t j = 0; j < J; ++j) {
        const double u = rng.uniform();
        if (V) V[j + static_cast<int64_t>(r) * J] = u;
      }
    for (int32_t r = 0; r < R; ++r)
      for (int64_t k = 0; k < K; ++k) {
        const double u = rng.uniform();
        if (W) W[k + static_cast<int64_t>(r) * K] = u;
      }
  });
}

extern "C" int p2g_initialize_random(uint64_t seed, int64_t K, int64_t J, int32_t R, double* H, double* S, double* V) {
  return guarded([&] {
    if (R < 1) throw InvalidArgument("rank must be at least 1");
    if (J < R)
      throw DataError("rank exceeds variables: J = " + std::to_string(J) + " < rank " + std::to_string(R));
    if (H)
      for (int32_t c = 0; c < R; ++c)
        for (int32_t r = 0; r < R; ++r) H[r + static_cast<int64_t>(c) * R] = r == c ? 1.0 : 0.0;
    if (S)
      for (int64_t i = 0; i < K * R; ++i) S[i] = 1.0;
    Rng rng(seed);
    for (int32_t r = 0; r < R; ++r)
      for (int64_t j = 0; j < J; ++j) {
        const double u = rng.uniform();
        if (V) V[j + static_cast<int64_t>(r) * J] = u;
      }
  });
}
