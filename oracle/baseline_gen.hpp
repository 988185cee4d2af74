// TEST INFRASTRUCTURE ONLY (see p2_oracle.hpp's header): the BASELINE
// synthetic workload of SURVEY.md §8(d), restated on the oracle side so the
// CPU arms of bench.py (`cpu_baseline`, `--impl reference`) build their
// inputs without mapping the product library.  tests/test_baseline_gen.py
// pins it bit-for-bit against libp2g's generator (p2g_gen_create).
//
// Stream layout (SURVEY.md §8d "Common rules", decisions D1/D2/D10/D11):
//   subject k draws from Rng(substream_seed(seed, k + 1)) (generator.hpp:118):
//     I_k (uniform rows_lo..rows_hi, or geometric with the given mean, capped),
//     then I_k <- max(I_k, R)                                           (D1)
//     per row: nnz_row (uniform, or 1 + Poisson(lambda) by inversion)   (D11)
//              distinct columns by rejection (uniform or Zipf), sorted
//              values 1 - uniform() (Uniform(0,1]) or 1 + below(5)
//   initial factors: H = I; Rng(seed) fills V r-outer/j-inner
//   (solver.hpp:128-132), then the same stream fills W r-outer/k-inner (D2).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <thread>
#include <vector>

#include "p2_oracle.hpp"

namespace p2o {
namespace baseline {

struct Spec {
  std::int64_t K = 0, J = 0;
  int rows_dist = 0;  // 0 uniform{rows_lo..rows_hi}, 1 geometric(mean) capped at rows_hi
  std::int64_t rows_lo = 1, rows_hi = 1;
  double rows_mean = 1.0;
  int nnz_dist = 0;  // 0 uniform{nnz_lo..nnz_hi}, 1 1 + Poisson(lambda)
  std::int64_t nnz_lo = 1, nnz_hi = 1;
  double lambda = 0.0;
  int col_dist = 0;  // 0 uniform over [0, J), 1 Zipf(s), popularity rank = column id
  double zipf_s = 1.0;
  int val_dist = 0;  // 0 Uniform(0,1], 1 integer 1..5
  std::uint64_t seed = 0;
  std::int64_t min_rows = 1;  // D1
};

/// BASELINE.json configs 1..5 with SURVEY.md §8(d)'s concrete parameters.
inline Spec config(int id, int R) {
  Spec s;
  s.min_rows = R;
  switch (id) {
    case 1:
      s.K = 1000; s.J = 500; s.rows_lo = 1; s.rows_hi = 50;
      s.nnz_dist = 0; s.nnz_lo = 1; s.nnz_hi = 10; s.seed = 101;
      break;
    case 2:
      s.K = 1000000; s.J = 5000; s.rows_lo = 1; s.rows_hi = 100;
      s.nnz_dist = 1; s.lambda = 0.235; s.seed = 102;
      break;
    case 3:
      s.K = 1000000; s.J = 5000; s.rows_lo = 1; s.rows_hi = 100;
      s.nnz_dist = 1; s.lambda = 3.29; s.seed = 103;
      break;
    case 4:
      s.K = 1000000; s.J = 5000; s.rows_lo = 1; s.rows_hi = 100;
      s.nnz_dist = 1; s.lambda = 7.58; s.seed = 104;
      break;
    case 5:
      s.K = 500000; s.J = 1500; s.rows_dist = 1; s.rows_lo = 1; s.rows_hi = 500; s.rows_mean = 30.0;
      s.nnz_dist = 1; s.lambda = 4.0; s.col_dist = 1; s.zipf_s = 1.1; s.val_dist = 1; s.seed = 105;
      break;
    default:
      throw std::invalid_argument("config id must be 1..5");
  }
  return s;
}

/// One pinned uniform -> Poisson(lambda) by summing the pmf until it passes u.
inline std::int64_t poisson_by_inversion(double lambda, double u) {
  std::int64_t k = 0;
  double pk = std::exp(-lambda), cdf = pk;
  while (u > cdf && k < 100000) {
    ++k;
    pk *= lambda / static_cast<double>(k);
    cdf += pk;
  }
  return k;
}

struct Csr {
  std::int64_t J = 0;
  std::vector<std::int64_t> subj_row_ptr, row_ptr;
  std::vector<std::int32_t> col_idx;
  std::vector<double> val;
};

/// Subjects [0, K_use) of the config's tensor (a prefix of the full
/// workload: subject k's stream does not depend on K).
inline Csr generate(const Spec& s, std::int64_t K_use, int threads) {
  if (K_use <= 0 || K_use > s.K) K_use = s.K;
  std::vector<double> zipf;  // cumulative popularity weights
  if (s.col_dist == 1) {
    zipf.resize(static_cast<std::size_t>(s.J));
    double run = 0.0;
    for (std::int64_t j = 0; j < s.J; ++j) zipf[static_cast<std::size_t>(j)] = run += 1.0 / std::pow(double(j + 1), s.zipf_s);
  }
  struct Part {
    std::vector<std::int64_t> rows;     // I_k per subject
    std::vector<std::int64_t> row_nnz;  // per row
    std::vector<std::int32_t> cols;
    std::vector<double> vals;
  };
  const int nt = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(threads > 0 ? threads : 1, K_use)));
  std::vector<Part> parts(static_cast<std::size_t>(nt));
  auto make = [&](int t) {
    Part& P = parts[static_cast<std::size_t>(t)];
    std::vector<std::uint8_t> taken(static_cast<std::size_t>(s.J), 0);
    std::vector<std::int32_t> row;
    for (std::int64_t k = K_use * t / nt; k < K_use * (t + 1) / nt; ++k) {
      Rng g(substream_seed(s.seed, static_cast<std::uint64_t>(k + 1)));
      std::int64_t I = 0;
      if (s.rows_dist == 0) {
        I = s.rows_lo + static_cast<std::int64_t>(g.below(static_cast<std::uint64_t>(s.rows_hi - s.rows_lo + 1)));
      } else {
        const double fails = std::floor(std::log1p(-g.uniform()) / std::log1p(-1.0 / s.rows_mean));
        I = std::min<std::int64_t>(1 + static_cast<std::int64_t>(std::min(fails, 1e15)), s.rows_hi);
      }
      if (I < s.min_rows) I = s.min_rows;
      P.rows.push_back(I);
      for (std::int64_t i = 0; i < I; ++i) {
        std::int64_t n = s.nnz_dist == 0
                             ? s.nnz_lo + static_cast<std::int64_t>(g.below(static_cast<std::uint64_t>(s.nnz_hi - s.nnz_lo + 1)))
                             : 1 + poisson_by_inversion(s.lambda, g.uniform());
        if (n > s.J) n = s.J;
        row.clear();
        while (static_cast<std::int64_t>(row.size()) < n) {
          std::int64_t c;
          if (s.col_dist == 0) {
            c = static_cast<std::int64_t>(g.below(static_cast<std::uint64_t>(s.J)));
          } else {
            const double x = g.uniform() * zipf.back();
            c = std::min<std::int64_t>(static_cast<std::int64_t>(std::upper_bound(zipf.begin(), zipf.end(), x) - zipf.begin()),
                                       s.J - 1);
          }
          if (taken[static_cast<std::size_t>(c)]) continue;
          taken[static_cast<std::size_t>(c)] = 1;
          row.push_back(static_cast<std::int32_t>(c));
        }
        std::sort(row.begin(), row.end());
        for (const std::int32_t c : row) {
          taken[static_cast<std::size_t>(c)] = 0;
          P.cols.push_back(c);
          P.vals.push_back(s.val_dist == 0 ? 1.0 - g.uniform() : 1.0 + static_cast<double>(g.below(5)));
        }
        P.row_nnz.push_back(n);
      }
    }
  };
  {
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(make, t);
    make(0);
    for (auto& th : pool) th.join();
  }
  Csr out;
  out.J = s.J;
  out.subj_row_ptr.assign(1, 0);
  out.row_ptr.assign(1, 0);
  for (const Part& P : parts) {
    for (const std::int64_t I : P.rows) out.subj_row_ptr.push_back(out.subj_row_ptr.back() + I);
    for (const std::int64_t n : P.row_nnz) out.row_ptr.push_back(out.row_ptr.back() + n);
    out.col_idx.insert(out.col_idx.end(), P.cols.begin(), P.cols.end());
    out.val.insert(out.val.end(), P.vals.begin(), P.vals.end());
  }
  return out;
}

/// D2: H = I, V then W (first K_use of K rows) from one Rng(seed) stream;
/// column-major (V J x R, W K_use x R).
inline void init_factors(std::uint64_t seed, std::int64_t K, std::int64_t K_use, std::int64_t J, int R,
                         std::vector<double>& H, std::vector<double>& V, std::vector<double>& W) {
  if (K_use <= 0 || K_use > K) K_use = K;
  H.assign(static_cast<std::size_t>(R) * R, 0.0);
  for (int r = 0; r < R; ++r) H[static_cast<std::size_t>(r) * R + r] = 1.0;
  V.resize(static_cast<std::size_t>(J) * R);
  W.resize(static_cast<std::size_t>(K_use) * R);
  Rng g(seed);
  for (int r = 0; r < R; ++r)
    for (std::int64_t j = 0; j < J; ++j) V[static_cast<std::size_t>(r) * J + j] = g.uniform();
  for (int r = 0; r < R; ++r)
    for (std::int64_t k = 0; k < K; ++k) {
      const double x = g.uniform();
      if (k < K_use) W[static_cast<std::size_t>(r) * K_use + k] = x;
    }
}

}  // namespace baseline
}  // namespace p2o
