// Reference tests restated through the drop-in C++ headers (include/parafac2)
// on top of libp2g — the way a reference user would call the engine.
// Each CHECK mirrors an assertion of /root/reference/proj/tests/*.cpp (cited).
// Exit code 0 iff every check passed.
#include <cmath>
#include <cstdio>
#include <functional>
#include <sstream>
#include <string>

#include "parafac2/parafac2.hpp"

using namespace parafac2;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                             \
  do {                                                                          \
    if (cond) {                                                                 \
      ++g_pass;                                                                 \
    } else {                                                                    \
      ++g_fail;                                                                 \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);               \
    }                                                                           \
  } while (0)

template <typename Ex, typename Fn>
static bool throws(Fn&& fn) {
  try {
    fn();
  } catch (const Ex&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static double maxabs(const Matrix& a) {
  double m = 0.0;
  for (Index i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a.data()[i]));
  return m;
}

// helpers.hpp:62-93
static SparseSlice random_slice(Rng& rng, Index rows, Index cols, double density) {
  std::vector<Triplet> e;
  for (Index i = 0; i < rows; ++i)
    for (Index j = 0; j < cols; ++j)
      if (rng.uniform() < density) e.push_back({i, j, rng.uniform(-1.0, 1.0)});
  if (e.empty()) {
    const Index i = static_cast<Index>(rng.below(static_cast<std::uint64_t>(rows)));
    const Index j = static_cast<Index>(rng.below(static_cast<std::uint64_t>(cols)));
    e.push_back({i, j, rng.uniform(0.5, 1.5)});
  }
  return SparseSlice::from_triplets(rows, cols, e);
}
static IrregularTensor random_tensor(Rng& rng, Index n, Index cols, Index lo, Index hi, double density) {
  std::vector<SparseSlice> s;
  for (Index k = 0; k < n; ++k) {
    Index rows = lo;
    if (hi > lo) rows += static_cast<Index>(rng.below(static_cast<std::uint64_t>(hi - lo + 1)));
    s.push_back(random_slice(rng, rows, cols, density));
  }
  return IrregularTensor::from_slices(cols, std::move(s));
}
// helpers.hpp:132-141
static double dense_residual(const IrregularTensor& x, const Parafac2Factors& f) {
  double total = 0.0;
  for (Index k = 0; k < x.n_slices(); ++k) {
    Matrix HS = f.H;
    for (Index c = 0; c < HS.cols(); ++c)
      for (Index r = 0; r < HS.rows(); ++r) HS(r, c) *= f.S(k, c);
    const Matrix model = f.Q[static_cast<std::size_t>(k)] * HS * f.V.transpose();
    total += (x.slice(k).dense() - model).squaredNorm();
  }
  return total;
}

int main() {
  // test_io.cpp:55-163, 212-222, 276-293 — ingest/export through io.hpp
  {
    auto parse = [](const std::string& t) {
      std::istringstream in(t);
      return parse_coordinate_stream(in);
    };
    ParsedTensor p = parse("2 3\n0 0 1 2.5\n1 0 0 1.0\n");
    CHECK(p.tensor.n_slices() == 2 && p.tensor.slice(0).dense()(0, 1) == 2.5 && p.filtered_rows == 0);
    CHECK(parse("1 3\n0 5 1 2.0\n").filtered_rows == 5);
    bool msg_ok = false;
    try {
      parse("1 3\n0 0 5 1.0\n");
    } catch (const DataError& e) {
      msg_ok = std::string(e.what()).find("column index out of range at line 2") != std::string::npos;
    }
    CHECK(msg_ok);
    CHECK(throws<DataError>([&] { parse(""); }));
    auto t = IrregularTensor::from_slices(
        3, {SparseSlice::from_triplets(2, 3, {{1, 2, 2.5}, {0, 0, 1.5}}), SparseSlice::from_triplets(1, 3, {{0, 1, -3.0}})});
    std::ostringstream ser;
    write_coordinate_stream(ser, t, {"demo"});
    CHECK(ser.str() == "# demo\n2 3\n0 0 0 1.5\n0 1 2 2.5\n1 0 1 -3\n");
    Matrix m = Matrix::FromRows(2, 2, {1.5, -3.0, 0.25, 100.0});
    std::ostringstream ms;
    write_matrix_stream(ms, m, "demo");
    CHECK(ms.str() == "# demo\n2 2\n1.5 -3\n0.25 100\n");
    std::istringstream mi(ms.str());
    CHECK(read_matrix_stream(mi) == m);
    FitTrace tr;
    IterationStats a, b;
    a.iter = 1, a.residual_sq = 2.5, a.fit = 0.5, a.ms_procrustes = 123.0;
    b.iter = 2, b.residual_sq = 1.25, b.fit = 0.75;
    tr.iterations = {a, b};
    std::ostringstream ts;
    write_trace_tsv(ts, tr);
    CHECK(ts.str() == "iter\tresidual_sq\tfit\n1\t2.5\t0.5\n2\t1.25\t0.75\n");
  }
  // test_mttkrp.cpp:36-101 — mode KATs
  {
    Matrix y = Matrix::FromRows(2, 2, {1, 0, 0, 2});
    auto Y = ProjectedSlices::from_dense(2, {y});
    Matrix w = Matrix::FromRows(1, 2, {3, 5});
    CHECK(mttkrp_mode1(Y, Matrix::Ones(2, 2), w) == Matrix::FromRows(2, 2, {3, 5, 6, 10}));
    CHECK(mttkrp_mode2(Y, Matrix::Identity(2, 2), w) == Matrix::FromRows(2, 2, {3, 0, 0, 10}));
    Matrix m3 = mttkrp_mode3(Y, Matrix::FromRows(2, 2, {1, 2, 3, 4}), Matrix::Ones(2, 2));
    CHECK(m3(0, 0) == 7.0 && m3(0, 1) == 10.0);
    auto Y2 = ProjectedSlices::from_packed(1, 3, {Matrix::Constant(1, 1, 4), Matrix::Constant(1, 1, 7)}, {{0}, {2}});
    Matrix m2 = mttkrp_mode2(Y2, Matrix::Constant(1, 1, 1), Matrix::FromRows(2, 1, {1, 10}));
    CHECK(m2(0, 0) == 4.0 && m2(1, 0) == 0.0 && m2(2, 0) == 70.0);
    CHECK(throws<std::invalid_argument>([&] { mttkrp(Y, Matrix::Ones(3, 2), Matrix::Ones(2, 2), w, 1); }));
    CHECK(throws<std::invalid_argument>([&] { mttkrp(Y, Matrix::Identity(2, 2), Matrix::Ones(2, 2), w, 4); }));
  }
  // test_kernels.cpp:85-201 — gram, pinv, nnls KATs
  {
    CHECK(gram(Matrix::FromRows(2, 2, {1, 2, 3, 4})) == Matrix::FromRows(2, 2, {10, 14, 14, 20}));
    CHECK(maxabs(pinv_small(Matrix::FromRows(2, 2, {2, 1, 1, 2})) -
                 Matrix::FromRows(2, 2, {2.0 / 3, -1.0 / 3, -1.0 / 3, 2.0 / 3})) < 1e-14);
    CHECK(maxabs(pinv_small(Matrix::FromRows(2, 2, {4, 0, 0, 0})) - Matrix::FromRows(2, 2, {0.25, 0, 0, 0})) < 1e-14);
    Matrix x = nnls_rowwise(Matrix::Identity(2, 2), Matrix::FromRows(1, 2, {1, -2}));
    CHECK(std::abs(x(0, 0) - 1.0) < 1e-12 && x(0, 1) == 0.0);
    x = nnls_rowwise(Matrix::FromRows(2, 2, {2, 1, 1, 2}), Matrix::FromRows(1, 2, {1, 1}));
    CHECK(std::abs(x(0, 0) - 1.0 / 3) < 1e-12 && std::abs(x(0, 1) - 1.0 / 3) < 1e-12);
    CHECK(throws<NumericalError>([] { nnls_rowwise(Matrix::Identity(2, 2), Matrix::FromRows(1, 2, {3, 4}), 1, 1); }));
  }
  // test_kernels.cpp:133-154 — economy_svd of a diagonal and of a zero matrix
  {
    EconomySvd svd = economy_svd(Matrix::FromRows(2, 2, {3, 0, 0, 2}));
    CHECK(svd.sigma.size() == 2 && std::abs(svd.sigma[0] - 3.0) < 1e-12 && std::abs(svd.sigma[1] - 2.0) < 1e-12);
    for (Index c = 0; c < 2; ++c) CHECK(std::abs(std::abs(svd.P(c, c)) - 1.0) < 1e-12);
    EconomySvd z = economy_svd(Matrix::Zero(2, 3));
    CHECK(z.sigma.size() == 2 && z.sigma[0] == 0.0 && z.sigma[1] == 0.0 && z.P(0, 0) == 1.0 && z.Z(1, 1) == 1.0);
  }
  // test_cp.cpp:77-94 — rank-1 closed form
  {
    auto Y = ProjectedSlices::from_dense(2, {Matrix::FromRows(1, 2, {2, 4})});
    CpFactors f{Matrix::Ones(1, 1), Matrix::Ones(2, 1), Matrix::Ones(1, 1), Vector(1, 1.0)};
    CpFactors o = cp_als_iteration(Y, f);
    const double s5 = std::sqrt(5.0);
    CHECK(std::abs(o.H(0, 0) - 1.0) < 1e-12 && std::abs(o.V(0, 0) - 1 / s5) < 1e-12 &&
          std::abs(o.V(1, 0) - 2 / s5) < 1e-12 && std::abs(o.W(0, 0) - 2 * s5) < 1e-12);
  }
  // test_solver.cpp:173-180 — degenerate target still orthonormal, = I block
  {
    SparseSlice xs = SparseSlice::from_triplets(4, 3, {{2, 1, 5.0}});
    Matrix q = procrustes_update(xs, Matrix::Identity(2, 2), Vector(2, 1.0), Matrix::Zero(3, 2));
    CHECK(q.rows() == 4 && q.cols() == 2);
    CHECK((q.transpose() * q - Matrix::Identity(2, 2)).norm() < 1e-12);
  }
  // test_solver.cpp:216-280 — one iteration stop, invariants, residual identity
  {
    Rng rng(49);
    auto x = random_tensor(rng, 5, 6, 3, 8, 0.5);
    SolverConfig cfg;
    cfg.rank = 2;
    cfg.tol = std::numeric_limits<double>::infinity();
    cfg.max_iters = 50;
    auto [f, tr] = fit_parafac2(x, cfg);
    CHECK(tr.iterations.size() == 1 && tr.converged && f.Q.size() == 5);
    for (const Matrix& qk : f.Q) CHECK((qk.transpose() * qk - Matrix::Identity(2, 2)).norm() < 1e-8);
    CHECK(std::abs(tr.iterations[0].residual_sq - dense_residual(x, f)) <= 1e-9 * std::max(1.0, dense_residual(x, f)));
    Rng rng2(51);
    auto x2 = random_tensor(rng2, 4, 6, 3, 7, 1.0);
    SolverConfig c2;
    c2.rank = 2;
    c2.max_iters = 8;
    c2.tol = 1e-14;
    std::vector<double> eff, direct;
    fit_parafac2(x2, c2, [&](const Parafac2Factors& s, const IterationStats& st) {
      eff.push_back(st.residual_sq);
      direct.push_back(dense_residual(x2, s));
    });
    CHECK(!eff.empty());
    for (std::size_t i = 0; i < eff.size(); ++i) CHECK(std::abs(eff[i] - direct[i]) <= 1e-9 * std::max(1.0, direct[i]));
    for (std::size_t i = 1; i < eff.size(); ++i) CHECK(eff[i] <= eff[i - 1] + 1e-7 * std::max(1.0, eff[i - 1]));
  }
  // test_solver.cpp:86-120, 300-319 — error semantics
  {
    Rng rng(42);
    auto x = random_tensor(rng, 3, 4, 2, 3, 1.0);
    SolverConfig c;
    c.rank = 5;
    CHECK(throws<DataError>([&] { fit_parafac2(x, c); }));
    c.rank = 4;
    CHECK(throws<DataError>([&] { fit_parafac2(x, c); }));
    c.rank = 0;
    CHECK(throws<std::invalid_argument>([&] { fit_parafac2(x, c); }));
    auto empty = IrregularTensor::from_slices(3, {SparseSlice::from_triplets(3, 3, {}), SparseSlice::from_triplets(2, 3, {})});
    SolverConfig c1;
    CHECK(throws<DataError>([&] { fit_parafac2(empty, c1); }));
    auto big = IrregularTensor::from_slices(
        2, {SparseSlice::from_triplets(2, 2, {{0, 0, 1e200}, {0, 1, 1e200}, {1, 0, 1e200}, {1, 1, 1e200}})});
    SolverConfig c3;
    c3.rank = 2;
    c3.max_iters = 10;
    CHECK(throws<NumericalError>([&] { fit_parafac2(big, c3); }));
  }
  std::printf("dropin_test: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
