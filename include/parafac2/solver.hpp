// Drop-in replacement for /root/reference/proj/include/parafac2/solver.hpp.
// fit_parafac2 runs the whole PARAFAC2-ALS loop on the GPU (p2g_fit); the
// per-subject entry points (procrustes_update, project_slice(s)) go through
// the C-ABI parity hooks.  Same types, names, argument meaning and exception
// types as the reference.
#pragma once

#include <chrono>
#include <functional>

#include "cp.hpp"

namespace parafac2 {

struct SolverConfig {
  enum class Init { random, eye };
  Index rank = 1;
  int max_iters = 200;
  double tol = 1e-8;
  bool nonneg = true;
  Init init = Init::random;
  std::uint64_t seed = 0;
  int threads = 1;  // host-only in the reference; ignored on the GPU path
};

struct Parafac2Factors {
  std::vector<Matrix> Q;
  Matrix H, S, V;
  Index rank = 0;
};

struct IterationStats {
  int iter = 0;
  double residual_sq = 0;
  double fit = 0;
  double ms_procrustes = 0;  // device-timed (CUDA events): Procrustes + fused mode-1 partial
  double ms_project = 0;     // 0: the device loop is Q-based and never forms Y_k
  double ms_cp = 0;          // MTTKRP modes 2-3, H/V/W updates, fit scalars
};

struct FitTrace {
  std::vector<IterationStats> iterations;
  double total_ms = 0;
  bool converged = false;
};

using IterationObserver = std::function<void(const Parafac2Factors&, const IterationStats&)>;

namespace detail {
inline void load(p2g_ctx* ctx, const IrregularTensor& X) {
  const Csr c = X.to_csr();
  check(p2g_load_csr(ctx, c.K, c.J, c.subj_row_ptr.data(), c.row_ptr.data(), c.col_idx.data(), c.val.data()));
}
inline std::vector<Matrix> unpack_q(const IrregularTensor& X, const std::vector<double>& Qp, Index R) {
  std::vector<Matrix> Q;
  std::size_t row = 0;
  for (Index k = 0; k < X.n_slices(); ++k) {
    Matrix q(X.slice(k).n_rows(), R);
    for (Index i = 0; i < q.rows(); ++i, ++row)
      for (Index r = 0; r < R; ++r) q(i, r) = Qp[row * static_cast<std::size_t>(R) + static_cast<std::size_t>(r)];
    Q.push_back(std::move(q));
  }
  return Q;
}
}  // namespace detail

/// solver.hpp:104-166 (random initialisation on the host, eye initialisation
/// on the device: p2g_initialize_eye).
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
  f.H = Matrix(R, R);
  f.S = Matrix(X.n_slices(), R);
  f.V = Matrix(X.n_cols(), R);
  check(p2g_initialize_random(cfg.seed, X.n_slices(), X.n_cols(), static_cast<int32_t>(R), f.H.data(), f.S.data(),
                              f.V.data()));
  if (cfg.init == SolverConfig::Init::eye) {
    p2g_ctx* ctx = Device::get().ctx();
    detail::load(ctx, X);
    check(p2g_initialize_eye(ctx, static_cast<int32_t>(R), f.V.data()));
  }
  return f;
}

/// solver.hpp:173-193 for one subject (canonical rule D5 for rank-deficient
/// targets).
inline Matrix procrustes_update(const SparseSlice& Xk, const Matrix& H, const Vector& s, const Matrix& V) {
  const Index R = H.rows();
  if (H.cols() != R) throw std::invalid_argument("H must be square");
  if (static_cast<Index>(s.size()) != R || V.cols() != R || V.rows() != Xk.n_cols())
    throw std::invalid_argument("procrustes factors have mismatched shapes");
  if (Xk.n_rows() < R) throw std::invalid_argument("rank exceeds observations in procrustes step");
  p2g_ctx* ctx = Device::get().ctx();
  detail::load(ctx, IrregularTensor::from_slices(Xk.n_cols(), {Xk}));
  Matrix W(1, R);
  for (Index r = 0; r < R; ++r) W(0, r) = s[static_cast<std::size_t>(r)];
  std::vector<double> Qp(static_cast<std::size_t>(Xk.n_rows() * R));
  check(p2g_procrustes(ctx, static_cast<int32_t>(R), H.data(), V.data(), W.data(), Qp.data(), nullptr, nullptr));
  Matrix Q(Xk.n_rows(), R);
  for (Index i = 0; i < Q.rows(); ++i)
    for (Index r = 0; r < R; ++r) Q(i, r) = Qp[static_cast<std::size_t>(i * R + r)];
  return Q;
}

/// solver.hpp:212-235
inline ProjectedSlices project_slices(const IrregularTensor& X, const std::vector<Matrix>& Q, int /*threads*/ = 1) {
  if (static_cast<Index>(Q.size()) != X.n_slices()) throw std::invalid_argument("projection: one Q_k per slice required");
  const Index R = Q.empty() ? 0 : Q.front().cols();
  p2g_ctx* ctx = Device::get().ctx();
  detail::load(ctx, X);
  std::vector<double> Qp;
  for (Index k = 0; k < X.n_slices(); ++k) {
    const Matrix& q = Q[static_cast<std::size_t>(k)];
    if (q.rows() != X.slice(k).n_rows()) throw std::invalid_argument("projection: Q_k row count mismatch");
    for (Index i = 0; i < q.rows(); ++i)
      for (Index r = 0; r < R; ++r) Qp.push_back(q(i, r));
  }
  std::vector<std::int64_t> ptr(static_cast<std::size_t>(X.n_slices() + 1));
  check(p2g_project(ctx, static_cast<int32_t>(R), nullptr, ptr.data(), nullptr, nullptr));
  std::vector<std::int32_t> cols(static_cast<std::size_t>(std::max<std::int64_t>(ptr.back(), 1)));
  std::vector<double> Y(static_cast<std::size_t>(std::max<std::int64_t>(ptr.back() * R, 1)));
  check(p2g_project(ctx, static_cast<int32_t>(R), Qp.data(), ptr.data(), cols.data(), Y.data()));
  std::vector<Matrix> packed;
  std::vector<std::vector<Index>> cl;
  for (Index k = 0; k < X.n_slices(); ++k) {
    const std::int64_t c0 = ptr[static_cast<std::size_t>(k)], c1 = ptr[static_cast<std::size_t>(k + 1)];
    Matrix b(R, c1 - c0);
    std::memcpy(b.data(), Y.data() + c0 * R, sizeof(double) * static_cast<std::size_t>((c1 - c0) * R));
    packed.push_back(std::move(b));
    cl.emplace_back(cols.begin() + c0, cols.begin() + c1);
  }
  return ProjectedSlices::from_packed(R, X.n_cols(), std::move(packed), std::move(cl));
}

/// solver.hpp:197-208
inline Matrix project_slice(const SparseSlice& Xk, const Matrix& Qk) {
  if (Qk.rows() != Xk.n_rows()) throw std::invalid_argument("projection: Q_k row count mismatch");
  return project_slices(IrregularTensor::from_slices(Xk.n_cols(), {Xk}), {Qk}).packed(0);
}

/// solver.hpp:238-243
inline std::vector<Matrix> assemble_U(const Parafac2Factors& f) {
  std::vector<Matrix> U;
  for (const Matrix& Qk : f.Q) U.push_back(Qk * f.H);
  return U;
}

/// solver.hpp:251-321.  Without an observer the whole loop runs on the GPU in
/// one call; with an observer each iteration is one call seeded with the
/// previous factors (the observer needs every Q_k on the host).
inline std::pair<Parafac2Factors, FitTrace> fit_parafac2(const IrregularTensor& X, const SolverConfig& config,
                                                         const IterationObserver& observer = nullptr) {
  const auto t0 = std::chrono::steady_clock::now();
  Parafac2Factors state = initialize(X, config);
  const Index R = config.rank;
  p2g_ctx* ctx = Device::get().ctx();
  detail::load(ctx, X);
  FitTrace trace;
  std::vector<double> Qp(static_cast<std::size_t>(X.to_csr().subj_row_ptr.back() * R));
  std::vector<double> phases;
  auto run = [&](int iters, bool explicit_init, std::vector<double>& fit, std::vector<double>& res,
                 std::vector<double>& ms, p2g_fit_summary& sum) {
    // initialize() above already produced the reference's initial state
    // (random or eye): the loop always starts from it
    (void)explicit_init;
    p2g_fit_config c{static_cast<int32_t>(R), iters, config.tol, config.nonneg ? 1 : 0, 2, config.seed};
    fit.assign(static_cast<std::size_t>(iters), 0.0);
    res.assign(static_cast<std::size_t>(iters), 0.0);
    ms.assign(static_cast<std::size_t>(iters), 0.0);
    Matrix H = state.H, V = state.V, S = state.S;
    check(p2g_fit(ctx, &c, H.data(), V.data(), S.data(), state.H.data(), state.V.data(), state.S.data(), Qp.data(),
                  nullptr, fit.data(), res.data(), ms.data(), &sum));
    phases.assign(static_cast<std::size_t>(3 * iters), 0.0);
    int32_t np = 0;
    check(p2g_fit_phase_ms(ctx, iters, phases.data(), &np));
  };
  auto stats = [&](IterationStats& st, int i) {  // IterationStats timers (solver.hpp:278-297), device-timed
    st.ms_procrustes = phases[static_cast<std::size_t>(3 * i)];
    st.ms_project = phases[static_cast<std::size_t>(3 * i + 1)];
    st.ms_cp = phases[static_cast<std::size_t>(3 * i + 2)];
  };
  std::vector<double> fit, res, ms;
  p2g_fit_summary sum{};
  if (!observer) {
    run(config.max_iters, false, fit, res, ms, sum);
    for (int i = 0; i < sum.iterations; ++i) {
      IterationStats st;
      st.iter = i + 1;
      st.fit = fit[static_cast<std::size_t>(i)];
      st.residual_sq = res[static_cast<std::size_t>(i)];
      stats(st, i);
      trace.iterations.push_back(st);
    }
    trace.converged = sum.converged != 0;
  } else {
    double prev = 0.0;
    for (int it = 1; it <= config.max_iters; ++it) {
      run(1, true, fit, res, ms, sum);
      IterationStats st;
      st.iter = it;
      st.fit = fit[0];
      st.residual_sq = res[0];
      stats(st, 0);
      trace.iterations.push_back(st);
      state.Q = detail::unpack_q(X, Qp, R);
      observer(state, st);
      const double change = std::abs(st.fit - prev) / std::max(prev, std::numeric_limits<double>::epsilon());
      prev = st.fit;
      if (change < config.tol) {
        trace.converged = true;
        break;
      }
    }
  }
  state.Q = detail::unpack_q(X, Qp, R);
  trace.total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return {std::move(state), std::move(trace)};
}

}  // namespace parafac2
