// pybind11 bindings of the CPU oracle (p2_oracle.hpp) for tests/ and the
// bench.py cpu_baseline / --impl reference legs.  TEST INFRASTRUCTURE ONLY:
// the product path never imports this module.
#include <pybind11/functional.h>
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include "baseline_gen.hpp"
#include "p2_oracle.hpp"

namespace py = pybind11;
using namespace p2o;

using F64 = py::array_t<double, py::array::c_style | py::array::forcecast>;
using I64 = py::array_t<std::int64_t, py::array::c_style | py::array::forcecast>;
using I32 = py::array_t<std::int32_t, py::array::c_style | py::array::forcecast>;

static Mat to_mat(const F64& a) {
  if (a.ndim() == 1) {
    Mat m(a.shape(0), 1);
    for (Index i = 0; i < a.shape(0); ++i) m(i, 0) = a.at(i);
    return m;
  }
  if (a.ndim() != 2) throw std::invalid_argument("expected a 2-D array");
  Mat m(a.shape(0), a.shape(1));
  auto r = a.unchecked<2>();
  for (Index i = 0; i < m.rows(); ++i)
    for (Index j = 0; j < m.cols(); ++j) m(i, j) = r(i, j);
  return m;
}

static py::array_t<double> from_mat(const Mat& m) {
  py::array_t<double> out({m.rows(), m.cols()});
  auto w = out.mutable_unchecked<2>();
  for (Index i = 0; i < m.rows(); ++i)
    for (Index j = 0; j < m.cols(); ++j) w(i, j) = m(i, j);
  return out;
}

static Vec to_vec(const F64& a) {
  Vec v(static_cast<std::size_t>(a.size()));
  for (Index i = 0; i < a.size(); ++i) v[static_cast<std::size_t>(i)] = a.data()[i];
  return v;
}

static py::array_t<double> from_vec(const Vec& v) {
  py::array_t<double> out(static_cast<py::ssize_t>(v.size()));
  std::copy(v.begin(), v.end(), out.mutable_data());
  return out;
}

/// Flattened CSR (the GPU layout) -> per-subject slices.
/// Within a row, entries keep their CSR order; from_triplets re-sorts by
/// (col,row) exactly as the reference does.
static IrregularTensor tensor_from_csr(Index J, const I64& subj_row_ptr, const I64& row_ptr, const I32& col_idx,
                                       const F64& val) {
  const Index K = subj_row_ptr.size() - 1;
  std::vector<SparseSlice> slices;
  slices.reserve(static_cast<std::size_t>(K));
  const auto* srp = subj_row_ptr.data();
  const auto* rp = row_ptr.data();
  const auto* ci = col_idx.data();
  const auto* v = val.data();
  std::vector<Triplet> t;
  for (Index k = 0; k < K; ++k) {
    t.clear();
    const Index r0 = srp[k], r1 = srp[k + 1];
    for (Index r = r0; r < r1; ++r)
      for (std::int64_t p = rp[r]; p < rp[r + 1]; ++p) t.push_back({r - r0, static_cast<Index>(ci[p]), v[p]});
    slices.push_back(SparseSlice::from_triplets(r1 - r0, J, t));
  }
  return IrregularTensor::from_slices(J, std::move(slices));
}

/// Per-subject CSC -> flattened CSR (rows ascending, columns ascending in a row).
static py::tuple tensor_to_csr(const IrregularTensor& X) {
  const Index K = X.n_slices();
  std::vector<std::int64_t> srp(static_cast<std::size_t>(K + 1), 0);
  for (Index k = 0; k < K; ++k) srp[static_cast<std::size_t>(k + 1)] = srp[static_cast<std::size_t>(k)] + X.slice(k).n_rows();
  const Index NR = srp.back();
  std::vector<std::int64_t> rp(static_cast<std::size_t>(NR + 1), 0);
  for (Index k = 0; k < K; ++k) {
    const SparseSlice& s = X.slice(k);
    for (Index p = 0; p < s.nnz(); ++p) rp[static_cast<std::size_t>(srp[static_cast<std::size_t>(k)] + s.entry_row(p) + 1)]++;
  }
  for (Index r = 0; r < NR; ++r) rp[static_cast<std::size_t>(r + 1)] += rp[static_cast<std::size_t>(r)];
  const Index nnz = rp.back();
  std::vector<std::int64_t> fill(rp.begin(), rp.end() - 1);
  py::array_t<std::int32_t> ci(nnz);
  py::array_t<double> va(nnz);
  auto* cip = ci.mutable_data();
  auto* vap = va.mutable_data();
  for (Index k = 0; k < K; ++k) {
    const SparseSlice& s = X.slice(k);
    for (Index c = 0; c < s.n_nnz_cols(); ++c) {  // column ascending -> row-wise ascending columns
      auto [p0, p1] = s.col_range(c);
      for (Index p = p0; p < p1; ++p) {
        const std::size_t r = static_cast<std::size_t>(srp[static_cast<std::size_t>(k)] + s.entry_row(p));
        const std::int64_t dst = fill[r]++;
        cip[dst] = static_cast<std::int32_t>(s.col(c));
        vap[dst] = s.entry_value(p);
      }
    }
  }
  return py::make_tuple(X.n_cols(), py::array_t<std::int64_t>(srp.size(), srp.data()),
                        py::array_t<std::int64_t>(rp.size(), rp.data()), ci, va);
}

/// Q_k list (I_k x R) <-> packed row-major (sum I_k) x R (the C-ABI layout).
static py::array_t<double> pack_q(const std::vector<Mat>& Q, Index R) {
  Index n = 0;
  for (const Mat& q : Q) n += q.rows();
  py::array_t<double> out({n, R});
  auto w = out.mutable_unchecked<2>();
  Index row = 0;
  for (const Mat& q : Q)
    for (Index i = 0; i < q.rows(); ++i, ++row)
      for (Index r = 0; r < R; ++r) w(row, r) = q(i, r);
  return out;
}

static std::vector<Mat> unpack_q(const IrregularTensor& X, const F64& Qp) {
  std::vector<Mat> Q;
  auto r = Qp.unchecked<2>();
  Index row = 0;
  const Index R = Qp.shape(1);
  for (Index k = 0; k < X.n_slices(); ++k) {
    Mat q(X.slice(k).n_rows(), R);
    for (Index i = 0; i < q.rows(); ++i, ++row)
      for (Index c = 0; c < R; ++c) q(i, c) = r(row, c);
    Q.push_back(std::move(q));
  }
  return Q;
}

/// ProjectedSlices <-> (rank, J, list of R x c_k blocks, list of col lists).
static ProjectedSlices projected_from_py(Index rank, Index J, const std::vector<F64>& blocks,
                                         const std::vector<std::vector<Index>>& cols) {
  std::vector<Mat> packed;
  for (const auto& b : blocks) packed.push_back(to_mat(b));
  for (std::size_t k = 0; k < packed.size(); ++k)  // allow (R, 0) blocks given as empty
    if (packed[k].size() == 0) packed[k] = Mat(rank, 0);
  return ProjectedSlices::from_packed(rank, J, std::move(packed), cols);
}

static py::dict projected_to_py(const ProjectedSlices& Y) {
  py::list blocks, cols;
  for (Index k = 0; k < Y.n_slices(); ++k) {
    blocks.append(from_mat(Y.packed(k)));
    cols.append(Y.cols(k));
  }
  py::dict d;
  d["rank"] = Y.rank();
  d["n_cols"] = Y.n_cols();
  d["blocks"] = blocks;
  d["cols"] = cols;
  return d;
}

static SolverConfig make_cfg(Index rank, int max_iters, double tol, bool nonneg, const std::string& init,
                             std::uint64_t seed, int threads) {
  SolverConfig c;
  c.rank = rank;
  c.max_iters = max_iters;
  c.tol = tol;
  c.nonneg = nonneg;
  c.init = init == "eye" ? SolverConfig::Init::eye : SolverConfig::Init::random;
  c.seed = seed;
  c.threads = threads;
  return c;
}

PYBIND11_MODULE(p2oracle, m) {
  m.doc() = "CPU fp64 oracle restating /root/reference/proj/include/parafac2 (test infrastructure only)";

  py::register_exception<DataError>(m, "DataError", PyExc_RuntimeError);
  py::register_exception<NumericalError>(m, "NumericalError", PyExc_ArithmeticError);

  py::class_<Rng>(m, "Rng")
      .def(py::init<std::uint64_t>())
      .def("next_u64", &Rng::next_u64)
      .def("uniform", py::overload_cast<>(&Rng::uniform))
      .def("uniform_range", py::overload_cast<double, double>(&Rng::uniform))
      .def("normal", &Rng::normal)
      .def("below", &Rng::below);
  m.def("substream_seed", &substream_seed);
  // BASELINE workload, oracle side: (J, subj_row_ptr, row_ptr, col_idx, val) of the first
  // K subjects of config `config_id` at rank R (K <= 0: all), and the D2 initial factors.
  m.def(
      "baseline_generate",
      [](int config_id, int R, std::int64_t K, int threads) {
        const baseline::Spec s = baseline::config(config_id, R);
        baseline::Csr c;
        {
          py::gil_scoped_release rel;
          c = baseline::generate(s, K, threads);
        }
        return py::make_tuple(c.J, py::array_t<std::int64_t>(c.subj_row_ptr.size(), c.subj_row_ptr.data()),
                              py::array_t<std::int64_t>(c.row_ptr.size(), c.row_ptr.data()),
                              py::array_t<std::int32_t>(c.col_idx.size(), c.col_idx.data()),
                              py::array_t<double>(c.val.size(), c.val.data()));
      },
      py::arg("config_id"), py::arg("R"), py::arg("K") = 0, py::arg("threads") = 1);
  m.def(
      "baseline_spec",
      [](int config_id, int R) {
        const baseline::Spec s = baseline::config(config_id, R);
        py::dict d;
        d["K"] = s.K;
        d["J"] = s.J;
        d["seed"] = s.seed;
        return d;
      },
      py::arg("config_id"), py::arg("R"));
  m.def(
      "baseline_init",
      [](std::uint64_t seed, std::int64_t K, std::int64_t J, int R, std::int64_t K_use) {
        std::vector<double> H, V, W;
        baseline::init_factors(seed, K, K_use, J, R, H, V, W);
        if (K_use <= 0 || K_use > K) K_use = K;
        // column-major buffers -> (rows, cols) arrays
        auto colmajor = [](const std::vector<double>& a, std::int64_t rows, std::int64_t cols) {
          py::array_t<double> out({rows, cols});
          auto w = out.mutable_unchecked<2>();
          for (std::int64_t c = 0; c < cols; ++c)
            for (std::int64_t r = 0; r < rows; ++r) w(r, c) = a[static_cast<std::size_t>(c * rows + r)];
          return out;
        };
        return py::make_tuple(colmajor(H, R, R), colmajor(V, J, R), colmajor(W, K_use, R));
      },
      py::arg("seed"), py::arg("K"), py::arg("J"), py::arg("R"), py::arg("K_use") = 0);

  m.def("partition_even", &partition_even);
  m.def("partition_weighted", &partition_weighted);

  py::class_<IrregularTensor>(m, "Tensor")
      .def_static("from_csr", &tensor_from_csr, py::arg("J"), py::arg("subj_row_ptr"), py::arg("row_ptr"),
                  py::arg("col_idx"), py::arg("val"))
      .def_static("from_triplets",
                  [](Index J, const std::vector<std::tuple<Index, std::vector<std::tuple<Index, Index, double>>>>& sl) {
                    std::vector<SparseSlice> slices;
                    for (const auto& [rows, trip] : sl) {
                      std::vector<Triplet> t;
                      for (const auto& [i, j, v] : trip) t.push_back({i, j, v});
                      slices.push_back(SparseSlice::from_triplets(rows, J, t));
                    }
                    return IrregularTensor::from_slices(J, std::move(slices));
                  })
      .def("to_csr", &tensor_to_csr)
      .def_property_readonly("n_slices", &IrregularTensor::n_slices)
      .def_property_readonly("n_cols", &IrregularTensor::n_cols)
      .def_property_readonly("total_nnz", &IrregularTensor::total_nnz)
      .def_property_readonly("max_rows", &IrregularTensor::max_rows)
      .def("slice_dense", [](const IrregularTensor& X, Index k) { return from_mat(X.slice(k).dense()); })
      .def("slice_rows", [](const IrregularTensor& X, Index k) { return X.slice(k).n_rows(); })
      .def("slice_nnz_cols", [](const IrregularTensor& X, Index k) { return X.slice(k).nnz_cols(); })
      .def("frobenius_sq", [](const IrregularTensor& X) { return frobenius_sq(X); });

  // --- dense kernels -------------------------------------------------------
  m.def("gram", [](const F64& a) { return from_mat(gram(to_mat(a))); });
  m.def("hadamard", [](const F64& a, const F64& b) { return from_mat(hadamard(to_mat(a), to_mat(b))); });
  m.def("khatri_rao", [](const F64& a, const F64& b) { return from_mat(khatri_rao(to_mat(a), to_mat(b))); });
  m.def("pinv_small", [](const F64& a) { return from_mat(pinv_small(to_mat(a))); });
  m.def("sym_eig", [](const F64& a) {
    const SymEig e = sym_eig(to_mat(a));
    return py::make_tuple(from_vec(e.values), from_mat(e.vectors));
  });
  m.def("economy_svd", [](const F64& a) {
    const EconomySvd s = economy_svd(to_mat(a));
    return py::make_tuple(from_mat(s.P), from_vec(s.sigma), from_mat(s.Z));
  });
  m.def("canonical_polar", [](const F64& a) {
    PolarInfo pi;
    const Mat q = canonical_polar(to_mat(a), &pi);
    return py::make_tuple(from_mat(q), pi.flag, pi.rho, pi.lambda_ratio);
  });
  m.def(
      "nnls_rowwise",
      [](const F64& g, const F64& b, int threads, int max_iter) {
        return from_mat(nnls_rowwise(to_mat(g), to_mat(b), threads, max_iter));
      },
      py::arg("G"), py::arg("B"), py::arg("threads") = 1, py::arg("max_iter") = 0);
  m.def("random_orthonormal",
        [](Rng& rng, Index rows, Index cols) { return from_mat(random_orthonormal(rng, rows, cols)); });
  m.def("random_matrix",
        [](Rng& rng, Index rows, Index cols, double lo, double hi) {
          return from_mat(fixtures::random_matrix(rng, rows, cols, lo, hi));
        },
        py::arg("rng"), py::arg("rows"), py::arg("cols"), py::arg("lo") = -1.0, py::arg("hi") = 1.0);
  m.def("random_tensor", &fixtures::random_tensor, py::arg("rng"), py::arg("n_slices"), py::arg("n_cols"),
        py::arg("min_rows"), py::arg("max_rows"), py::arg("density"), py::arg("lo") = -1.0, py::arg("hi") = 1.0);
  m.def("random_slice_tensor",
        [](Rng& rng, Index rows, Index cols, double density, double lo, double hi) {
          std::vector<SparseSlice> s{fixtures::random_slice(rng, rows, cols, density, lo, hi)};
          return IrregularTensor::from_slices(cols, std::move(s));
        },
        py::arg("rng"), py::arg("rows"), py::arg("cols"), py::arg("density"), py::arg("lo") = -1.0,
        py::arg("hi") = 1.0);
  m.def("random_projected",
        [](Rng& rng, Index rank, Index n_cols, Index n_slices, double density, double lo, double hi) {
          return projected_to_py(fixtures::random_projected(rng, rank, n_cols, n_slices, density, lo, hi));
        },
        py::arg("rng"), py::arg("rank"), py::arg("n_cols"), py::arg("n_slices"), py::arg("density"),
        py::arg("lo") = -1.0, py::arg("hi") = 1.0);
  m.def("generate_synthetic", [](Index subjects, Index cols, Index max_rows, Index rank, double density,
                                 std::uint64_t seed, bool nonneg) {
    GeneratorSpec s{subjects, cols, max_rows, rank, density, seed, nonneg};
    GeneratedTensor g = generate_synthetic(s);
    return py::make_tuple(std::move(g.tensor), g.dropped_subjects);
  });

  // --- MTTKRP on packed projected slices -------------------------------------
  m.def("mttkrp",
        [](Index rank, Index J, const std::vector<F64>& blocks, const std::vector<std::vector<Index>>& cols,
           const F64& H, const F64& V, const F64& W, int mode, int threads) {
          const ProjectedSlices Y = projected_from_py(rank, J, blocks, cols);
          return from_mat(mttkrp(Y, to_mat(H), to_mat(V), to_mat(W), mode, threads));
        },
        py::arg("rank"), py::arg("J"), py::arg("blocks"), py::arg("cols"), py::arg("H"), py::arg("V"), py::arg("W"),
        py::arg("mode"), py::arg("threads") = 1);
  m.def("naive_mttkrp", [](Index rank, Index J, const std::vector<F64>& blocks,
                           const std::vector<std::vector<Index>>& cols, const F64& H, const F64& V, const F64& W,
                           int mode) {
    const ProjectedSlices Y = projected_from_py(rank, J, blocks, cols);
    return from_mat(naive_mttkrp(Y, to_mat(H), to_mat(V), to_mat(W), mode));
  });
  m.def("naive_mttkrp_bytes", &naive_mttkrp_bytes);
  m.def("cp_als_iteration",
        [](Index rank, Index J, const std::vector<F64>& blocks, const std::vector<std::vector<Index>>& cols,
           const F64& H, const F64& V, const F64& W, bool nonneg, bool normalize_w, int threads) {
          const ProjectedSlices Y = projected_from_py(rank, J, blocks, cols);
          CpFactors f{to_mat(H), to_mat(V), to_mat(W), Vec(static_cast<std::size_t>(rank), 1.0)};
          Mat m3;
          CpStepDump d;
          CpFactors o = cp_als_iteration(Y, f, CpOptions{nonneg, normalize_w, threads}, &m3, &d);
          py::dict r;
          r["H"] = from_mat(o.H);
          r["V"] = from_mat(o.V);
          r["W"] = from_mat(o.W);
          r["lambda"] = from_vec(o.lambda);
          r["m1"] = from_mat(d.m1);
          r["m2"] = from_mat(d.m2);
          r["m3"] = from_mat(d.m3);
          r["norm_h"] = from_vec(d.norm_h);
          r["norm_v"] = from_vec(d.norm_v);
          return r;
        },
        py::arg("rank"), py::arg("J"), py::arg("blocks"), py::arg("cols"), py::arg("H"), py::arg("V"), py::arg("W"),
        py::arg("nonneg") = true, py::arg("normalize_w") = false, py::arg("threads") = 1);
  m.def("cp_objective", [](Index rank, Index J, const std::vector<F64>& blocks,
                           const std::vector<std::vector<Index>>& cols, const F64& H, const F64& V, const F64& W,
                           const F64& lambda) {
    const ProjectedSlices Y = projected_from_py(rank, J, blocks, cols);
    CpFactors f{to_mat(H), to_mat(V), to_mat(W), to_vec(lambda)};
    return cp_objective(Y, f);
  });
  m.def("dense_cp_objective", [](Index rank, Index J, const std::vector<F64>& blocks,
                                 const std::vector<std::vector<Index>>& cols, const F64& H, const F64& V,
                                 const F64& W, const F64& lambda) {
    const ProjectedSlices Y = projected_from_py(rank, J, blocks, cols);
    CpFactors f{to_mat(H), to_mat(V), to_mat(W), to_vec(lambda)};
    return fixtures::dense_cp_objective(Y, f);
  });

  // --- solver pieces ---------------------------------------------------------
  m.def("procrustes_update", [](const IrregularTensor& X, Index k, const F64& H, const F64& s, const F64& V) {
    PolarInfo pi;
    const Mat q = procrustes_update(X.slice(k), to_mat(H), to_vec(s), to_mat(V), &pi);
    return py::make_tuple(from_mat(q), pi.flag, pi.lambda_ratio);
  });
  m.def(
      "procrustes_all",
      [](const IrregularTensor& X, const F64& H, const F64& V, const F64& W, int threads) {
        const Mat h = to_mat(H), v = to_mat(V), w = to_mat(W);
        const Index K = X.n_slices(), R = h.rows();
        std::vector<Mat> Q(static_cast<std::size_t>(K));
        std::vector<int> flags(static_cast<std::size_t>(K));
        std::vector<double> ratio(static_cast<std::size_t>(K));
        std::vector<std::uint64_t> wt(static_cast<std::size_t>(K));
        for (Index k = 0; k < K; ++k) wt[static_cast<std::size_t>(k)] = X.slice(k).nnz() + X.slice(k).n_rows();
        {
          py::gil_scoped_release rel;
          run_chunks(partition_weighted(wt, threads), [&](std::size_t, Index b, Index e) {
            Vec s(static_cast<std::size_t>(R));
            for (Index k = b; k < e; ++k) {
              for (Index r = 0; r < R; ++r) s[static_cast<std::size_t>(r)] = w(k, r);
              PolarInfo pi;
              Q[static_cast<std::size_t>(k)] = procrustes_update(X.slice(k), h, s, v, &pi);
              flags[static_cast<std::size_t>(k)] = pi.flag;
              ratio[static_cast<std::size_t>(k)] = pi.lambda_ratio;
            }
          });
        }
        return py::make_tuple(pack_q(Q, R), py::array_t<int>(flags.size(), flags.data()),
                              py::array_t<double>(ratio.size(), ratio.data()));
      },
      py::arg("X"), py::arg("H"), py::arg("V"), py::arg("W"), py::arg("threads") = 1);
  m.def(
      "project_slices",
      [](const IrregularTensor& X, const F64& Qp, int threads) {
        return projected_to_py(project_slices(X, unpack_q(X, Qp), threads));
      },
      py::arg("X"), py::arg("Q"), py::arg("threads") = 1);
  m.def("initialize", [](const IrregularTensor& X, Index rank, int max_iters, double tol, bool nonneg,
                         const std::string& init, std::uint64_t seed) {
    const Parafac2Factors f = initialize(X, make_cfg(rank, max_iters, tol, nonneg, init, seed, 1));
    return py::make_tuple(from_mat(f.H), from_mat(f.S), from_mat(f.V));
  });
  m.def("dense_residual", [](const IrregularTensor& X, const F64& Qp, const F64& H, const F64& S, const F64& V) {
    Parafac2Factors f;
    f.Q = unpack_q(X, Qp);
    f.H = to_mat(H);
    f.S = to_mat(S);
    f.V = to_mat(V);
    return fixtures::dense_residual(X, f);
  });
  m.def(
      "fit_parafac2",
      [](const IrregularTensor& X, Index rank, int max_iters, double tol, bool nonneg, const std::string& init,
         std::uint64_t seed, int threads, py::object H0, py::object V0, py::object W0, bool dumps,
         py::object observer) {
        const SolverConfig cfg = make_cfg(rank, max_iters, tol, nonneg, init, seed, threads);
        InitialFactors ini;
        const bool have_init = !H0.is_none();
        if (have_init) {
          ini.H = to_mat(H0.cast<F64>());
          ini.V = to_mat(V0.cast<F64>());
          ini.W = to_mat(W0.cast<F64>());
        }
        std::vector<IterationDump> dv;
        IterationObserver obs = nullptr;
        if (!observer.is_none()) {
          obs = [&](const Parafac2Factors& f, const IterationStats& s) {
            py::gil_scoped_acquire acq;
            observer(pack_q(f.Q, f.rank), from_mat(f.H), from_mat(f.S), from_mat(f.V), s.iter, s.residual_sq, s.fit);
          };
        }
        std::pair<Parafac2Factors, FitTrace> res;
        {
          py::gil_scoped_release rel;
          res = fit_parafac2(X, cfg, obs, have_init ? &ini : nullptr, dumps ? &dv : nullptr);
        }
        const auto& [f, tr] = res;
        py::dict r;
        r["Q"] = pack_q(f.Q, f.rank);
        r["H"] = from_mat(f.H);
        r["S"] = from_mat(f.S);
        r["V"] = from_mat(f.V);
        std::vector<double> fits, res2, msp, msj, msc, msv;
        std::vector<std::int64_t> ndef, ndeg;
        std::vector<double> minrat;
        for (const auto& s : tr.iterations) {
          fits.push_back(s.fit);
          res2.push_back(s.residual_sq);
          msp.push_back(s.ms_procrustes);
          msj.push_back(s.ms_project);
          msc.push_back(s.ms_cp);
          msv.push_back(s.ms_v_update);
          ndef.push_back(s.n_deficient);
          ndeg.push_back(s.n_degenerate);
          minrat.push_back(s.min_lambda_ratio);
        }
        r["fit"] = fits;
        r["residual_sq"] = res2;
        r["ms_procrustes"] = msp;
        r["ms_project"] = msj;
        r["ms_cp"] = msc;
        r["ms_v_update"] = msv;
        r["n_deficient"] = ndef;
        r["n_degenerate"] = ndeg;
        r["min_lambda_ratio"] = minrat;
        r["total_ms"] = tr.total_ms;
        r["converged"] = tr.converged;
        r["iterations"] = tr.iterations.size();
        if (dumps) {
          py::list dl;
          for (const auto& d : dv) {
            py::dict e;
            e["H_in"] = from_mat(d.H_in);
            e["V_in"] = from_mat(d.V_in);
            e["W_in"] = from_mat(d.W_in);
            e["Q"] = pack_q(d.Q, f.rank);
            e["flags"] = d.flags;
            e["m1"] = from_mat(d.cp.m1);
            e["m2"] = from_mat(d.cp.m2);
            e["m3"] = from_mat(d.cp.m3);
            e["norm_h"] = from_vec(d.cp.norm_h);
            e["norm_v"] = from_vec(d.cp.norm_v);
            e["H"] = from_mat(d.H);
            e["V"] = from_mat(d.V);
            e["W"] = from_mat(d.W);
            e["fit"] = d.fit;
            e["residual_sq"] = d.residual_sq;
            dl.append(e);
          }
          r["dumps"] = dl;
        }
        return r;
      },
      py::arg("X"), py::arg("rank"), py::arg("max_iters") = 200, py::arg("tol") = 1e-8, py::arg("nonneg") = true,
      py::arg("init") = "random", py::arg("seed") = 0, py::arg("threads") = 1, py::arg("H0") = py::none(),
      py::arg("V0") = py::none(), py::arg("W0") = py::none(), py::arg("dumps") = false,
      py::arg("observer") = py::none());
}
