"""GPU parity: every kernel through the C ABI against the CPU oracle.

Tolerances (north_star): per-step outputs (MTTKRPs, Q, factors) relative
Frobenius error <= 1e-9 when teacher-forced with oracle state; fit trajectory
|fit_gpu - fit_oracle| <= 1e-7 over 10 free-running iterations; integer
bookkeeping (partition, flags/deficiency counts) bit-exact.
"""
import numpy as np
import pytest

from tests.helpers import assert_q_close, oracle_from_csr, rel_err, rel_frob

pytestmark = pytest.mark.gpu

TOL_STEP = 1e-9
TOL_FIT = 1e-7


def canonical_flags(flags):
    """GPU flags in the oracle's vocabulary: P2G_FLAG_ACCURATE (2, full rank
    solved by the accurate path) is full rank (0); deficient (1) and
    degenerate (3) must match exactly."""
    f = np.array(flags, copy=True)
    f[f == 2] = 0
    return f


def proj(P):
    return P["rank"], P["n_cols"], P["blocks"], P["cols"]


# ---------------------------------------------------------------------------
# Boundary kernels on packed projected slices (mttkrp.hpp, kernels.hpp)
# ---------------------------------------------------------------------------
def test_packed_mode_kats(ctx):  # test_mttkrp.cpp:36-101 through the C ABI
    b, c = [np.array([[1.0, 0.0], [0.0, 2.0]])], [[0, 1]]
    w = np.array([[3.0, 5.0]])
    assert np.array_equal(ctx.mttkrp_packed(1, 2, 2, b, c, np.eye(2), np.ones((2, 2)), w), [[3, 5], [6, 10]])
    assert np.array_equal(ctx.mttkrp_packed(2, 2, 2, b, c, np.eye(2), np.ones((2, 2)), w), [[3, 0], [0, 10]])
    m = ctx.mttkrp_packed(2, 1, 3, [np.array([[4.0]]), np.array([[7.0]])], [[0], [2]], np.array([[1.0]]),
                          np.ones((3, 1)), np.array([[1.0], [10.0]]))
    assert m[0, 0] == 4 and m[1, 0] == 0 and m[2, 0] == 70
    m = ctx.mttkrp_packed(3, 2, 2, b, c, np.eye(2), np.ones((2, 2)), np.ones((1, 2)))
    assert m[0, 0] == 1 and m[0, 1] == 2
    m = ctx.mttkrp_packed(3, 2, 2, b, c, np.array([[1.0, 2], [3, 4]]), np.ones((2, 2)), np.ones((1, 2)))
    assert m[0, 0] == 7 and m[0, 1] == 10


def test_packed_vs_oracle_random(ctx, oracle, p2g):  # test_mttkrp.cpp:139-156 + acceptance c1 style
    o = oracle
    rng = o.Rng(24)
    for trial in range(40):
        rank = 1 + rng.below(4)
        n_cols = 2 + rng.below(12)
        n_slices = 1 + rng.below(8)
        density = 1.0 if trial % 3 == 0 else (0.5 if trial % 3 == 1 else 0.15)
        P = o.random_projected(rng, rank, n_cols, n_slices, density)
        h = o.random_matrix(rng, rank, rank)
        v = o.random_matrix(rng, n_cols, rank)
        w = o.random_matrix(rng, n_slices, rank)
        for mode in (1, 2, 3):
            gpu = ctx.mttkrp_packed(mode, *proj(P), h, v, w)
            assert rel_frob(gpu, o.naive_mttkrp(*proj(P), h, v, w, mode)) < 1e-10
            assert rel_frob(gpu, o.mttkrp(*proj(P), h, v, w, mode)) < 1e-13
    # determinism (test_mttkrp.cpp:218-229) and shape checks (:235-247)
    P = o.random_projected(o.Rng(27), 3, 10, 6, 0.5)
    h, v, w = np.eye(3), np.ones((10, 3)), np.ones((6, 3))
    for mode in (1, 2, 3):
        assert np.array_equal(ctx.mttkrp_packed(mode, *proj(P), h, v, w), ctx.mttkrp_packed(mode, *proj(P), h, v, w))
    with pytest.raises(p2g.InvalidArgument):
        ctx.mttkrp_packed(0, *proj(P), h, v, w)
    with pytest.raises(p2g.InvalidArgument):
        ctx.mttkrp_packed(1, *proj(P), np.ones((3, 2)), v, w)
    with pytest.raises(p2g.InvalidArgument):
        ctx.mttkrp_packed(1, 2, 3, [np.ones((2, 2))], [[1, 1]], np.eye(2), np.ones((3, 2)), np.ones((1, 2)))


def test_nnls_pinv_gram_vs_oracle(ctx, oracle, p2g):  # test_kernels.cpp:85-254
    o = oracle
    x = ctx.nnls_rowwise(np.eye(2), np.array([[1.0, -2.0]]))
    assert abs(x[0, 0] - 1) < 1e-12 and x[0, 1] == 0.0
    x = ctx.nnls_rowwise(np.eye(2), np.array([[3.0, 4.0]]))
    assert abs(x[0, 0] - 3) < 1e-12 and abs(x[0, 1] - 4) < 1e-12
    x = ctx.nnls_rowwise(np.array([[2.0, 1], [1, 2]]), np.array([[1.0, 1.0]]))
    assert np.abs(x - 1 / 3).max() < 1e-12
    with pytest.raises(p2g.NumericalError, match="NNLS did not converge"):
        ctx.nnls_rowwise(np.eye(2), np.array([[3.0, 4.0]]), max_iter=1)
    with pytest.raises(p2g.NumericalError):
        ctx.nnls_rowwise(np.eye(2), np.array([[np.nan, 1.0]]))
    rng = o.Rng(16)
    for n in (1, 3, 5, 10, 17, 40):
        f = o.random_matrix(rng, n + 2, n)
        g = o.gram(f) + 0.01 * np.eye(n)
        b = o.random_matrix(rng, 200, n, -2.0, 2.0)
        assert rel_frob(ctx.nnls_rowwise(g, b), o.nnls_rowwise(g, b)) < 1e-9
        assert rel_frob(ctx.pinv_small(g), o.pinv_small(g)) < 1e-9
        assert np.array_equal(ctx.gram(f), ctx.gram(f).T)
        assert rel_frob(ctx.gram(f), o.gram(f)) < 1e-14
    assert np.abs(ctx.pinv_small(np.array([[4.0, 0], [0, 0]])) - np.array([[0.25, 0], [0, 0]])).max() < 1e-14
    assert np.array_equal(ctx.gram(np.array([[1.0, 2], [3, 4]])), [[10, 14], [14, 20]])


def test_economy_svd(ctx, oracle, p2g):  # test_kernels.cpp:133-175
    o = oracle
    P, sig, Z = ctx.economy_svd(np.array([[3.0, 0], [0, 2]]))  # diagonal: recovers the diagonal
    assert sig.shape == (2,) and abs(sig[0] - 3.0) < 1e-12 and abs(sig[1] - 2.0) < 1e-12
    for c in range(2):
        assert abs(abs(P[c, c]) - 1.0) < 1e-12 and abs((P[:, c] * Z[:, c]).sum() - 1.0) < 1e-12
    P, sig, Z = ctx.economy_svd(np.zeros((2, 3)))  # zero matrix: zero sigma, identity-block bases
    assert sig.shape == (2,) and (sig == 0.0).all()
    assert np.array_equal(P, np.eye(2)) and np.array_equal(Z, np.eye(3)[:, :2])
    rng = o.Rng(14)
    shapes = [(1 + rng.below(6), 1 + rng.below(8)) for _ in range(20)] + [(60, 40), (40, 60), (97, 10), (5, 33)]
    for rows, cols in shapes:  # random matrices: reconstruction, orthonormal factors, ordered sigma, oracle's sigma
        m = o.random_matrix(rng, rows, cols)
        P, sig, Z = ctx.economy_svd(m)
        rho = min(rows, cols)
        assert P.shape == (rows, rho) and Z.shape == (cols, rho) and sig.shape == (rho,)
        assert np.linalg.norm(P @ np.diag(sig) @ Z.T - m) < 1e-10 * max(1.0, np.linalg.norm(m))
        assert np.linalg.norm(P.T @ P - np.eye(rho)) < 1e-10 and np.linalg.norm(Z.T @ Z - np.eye(rho)) < 1e-10
        assert (np.diff(sig) <= 0).all() and sig[-1] >= 0.0
        _, sref, _ = o.economy_svd(m)
        assert np.abs(sig - np.asarray(sref)).max() <= 1e-12 * max(1.0, sig[0])
    # rank-deficient: an orthonormal completion of the null columns, exact reconstruction
    a = o.random_matrix(rng, 9, 2)
    m = a @ o.random_matrix(rng, 2, 5)
    P, sig, Z = ctx.economy_svd(m)
    assert np.linalg.norm(P @ np.diag(sig) @ Z.T - m) < 1e-10 * np.linalg.norm(m) and sig[2] <= 1e-13 * sig[0]
    assert np.linalg.norm(P.T @ P - np.eye(5)) < 1e-10 and np.linalg.norm(Z.T @ Z - np.eye(5)) < 1e-10
    with pytest.raises(p2g.NumericalError, match="svd operand"):
        ctx.economy_svd(np.array([[1.0, np.nan], [0.0, 1.0]]))


def test_cp_als_iteration_vs_oracle(ctx, oracle):  # cp.hpp:99-145
    o = oracle
    rng = o.Rng(32)
    for trial in range(20):
        rank = 1 + rng.below(4)
        n_cols = 2 + rng.below(9)
        n_slices = 1 + rng.below(8)
        P = o.random_projected(rng, rank, n_cols, n_slices, 1.0 if trial % 2 == 0 else 0.4)
        nonneg = trial % 2 == 0
        lo = 0.0 if nonneg else -1.0
        h = o.random_matrix(rng, rank, rank)
        v = o.random_matrix(rng, n_cols, rank, lo, 1.0)
        w = o.random_matrix(rng, n_slices, rank, lo, 1.0)
        ref = o.cp_als_iteration(*proj(P), h, v, w, nonneg, trial % 4 == 1)
        got = ctx.cp_als_iteration(*proj(P), h, v, w, nonneg, trial % 4 == 1)
        for key in ("H", "V", "W", "m3", "lambda"):
            assert rel_err(got[key], ref[key]) <= TOL_STEP, (trial, key)


# ---------------------------------------------------------------------------
# The fused-loop kernels on the BASELINE cfg1 workload, teacher-forced
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def cfg1(p2g, oracle):
    X = p2g.generate_baseline(1, 5)
    H0, V0, W0 = p2g.init_factors(101, X.K, X.J, 5)
    T = oracle_from_csr(oracle, X)
    dumps = {}
    for nonneg in (False, True):
        dumps[nonneg] = oracle.fit_parafac2(T, 5, max_iters=10, tol=1e-300, nonneg=nonneg, threads=4, H0=H0, V0=V0,
                                            W0=W0, dumps=True)
    return X, T, (H0, V0, W0), dumps


@pytest.mark.parametrize("nonneg", [False, True])
def test_procrustes_teacher_forced(ctx, oracle, cfg1, nonneg):
    X, T, _, dumps = cfg1
    ctx.load(X)
    for it, d in enumerate(dumps[nonneg]["dumps"]):
        Q, flags, m1 = ctx.procrustes(d["H_in"], d["V_in"], d["W_in"])
        oq = d["Q"]
        # integer gate: rank-deficient subjects identical
        ofl = np.array(d["flags"])
        assert np.array_equal(canonical_flags(flags), ofl), it
        assert rel_err(Q, oq) <= TOL_STEP, it
        assert rel_err(m1, d["m1"]) <= TOL_STEP, it
        # every Q_k column-orthonormal (acceptance c3)
        for k in range(0, X.K, 37):
            qk = Q[X.subj_row_ptr[k]:X.subj_row_ptr[k + 1]]
            assert np.linalg.norm(qk.T @ qk - np.eye(5)) < 1e-8


@pytest.mark.parametrize("nonneg", [False, True])
def test_mttkrp_q_and_project_teacher_forced(ctx, oracle, cfg1, nonneg):
    X, T, _, dumps = cfg1
    ctx.load(X)
    for it, d in enumerate(dumps[nonneg]["dumps"][:4]):
        Q = d["Q"]
        P = oracle.project_slices(T, Q)
        H, V, W = d["H"], d["V"], d["W"]
        for mode in (1, 2, 3):
            ref = oracle.mttkrp(*proj(P), H, V, W, mode)
            got = ctx.mttkrp_q(mode, Q, H, V, W)
            assert rel_err(got, ref) <= TOL_STEP, (it, mode)
        ptr, cols, blocks = ctx.project(Q, 5)
        for k in range(0, X.K, 11):
            assert list(cols[ptr[k]:ptr[k + 1]]) == P["cols"][k]
            assert rel_err(blocks[k], P["blocks"][k]) <= 1e-12


@pytest.mark.parametrize("nonneg", [False, True])
def test_fit_trajectory_cfg1(ctx, oracle, p2g, cfg1, nonneg):
    X, T, (H0, V0, W0), dumps = cfg1
    ctx.load(X)
    ref = dumps[nonneg]
    cfg = p2g.SolverConfig(rank=5, max_iters=10, tol=1e-300, nonneg=nonneg)
    res = ctx.fit(cfg, H0, V0, W0)
    assert res.iterations == 10 and not res.converged
    assert np.abs(res.fit - np.array(ref["fit"])).max() <= TOL_FIT
    assert abs(res.norm_x - T.frobenius_sq()) <= 1e-12 * res.norm_x
    # factors after 10 free-running iterations (reported; step-gated above)
    assert rel_err(res.H, ref["H"]) < 1e-6
    assert rel_err(res.V, ref["V"]) < 1e-6
    assert rel_err(res.W, ref["S"]) < 1e-6


def test_fit_single_iteration_factors_exact(ctx, oracle, p2g, cfg1):
    """One iteration from identical inputs: H, V, W, Q within 1e-9."""
    X, T, (H0, V0, W0), dumps = cfg1
    ctx.load(X)
    for nonneg in (False, True):
        d = dumps[nonneg]["dumps"][0]
        res = ctx.fit(p2g.SolverConfig(rank=5, max_iters=1, tol=1e-300, nonneg=nonneg), H0, V0, W0)
        assert rel_err(res.H, d["H"]) <= TOL_STEP
        assert rel_err(res.V, d["V"]) <= TOL_STEP
        assert rel_err(res.W, d["W"]) <= TOL_STEP
        assert rel_err(res.Q, d["Q"]) <= TOL_STEP
        assert abs(res.fit[0] - d["fit"]) <= 1e-12


def test_reference_random_init_and_residual_identity(ctx, oracle, p2g):
    """fit with the reference's own initialisation (init=random, seed) and the
    efficient-residual identity (test_solver.cpp:256-280) on GPU outputs."""
    o = oracle
    rng = o.Rng(51)
    for trial in range(4):
        T = o.random_tensor(rng, 4, 6, 3, 7, 0.4 if trial % 2 else 1.0)
        rank = 1 + rng.below(3)
        X = p2g.CSRTensor(*T.to_csr())
        ctx.load(X)
        for iters in (1, 3, 8):
            cfg = p2g.SolverConfig(rank=rank, max_iters=iters, tol=1e-300, nonneg=trial % 2 == 0, seed=trial)
            res = ctx.fit(cfg)
            ref = o.fit_parafac2(T, rank, max_iters=iters, tol=1e-300, nonneg=trial % 2 == 0, seed=trial)
            assert np.abs(res.fit - np.array(ref["fit"])).max() <= TOL_FIT
            direct = o.dense_residual(T, res.Q, res.H, res.W, res.V)
            assert abs(res.residual_sq[-1] - direct) <= 1e-9 * max(1.0, direct)


def test_error_semantics(ctx, oracle, p2g):  # test_solver.cpp:86-120, 300-319
    o = oracle
    T = o.random_tensor(o.Rng(42), 3, 4, 2, 3, 1.0)
    ctx.load(p2g.CSRTensor(*T.to_csr()))
    with pytest.raises(p2g.DataError, match="rank exceeds variables"):
        ctx.fit(p2g.SolverConfig(rank=5))
    with pytest.raises(p2g.DataError, match="rank exceeds observations"):
        ctx.fit(p2g.SolverConfig(rank=4))
    for bad in (p2g.SolverConfig(rank=0), p2g.SolverConfig(rank=2, tol=0.0), p2g.SolverConfig(rank=2, max_iters=0)):
        with pytest.raises(p2g.InvalidArgument):
            ctx.fit(bad)
    T = o.Tensor.from_triplets(3, [(3, []), (2, [])])
    ctx.load(p2g.CSRTensor(*T.to_csr()))
    with pytest.raises(p2g.DataError, match="no non-zero entries"):
        ctx.fit(p2g.SolverConfig(rank=1))
    T = o.Tensor.from_triplets(2, [(2, [(0, 0, 1e200), (0, 1, 1e200), (1, 0, 1e200), (1, 1, 1e200)])])
    ctx.load(p2g.CSRTensor(*T.to_csr()))
    with pytest.raises(p2g.NumericalError):
        ctx.fit(p2g.SolverConfig(rank=2, max_iters=10))
    with pytest.raises(p2g.DataError):
        ctx.load(p2g.CSRTensor(3, np.array([0]), np.array([0]), np.array([], np.int32), np.array([])))


def test_cfg2_prefix_parity(ctx, oracle, p2g):
    """First 20,000 subjects of BASELINE cfg2 (R=10): 3 free-running iterations."""
    X = p2g.generate_baseline(2, 10, K=20000)
    H0, V0, W0 = p2g.init_factors(102, X.K, X.J, 10)
    T = oracle_from_csr(oracle, X)
    ref = oracle.fit_parafac2(T, 10, max_iters=3, tol=1e-300, nonneg=True, threads=8, H0=H0, V0=V0, W0=W0,
                              dumps=True)
    ctx.load(X)
    res = ctx.fit(p2g.SolverConfig(rank=10, max_iters=3, tol=1e-300, nonneg=True), H0, V0, W0)
    assert np.abs(res.fit - np.array(ref["fit"])).max() <= TOL_FIT
    d = ref["dumps"][0]
    Q, flags, m1 = ctx.procrustes(d["H_in"], d["V_in"], d["W_in"])
    assert rel_err(Q, d["Q"]) <= TOL_STEP and rel_err(m1, d["m1"]) <= TOL_STEP


@pytest.mark.parametrize("cfg_id,R,K", [(3, 40, 1500), (5, 40, 1500), (3, 24, 800), (5, 17, 800), (3, 33, 600),
                                        (2, 13, 1500), (5, 16, 800)])
def test_large_rank_prefix_parity(ctx, oracle, p2g, cfg_id, R, K):
    """R > 16 (warp-per-subject pipeline, R > 32 crosses the warp width) on
    prefixes of the BASELINE R=40 configs: teacher-forced Procrustes + M1 each
    iteration, the free-running fit trajectory and final factors."""
    X = p2g.generate_baseline(cfg_id, R, K=K)
    H0, V0, W0 = p2g.init_factors(int(p2g.baseline_spec(cfg_id, R).seed), X.K, X.J, R)
    T = oracle_from_csr(oracle, X)
    ref = oracle.fit_parafac2(T, R, max_iters=3, tol=1e-300, nonneg=True, threads=8, H0=H0, V0=V0, W0=W0,
                              dumps=True)
    ctx.load(X)
    for d in ref["dumps"]:
        Q, flags, m1 = ctx.procrustes(d["H_in"], d["V_in"], d["W_in"])
        assert np.array_equal(canonical_flags(flags), np.array(d["flags"]))
        assert rel_err(m1, d["m1"]) <= TOL_STEP
        assert_q_close(X, Q, np.asarray(d["Q"]), np.asarray(d["H_in"]), np.asarray(d["V_in"]), np.asarray(d["W_in"]))
    res = ctx.fit(p2g.SolverConfig(rank=R, max_iters=3, tol=1e-300, nonneg=True), H0, V0, W0)
    assert np.abs(res.fit - np.array(ref["fit"])).max() <= TOL_FIT
    last = ref["dumps"][-1]
    for key, got in (("H", res.H), ("V", res.V), ("W", res.W)):
        assert rel_err(got, last[key]) <= TOL_STEP, key


def test_cfg5_small_rank_prefix_parity(ctx, oracle, p2g):
    """cfg5's Zipf-hot columns (split CSC segments) through the R <= 16 pipeline."""
    R = 10
    X = p2g.generate_baseline(5, R, K=3000)
    H0, V0, W0 = p2g.init_factors(int(p2g.baseline_spec(5, R).seed), X.K, X.J, R)
    T = oracle_from_csr(oracle, X)
    ref = oracle.fit_parafac2(T, R, max_iters=3, tol=1e-300, nonneg=True, threads=8, H0=H0, V0=V0, W0=W0,
                              dumps=True)
    ctx.load(X)
    res = ctx.fit(p2g.SolverConfig(rank=R, max_iters=3, tol=1e-300, nonneg=True), H0, V0, W0)
    assert np.abs(res.fit - np.array(ref["fit"])).max() <= TOL_FIT
    last = ref["dumps"][-1]
    for key, got in (("H", res.H), ("V", res.V), ("W", res.W)):
        assert rel_err(got, last[key]) <= TOL_STEP, key


@pytest.mark.parametrize("R", [10, 40])
def test_fit_bitwise_deterministic(ctx, p2g, R):
    """Fixed-order reductions everywhere (CSC mode 2, partial sums, NNLS): two
    fits from the same inputs agree bit for bit."""
    X = p2g.generate_baseline(3 if R > 16 else 2, R, K=4000)
    H0, V0, W0 = p2g.init_factors(7, X.K, X.J, R)
    ctx.load(X)
    cfg = p2g.SolverConfig(rank=R, max_iters=4, tol=1e-300, nonneg=True)
    a = ctx.fit(cfg, H0, V0, W0)
    b = ctx.fit(cfg, H0, V0, W0)
    assert np.array_equal(a.fit, b.fit)
    for x, y in ((a.H, b.H), (a.V, b.V), (a.W, b.W), (a.Q, b.Q)):
        assert np.array_equal(x, y)


def test_load_validation_errors(ctx, p2g):
    """IrregularTensor::from_slices checks (sparse.hpp:176-193), run on the
    device for a single-rank load: same messages, first failing row wins, and
    a rejected tensor leaves the context reloadable."""
    good = dict(srp=np.array([0, 2, 3]), rp=np.array([0, 2, 3, 5]), ci=np.array([0, 2, 1, 0, 3], np.int32),
                val=np.ones(5))

    def load(**kw):
        d = dict(good)
        d.update(kw)
        ctx.load(p2g.CSRTensor(4, d["srp"], d["rp"], d["ci"], d["val"]))

    load()
    with pytest.raises(p2g.DataError, match="row_ptr must be non-decreasing"):
        load(rp=np.array([0, 2, 1, 5]))
    with pytest.raises(p2g.DataError, match="column index out of range"):
        load(ci=np.array([0, 2, 1, 0, 4], np.int32))
    with pytest.raises(p2g.DataError, match="strictly ascending"):
        load(ci=np.array([0, 2, 1, 3, 3], np.int32))
    with pytest.raises(p2g.DataError, match="strictly ascending"):  # row 0 before row 2's range error
        load(ci=np.array([2, 0, 1, 0, 9], np.int32))
    with pytest.raises(p2g.DataError, match="column index out of range"):  # row 0 before row 2's order error
        load(ci=np.array([0, 7, 1, 3, 3], np.int32))
    load()
    res = ctx.fit(p2g.SolverConfig(rank=1, max_iters=2, tol=1e-300))
    assert np.all(np.isfinite(res.fit))


@pytest.mark.parametrize("R", [10, 40])
def test_state_reuse_across_calls(ctx, p2g, R):
    """The fused loop carries state between passes (mode 3 leaves X V rows and,
    for R <= 16, the next Gram C for the following iteration; Jacobi warm
    starts; NNLS passive sets).  Per-step hooks and reloads in between must
    invalidate it: a fit after them equals a fit on a fresh context, bit for bit."""
    X = p2g.generate_baseline(3 if R > 16 else 2, R, K=3000)
    H0, V0, W0 = p2g.init_factors(11, X.K, X.J, R)
    cfg = p2g.SolverConfig(rank=R, max_iters=3, tol=1e-300, nonneg=True)
    ctx.load(X)
    a = ctx.fit(cfg, H0, V0, W0)
    Q, _, _ = ctx.procrustes(a.H, a.V, a.W)       # teacher-forced step: overwrites Q, flags, Ewarm
    ctx.mttkrp_q(3, Q, a.H, a.V, a.W)             # mode-3 hook: overwrites m3
    b = ctx.fit(cfg, H0, V0, W0)
    ctx.load(X)                                   # reload: new CSC build, state dropped
    c = ctx.fit(cfg, H0, V0, W0)
    for r in (b, c):
        assert np.array_equal(a.fit, r.fit)
        for x, y in ((a.H, r.H), (a.V, r.V), (a.W, r.W)):
            assert np.array_equal(x, y)
