"""SURVEY.md 8(f) rows f3 and f4 on the GPU, against the oracle.

f4 -- eye initialisation (solver.hpp:133-164): the column Gram matrix
sum_k X_k^T X_k over non-zero column pairs and |leading R eigenvectors|.
Eigenvectors are compared column by column with the perturbation bound
eps ||C|| / gap (two correct eigensolvers agree to that); the reference's
own KAT (test_solver.cpp:71-84) is exact to 1e-12.

f3 -- naive MTTKRP (mttkrp.hpp:208-235: materialised unfolding times the
Khatri-Rao product) and the specialized-vs-naive harness (bench.hpp:90-215,
acceptance criterion 7, acceptance.cpp:409-495).
"""
import numpy as np
import pytest

from tests.helpers import oracle_from_csr, rel_err

pytestmark = pytest.mark.gpu


def _eig_tol(C, R):
    w = np.linalg.eigvalsh(C)[::-1]
    tol = []
    for r in range(R):
        gap = min(abs(w[r] - w[r - 1]) if r > 0 else np.inf, abs(w[r] - w[r + 1]) if r + 1 < len(w) else np.inf)
        tol.append(1e-9 + 1e-13 * w[0] / max(gap, 1e-300))
    return np.array(tol)


def test_eye_init_kat(ctx, oracle, p2g):
    """test_solver.cpp:71-84: all mass in column 1 -> V = e_1."""
    T = oracle.Tensor.from_triplets(3, [(2, [(0, 1, 2.0), (1, 1, 1.0)]), (1, [(0, 1, 3.0)])])
    ctx.load(p2g.CSRTensor(*T.to_csr()))
    V = ctx.initialize_eye(1)
    assert np.abs(V[:, 0] - np.array([0.0, 1.0, 0.0])).max() < 1e-12


@pytest.mark.parametrize("seed,J,R", [(3, 20, 3), (4, 45, 5), (5, 60, 8)])
def test_eye_init_matches_oracle(ctx, oracle, p2g, seed, J, R):
    o = oracle
    T = o.random_tensor(o.Rng(seed), 30, J, R, R + 12, 0.3, 0.0, 1.0)
    X = p2g.CSRTensor(*T.to_csr())
    ctx.load(X)
    V = ctx.initialize_eye(R)
    _, _, Vo = o.initialize(T, R, 5, 1e-8, True, "eye", 0)
    dense = np.vstack([T.slice_dense(k) for k in range(T.n_slices)])
    tol = _eig_tol(dense.T @ dense, R)
    for r in range(R):
        err = np.linalg.norm(V[:, r] - Vo[:, r])
        assert err <= tol[r], (r, err, tol[r])


def test_eye_init_fit_matches_oracle(ctx, oracle, p2g):
    o = oracle
    T = o.random_tensor(o.Rng(77), 40, 30, 4, 12, 0.35, 0.0, 1.0)
    ctx.load(p2g.CSRTensor(*T.to_csr()))
    for nonneg in (True, False):
        res = ctx.fit(p2g.SolverConfig(rank=3, max_iters=6, tol=1e-300, nonneg=nonneg, init="eye"))
        ref = o.fit_parafac2(T, 3, max_iters=6, tol=1e-300, nonneg=nonneg, init="eye")
        assert np.abs(res.fit - np.array(ref["fit"])).max() <= 1e-7
        assert rel_err(res.V, ref["V"]) <= 1e-7


def test_eye_init_baseline_shape(ctx, p2g):
    """The J = 5000 column Gram of a cfg4 prefix: V is non-negative with unit
    columns, and two runs agree bitwise (fixed accumulation order)."""
    X = p2g.generate_baseline(4, 40, K=20000)
    ctx.load(X)
    V1 = ctx.initialize_eye(40)
    V2 = ctx.initialize_eye(40)
    assert np.array_equal(V1, V2)
    assert (V1 >= 0).all()
    assert np.allclose(np.linalg.norm(V1, axis=0), 1.0, atol=1e-12)


# ---------------------------------------------------------------------------
# f3: naive MTTKRP and the harness
# ---------------------------------------------------------------------------
def test_naive_mttkrp_kats(ctx, oracle):
    """test_mttkrp.cpp:158-176: naive against the mode KATs and the zero case."""
    b, c = [np.array([[1.0, 0.0], [0.0, 2.0]])], [[0, 1]]
    w = np.array([[3.0, 5.0]])
    assert np.array_equal(ctx.naive_mttkrp(1, 2, 2, b, c, np.eye(2), np.ones((2, 2)), w), [[3, 5], [6, 10]])
    assert np.array_equal(ctx.naive_mttkrp(2, 2, 2, b, c, np.eye(2), np.ones((2, 2)), w), [[3, 0], [0, 10]])
    m = ctx.naive_mttkrp(3, 2, 2, b, c, np.array([[1.0, 2], [3, 4]]), np.ones((2, 2)), np.ones((1, 2)))
    assert m[0, 0] == 7 and m[0, 1] == 10
    z = ctx.naive_mttkrp(2, 2, 3, [np.zeros((2, 0))], [[]], np.eye(2), np.ones((3, 2)), np.ones((1, 2)))
    assert np.array_equal(z, np.zeros((3, 2)))


def test_naive_vs_specialized_random(ctx, oracle):
    """test_mttkrp.cpp:139-156 / acceptance c1: naive == specialized (1e-10)
    on 40 random instances, both on the GPU, and == the oracle's naive."""
    o = oracle
    rng = o.Rng(25)
    for trial in range(40):
        rank = 1 + rng.below(4)
        n_cols = 2 + rng.below(12)
        n_slices = 1 + rng.below(8)
        P = o.random_projected(rng, rank, n_cols, n_slices, 1.0 if trial % 2 else 0.3)
        h, v, w = o.random_matrix(rng, rank, rank), o.random_matrix(rng, n_cols, rank), o.random_matrix(rng, n_slices, rank)
        for mode in (1, 2, 3):
            nv = ctx.naive_mttkrp(mode, rank, n_cols, P["blocks"], P["cols"], h, v, w)
            sp = ctx.mttkrp_packed(mode, rank, n_cols, P["blocks"], P["cols"], h, v, w)
            ref = o.naive_mttkrp(rank, n_cols, P["blocks"], P["cols"], h, v, w, mode)
            assert np.abs(nv - sp).max() <= 1e-10 * max(1.0, np.abs(sp).max())
            assert np.abs(nv - ref).max() <= 1e-10 * max(1.0, np.abs(ref).max())


def test_naive_bytes(p2g, oracle):
    """test_mttkrp.cpp:245-255 byte counts, bit-exact with the oracle."""
    for K, J, R in ((50000, 2000, 10), (5, 7, 3), (1, 1, 1)):
        for mode in (1, 2, 3):
            assert p2g.naive_mttkrp_bytes(K, J, R, mode) == oracle.naive_mttkrp_bytes(K, J, R, mode)


def test_bench_mttkrp_harness(ctx, p2g):
    """bench.hpp:90-215 on the GPU at a reduced scale: every cell timed, the
    naive sweep present, checksums of both kernels agree, and a budget below
    the materialisation marks the naive cells out-of-memory."""
    X = p2g.generate_baseline(1, 10, K=400)
    ctx.load(X)
    rep = ctx.bench_mttkrp(10, reps=2, budget_bytes=1 << 40, seed=9)
    assert rep["specialized_sweep_ms"] > 0 and rep["naive_sweep_ms"] > 0 and not rep["naive_oom"]
    assert abs(rep["checksum_specialized"] - rep["checksum_naive"]) <= 1e-9 * abs(rep["checksum_naive"])
    small = ctx.bench_mttkrp(10, reps=1, budget_bytes=1000, seed=9)
    assert small["naive_oom"] and all(c["oom"] for c in small["cells"] if c["kernel"] == "naive" and c["mode"])
