"""Pins the oracle's PARAFAC2 solver (Procrustes, projection, full loop)
against proj/tests/test_solver.cpp, test_sparse.cpp and acceptance criteria
2-6 (acceptance.cpp:147-398), same seeds."""
import numpy as np
import pytest

from tests.helpers import rel_frob


def slice_tensor(o, d):  # test_solver.cpp:31-38
    trip = [(i, j, float(d[i, j])) for i in range(d.shape[0]) for j in range(d.shape[1]) if d[i, j] != 0]
    return o.Tensor.from_triplets(d.shape[1], [(d.shape[0], trip)])


def procrustes_objective(x, q, h, s, v):
    return float(np.sum((x - q @ h @ np.diag(s) @ v.T) ** 2))


def test_initialize_defaults_and_validation(oracle):  # test_solver.cpp:47-120
    o = oracle
    x = o.random_tensor(o.Rng(41), 4, 5, 3, 7, 0.6)
    H, S, V = o.initialize(x, 2, 200, 1e-8, True, "random", 7)
    assert np.array_equal(H, np.eye(2)) and np.array_equal(S, np.ones((4, 2)))
    assert V.shape == (5, 2) and V.min() >= 0 and V.max() < 1
    assert np.array_equal(V, o.initialize(x, 2, 200, 1e-8, True, "random", 7)[2])
    assert not np.array_equal(V, o.initialize(x, 2, 200, 1e-8, True, "random", 8)[2])
    x3 = o.Tensor.from_triplets(3, [(2, [(0, 1, 2.0), (1, 1, 1.0)]), (1, [(0, 1, 3.0)])])
    V = o.initialize(x3, 1, 200, 1e-8, True, "eye", 0)[2]
    assert np.abs(V[:, 0] - np.array([0.0, 1.0, 0.0])).max() < 1e-12
    x = o.random_tensor(o.Rng(42), 3, 4, 2, 3, 1.0)
    for args in ((0, 200, 1e-8), (2, 200, 0.0), (2, 200, -1.0), (2, 0, 1e-8)):
        with pytest.raises(ValueError):
            o.initialize(x, args[0], args[1], args[2], True, "random", 0)
    with pytest.raises(RuntimeError, match="rank exceeds variables"):
        o.initialize(x, 5, 200, 1e-8, True, "random", 0)
    with pytest.raises(RuntimeError, match="rank exceeds observations"):
        o.initialize(x, 4, 200, 1e-8, True, "random", 0)


def test_procrustes_kats(oracle):  # test_solver.cpp:122-180
    o = oracle
    x = o.random_orthonormal(o.Rng(43), 6, 3)
    q, flag, _ = o.procrustes_update(slice_tensor(o, x), 0, np.eye(3), np.ones(3), np.eye(3))
    assert np.abs(q - x).max() < 1e-12 and flag == 0
    rng = o.Rng(44)
    for _ in range(10):
        rows = 5 + rng.below(6)
        rank = 1 + rng.below(3)
        cols = rank + rng.below(5)
        q_true = o.random_orthonormal(rng, rows, rank)
        h = o.random_matrix(rng, rank, rank, 0.2, 1.0)
        s = o.random_matrix(rng, rank, 1, 0.3, 1.0)[:, 0]
        v = o.random_matrix(rng, cols, rank, 0.1, 1.0)
        xd = q_true @ h @ np.diag(s) @ v.T
        q = o.procrustes_update(slice_tensor(o, xd), 0, h, s, v)[0]
        assert np.linalg.norm(q.T @ q - np.eye(rank)) < 1e-10
        assert procrustes_objective(xd, q, h, s, v) < 1e-18
    rng = o.Rng(45)
    for _ in range(5):
        rows = 4 + rng.below(5)
        rank = 1 + rng.below(3)
        cols = rank + rng.below(4)
        xs = o.random_slice_tensor(rng, rows, cols, 0.5)
        h = o.random_matrix(rng, rank, rank)
        s = o.random_matrix(rng, rank, 1, 0.1, 1.0)[:, 0]
        v = o.random_matrix(rng, cols, rank)
        q = o.procrustes_update(xs, 0, h, s, v)[0]
        xd = xs.slice_dense(0)
        best = procrustes_objective(xd, q, h, s, v)
        for _ in range(20):
            qc = o.random_orthonormal(rng, rows, rank)
            other = procrustes_objective(xd, qc, h, s, v)
            assert best <= other + 1e-12 * max(1.0, other)
    xs = o.Tensor.from_triplets(3, [(4, [(2, 1, 5.0)])])
    q, flag, _ = o.procrustes_update(xs, 0, np.eye(2), np.ones(2), np.zeros((3, 2)))
    assert q.shape == (4, 2) and np.linalg.norm(q.T @ q - np.eye(2)) < 1e-12
    assert np.array_equal(q, np.eye(4, 2)) and flag == 1  # kernels.hpp:101-104 identity block


def test_projection(oracle):  # test_solver.cpp:182-214
    o = oracle
    x = o.random_slice_tensor(o.Rng(46), 3, 6, 0.4)
    P = o.project_slices(x, np.eye(3))
    d = np.zeros((3, 6))
    for i, c in enumerate(P["cols"][0]):
        d[:, c] = P["blocks"][0][:, i]
    assert np.array_equal(d, x.slice_dense(0)) and P["cols"][0] == x.slice_nnz_cols(0)
    q = o.random_orthonormal(o.Rng(47), 5, 2)
    x = o.Tensor.from_triplets(4, [(5, [(3, 2, -2.5)])])
    P = o.project_slices(x, q)
    assert P["blocks"][0].shape == (2, 1) and np.array_equal(P["blocks"][0][:, 0], -2.5 * q[3])
    rng = o.Rng(48)
    x = o.random_tensor(rng, 6, 10, 3, 8, 0.25)
    qs = [o.random_orthonormal(rng, x.slice_rows(k), 3) for k in range(6)]
    P = o.project_slices(x, np.vstack(qs))
    for k in range(6):
        assert P["cols"][k] == x.slice_nnz_cols(k)
        d = np.zeros((3, 10))
        for i, c in enumerate(P["cols"][k]):
            d[:, c] = P["blocks"][k][:, i]
        assert rel_frob(d, qs[k].T @ x.slice_dense(k)) < 1e-13


def test_fit_loop_properties(oracle):  # test_solver.cpp:216-298
    o = oracle
    x = o.random_tensor(o.Rng(49), 5, 6, 3, 8, 0.5)
    r = o.fit_parafac2(x, 2, max_iters=50, tol=float("inf"))
    assert r["iterations"] == 1 and r["converged"]
    H, S, Q = r["H"], r["S"], r["Q"]
    phi = H.T @ H
    for k in range(5):
        qk = Q[sum(x.slice_rows(j) for j in range(k)):][:x.slice_rows(k)]
        assert np.linalg.norm(qk.T @ qk - np.eye(2)) < 1e-8
        u = qk @ H
        assert np.linalg.norm(u.T @ u - phi) / np.linalg.norm(phi) < 1e-6
    assert S.min() >= 0 and r["residual_sq"][0] >= 0 and r["fit"][0] <= 1
    x = o.random_tensor(o.Rng(50), 4, 5, 2, 6, 0.7)
    r = o.fit_parafac2(x, 2, max_iters=3, tol=1e-300)
    assert r["iterations"] == 3 and not r["converged"]
    rng = o.Rng(51)
    for trial in range(6):
        x = o.random_tensor(rng, 4, 6, 3, 7, 0.4 if trial % 2 else 1.0)
        rank = 1 + rng.below(3)
        eff, direct = [], []

        def obs(Q, H, S, V, it, res, fit):
            eff.append(res)
            direct.append(o.dense_residual(x, Q, H, S, V))

        o.fit_parafac2(x, rank, max_iters=8, tol=1e-14, nonneg=trial % 2 == 0, seed=trial, observer=obs)
        assert eff
        for a, b in zip(eff, direct):
            assert abs(a - b) <= 1e-9 * max(1.0, b)
    rng = o.Rng(52)
    for trial in range(4):
        x = o.random_tensor(rng, 5, 7, 3, 8, 0.5)
        r = o.fit_parafac2(x, 2, max_iters=15, tol=1e-14, nonneg=trial % 2 == 0)
        res = r["residual_sq"]
        for i in range(1, len(res)):
            assert res[i] <= res[i - 1] + 1e-7 * max(1.0, res[i - 1])


def test_fit_errors_and_determinism(oracle):  # test_solver.cpp:300-361
    o = oracle
    x = o.Tensor.from_triplets(3, [(3, []), (2, [])])
    with pytest.raises(RuntimeError, match="no non-zero entries"):
        o.fit_parafac2(x, 1)
    x = o.Tensor.from_triplets(2, [(2, [(0, 0, 1e200), (0, 1, 1e200), (1, 0, 1e200), (1, 1, 1e200)])])
    with pytest.raises(ArithmeticError):
        o.fit_parafac2(x, 2, max_iters=10)
    x = o.random_tensor(o.Rng(53), 6, 8, 3, 9, 0.4)
    a = o.fit_parafac2(x, 3, max_iters=10, seed=99)
    b = o.fit_parafac2(x, 3, max_iters=10, seed=99)
    for key in ("H", "V", "S", "Q"):
        assert np.array_equal(a[key], b[key])
    assert a["fit"] == b["fit"] and a["residual_sq"] == b["residual_sq"]
    x = o.random_tensor(o.Rng(54), 7, 6, 3, 8, 0.5)
    a = o.fit_parafac2(x, 2, max_iters=6, tol=1e-300, seed=5, threads=1)
    b = o.fit_parafac2(x, 2, max_iters=6, tol=1e-300, seed=5, threads=3)
    assert len(a["fit"]) == len(b["fit"])
    assert abs(a["residual_sq"][-1] - b["residual_sq"][-1]) <= 1e-9 * max(1.0, a["residual_sq"][-1])


def test_acceptance_c2_procrustes_optimal(oracle):  # acceptance.cpp:147-194
    o = oracle
    rng = o.Rng(2002)
    dens = (0.2, 0.6, 1.0)
    worst = -np.inf
    for i in range(50):
        R = 1 + rng.below(5)
        J = R + rng.below(16)
        I = R + rng.below(36)
        sl = o.random_slice_tensor(rng, I, J, dens[i % 3])
        H = o.random_matrix(rng, R, R)
        V = o.random_matrix(rng, J, R)
        s = np.array([rng.uniform_range(0.1, 1.5) for _ in range(R)])
        Xd = sl.slice_dense(0)
        q = o.procrustes_update(sl, 0, H, s, V)[0]
        f_star = procrustes_objective(Xd, q, H, s, V)
        for _ in range(100):
            qc = o.random_orthonormal(rng, I, R)
            f_c = procrustes_objective(Xd, qc, H, s, V)
            worst = max(worst, (f_star - f_c) / max(1.0, f_c))
    assert worst <= 1e-12


def fit_instance(o, i):  # acceptance.cpp:201-218
    rng = o.Rng(o.substream_seed(3003, i))
    R = 1 + rng.below(5)
    K = 2 + rng.below(49)
    J = max(R, 3) + rng.below(12)
    X = o.random_tensor(rng, K, J, R, 12, (0.25, 0.6, 1.0)[i % 3])
    return X, R, o.substream_seed(3300, i)


@pytest.mark.parametrize("nonneg", [False, True])
def test_acceptance_c3_c4_invariants(oracle, nonneg):  # acceptance.cpp:222-302 (first 12 fits)
    o = oracle
    worst_ortho = worst_cross = worst_id = 0.0
    worst_inc = -np.inf
    for i in range(12):
        X, R, seed = fit_instance(o, i)
        state = {"prev": np.inf}

        def obs(Q, H, S, V, it, res, fit):
            nonlocal worst_ortho, worst_cross, worst_id, worst_inc
            HtH = H.T @ H
            off = 0
            for k in range(X.n_slices):
                I = X.slice_rows(k)
                q = Q[off:off + I]
                off += I
                worst_ortho = max(worst_ortho, np.linalg.norm(q.T @ q - np.eye(R)))
                u = q @ H
                worst_cross = max(worst_cross, np.linalg.norm(u.T @ u - HtH) / max(np.linalg.norm(HtH), 1e-300))
            direct = o.dense_residual(X, Q, H, S, V)
            worst_id = max(worst_id, abs(res - direct) / max(1.0, direct))
            if it > 1:
                worst_inc = max(worst_inc, (res - state["prev"]) / max(1.0, state["prev"]))
            state["prev"] = res

        o.fit_parafac2(X, R, max_iters=40, tol=1e-12, nonneg=nonneg, seed=seed, observer=obs)
    assert worst_ortho < 1e-8 and worst_cross < 1e-6
    assert worst_id <= 1e-9 and worst_inc <= 1e-7


def test_acceptance_c5_recovery(oracle):  # acceptance.cpp:308-348
    o = oracle
    X, dropped = o.generate_synthetic(20, 15, 10, 3, 1.0, 42, True)
    best = -np.inf
    for r in range(5):
        res = o.fit_parafac2(X, 3, max_iters=500, tol=1e-10, nonneg=True, seed=o.substream_seed(5, r))
        best = max(best, res["fit"][-1])
    assert best >= 0.9999


def test_acceptance_c6_column_pattern(oracle):  # acceptance.cpp:355-398
    o = oracle
    rng = o.Rng(6006)
    dens = (0.05, 0.2, 0.6)
    for i in range(50):
        R = 1 + rng.below(4)
        K = 1 + rng.below(12)
        J = max(R, 3) + rng.below(22)
        X = o.random_tensor(rng, K, J, R, 12, dens[i % 3])
        qs = [o.random_orthonormal(rng, X.slice_rows(k), R) for k in range(K)]
        P = o.project_slices(X, np.vstack(qs))
        for k in range(K):
            exp = X.slice_nnz_cols(k)
            assert P["cols"][k] == exp
            D = qs[k].T @ X.slice_dense(k)
            assert [j for j in range(J) if (D[:, j] != 0).any()] == exp


def test_partition_and_sparse(oracle):  # parallel.hpp:34-79, test_sparse.cpp
    o = oracle
    assert o.partition_even(10, 3) == [(0, 3), (3, 6), (6, 10)]
    assert o.partition_weighted([0, 0, 0], 2) == [(0, 1), (1, 3)]
    assert o.partition_weighted([5, 1, 1, 1, 1, 1], 2) == [(0, 1), (1, 6)]
    assert o.partition_weighted([1], 4) == [(0, 1)]
    t = o.Tensor.from_triplets(3, [(3, [(1, 2, 5.0), (0, 0, 1.5), (1, 2, -2.0), (2, 1, 0.0), (0, 1, 3.0),
                                        (0, 1, -3.0)])])
    assert t.total_nnz == 2 and t.slice_nnz_cols(0) == [0, 2]
    J, srp, rp, ci, v = t.to_csr()
    assert list(srp) == [0, 3] and list(rp) == [0, 1, 2, 2] and list(ci) == [0, 2] and list(v) == [1.5, 3.0]
    with pytest.raises(ValueError):
        o.Tensor.from_triplets(2, [(2, [(2, 0, 1.0)])])
    with pytest.raises(RuntimeError):
        o.Tensor.from_triplets(2, [])
    t = o.Tensor.from_triplets(2, [(2, [(0, 0, 3.0), (1, 1, 4.0)])])
    assert t.frobenius_sq() == 25.0
