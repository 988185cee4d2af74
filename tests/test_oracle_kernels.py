"""Pins the oracle's dense kernels against the reference's own known-answer and
property tests (proj/tests/test_kernels.cpp), same seeds (the pinned Rng is
bit-exact), plus LAPACK cross-checks of the Jacobi eig/SVD that replace Eigen."""
import numpy as np
import pytest

from tests.helpers import rel_frob


def mat2(a, b, c, d):
    return np.array([[a, b], [c, d]], dtype=np.float64)


def random_psd(o, rng, n, deficient):  # test_kernels.cpp:36-39
    f = o.random_matrix(rng, n - 1 if deficient else n + 2, n)
    return o.gram(f)


def test_khatri_rao_kats(oracle):  # test_kernels.cpp:43-83
    o = oracle
    exp = np.array([[1, 0], [3, 0], [0, 2], [0, 4]], dtype=float)
    assert np.array_equal(o.khatri_rao(mat2(1, 0, 0, 1), mat2(1, 2, 3, 4)), exp)
    assert o.khatri_rao(np.array([[2.0]]), np.array([[3.0]]))[0, 0] == 6.0
    assert np.array_equal(o.khatri_rao(np.ones((1, 2)), np.ones((2, 2))), np.ones((2, 2)))
    rng = o.Rng(11)
    a = o.random_matrix(rng, 4, 3)
    b = o.random_matrix(rng, 5, 3)
    kr = o.khatri_rao(a, b)
    for k in range(4):
        for i in range(5):
            assert np.array_equal(kr[k * 5 + i], o.hadamard(b[i:i + 1], a[k:k + 1])[0])
    with pytest.raises(ValueError):
        o.khatri_rao(np.ones((2, 2)), np.ones((2, 3)))


def test_gram_kats(oracle):  # test_kernels.cpp:85-103
    o = oracle
    assert o.gram(np.array([[3.0], [4.0]]))[0, 0] == 25.0
    assert np.array_equal(o.gram(np.eye(2)), np.eye(2))
    assert np.array_equal(o.gram(mat2(1, 2, 3, 4)), mat2(10, 14, 14, 20))
    g = o.gram(o.random_matrix(o.Rng(12), 17, 6))
    assert np.array_equal(g, g.T)


def test_pinv_kats(oracle):  # test_kernels.cpp:105-131
    o = oracle
    assert np.array_equal(o.pinv_small(np.eye(3)), np.eye(3))
    p = o.pinv_small(mat2(2, 1, 1, 2))
    assert np.abs(p - mat2(2 / 3, -1 / 3, -1 / 3, 2 / 3)).max() < 1e-14
    p = o.pinv_small(mat2(4, 0, 0, 0))
    assert np.abs(p - mat2(0.25, 0, 0, 0)).max() < 1e-14
    rng = o.Rng(13)
    for trial in range(30):
        n = 2 + rng.below(5)
        g = random_psd(o, rng, n, trial % 3 == 0)
        p = o.pinv_small(g)
        assert rel_frob(p @ g @ p, p) < 1e-9
        assert rel_frob(g @ p @ g, g) < 1e-9
        assert rel_frob(g @ p, (g @ p).T) < 1e-9
    with pytest.raises(ValueError):
        o.pinv_small(np.ones((2, 3)))


def test_economy_svd_kats(oracle):  # test_kernels.cpp:133-175
    o = oracle
    P, s, Z = o.economy_svd(mat2(3, 0, 0, 2))
    assert abs(s[0] - 3) < 1e-12 and abs(s[1] - 2) < 1e-12
    for c in range(2):
        assert abs(abs(P[c, c]) - 1) < 1e-12
        assert abs(np.dot(P[:, c], Z[:, c]) - 1) < 1e-12
    P, s, Z = o.economy_svd(np.zeros((2, 3)))
    assert s[0] == 0 and s[1] == 0
    assert np.linalg.norm(P.T @ P - np.eye(2)) < 1e-10
    assert np.linalg.norm(Z.T @ Z - np.eye(2)) < 1e-10
    rng = o.Rng(14)
    for _ in range(20):
        rows = 1 + rng.below(6)
        cols = 1 + rng.below(8)
        m = o.random_matrix(rng, rows, cols)
        P, s, Z = o.economy_svd(m)
        rho = min(rows, cols)
        assert P.shape == (rows, rho) and Z.shape == (cols, rho) and len(s) == rho
        assert np.linalg.norm(P @ np.diag(s) @ Z.T - m) < 1e-10 * max(1.0, np.linalg.norm(m))
        assert np.linalg.norm(P.T @ P - np.eye(rho)) < 1e-10
        assert np.linalg.norm(Z.T @ Z - np.eye(rho)) < 1e-10
        assert all(s[i] >= s[i + 1] for i in range(rho - 1)) and s[-1] >= 0
        # LAPACK cross-check of the Jacobi SVD that replaces Eigen::JacobiSVD
        assert np.allclose(s, np.linalg.svd(m, compute_uv=False), rtol=1e-13, atol=1e-14)


def test_sym_eig_matches_lapack(oracle):
    o = oracle
    rng = o.Rng(99)
    for n in (1, 2, 5, 10, 17, 40):
        a = o.random_matrix(rng, n, n)
        s = a + a.T
        vals, vecs = o.sym_eig(s)
        ref = np.linalg.eigvalsh(s)
        assert np.allclose(vals, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
        assert np.linalg.norm(vecs.T @ vecs - np.eye(n)) < 1e-12
        assert np.linalg.norm(s @ vecs - vecs @ np.diag(vals)) < 1e-11 * np.abs(ref).max()


def test_nnls_kats(oracle):  # test_kernels.cpp:177-201
    o = oracle
    x = o.nnls_rowwise(np.eye(2), np.array([[1.0, -2.0]]))
    assert abs(x[0, 0] - 1) < 1e-12 and x[0, 1] == 0.0
    x = o.nnls_rowwise(np.eye(2), np.array([[3.0, 4.0]]))
    assert abs(x[0, 0] - 3) < 1e-12 and abs(x[0, 1] - 4) < 1e-12
    x = o.nnls_rowwise(mat2(2, 1, 1, 2), np.array([[1.0, 1.0]]))
    assert abs(x[0, 0] - 1 / 3) < 1e-12 and abs(x[0, 1] - 1 / 3) < 1e-12


def test_nnls_properties(oracle):  # test_kernels.cpp:203-254
    o = oracle
    rng = o.Rng(15)
    for _ in range(20):
        n = 1 + rng.below(5)
        g = random_psd(o, rng, n, False) + 0.05 * np.eye(n)
        xs = o.random_matrix(rng, 3, n, 0.0, 2.0)
        b = xs @ g
        assert rel_frob(o.nnls_rowwise(g, b), xs) < 1e-9
    rng = o.Rng(16)
    for _ in range(30):
        n = 1 + rng.below(6)
        g = random_psd(o, rng, n, False) + 0.01 * np.eye(n)
        b = o.random_matrix(rng, 4, n, -2.0, 2.0)
        x = o.nnls_rowwise(g, b)
        assert x.min() >= 0
        for r in range(4):
            grad = g @ x[r] - b[r]
            for j in range(n):
                if x[r, j] > 0:
                    assert abs(grad[j]) < 1e-8 * max(1.0, np.linalg.norm(b[r]))
                else:
                    assert grad[j] >= -1e-10
    with pytest.raises(ArithmeticError, match="NNLS did not converge"):
        o.nnls_rowwise(np.eye(2), np.array([[3.0, 4.0]]), 1, 1)
    rng = o.Rng(17)
    g = random_psd(o, rng, 4, False) + 0.05 * np.eye(4)
    b = o.random_matrix(rng, 9, 4, -1.0, 3.0)
    assert np.array_equal(o.nnls_rowwise(g, b, 1), o.nnls_rowwise(g, b, 3))


def test_hadamard_and_nonfinite(oracle):  # test_kernels.cpp:256-285
    o = oracle
    r = o.hadamard(np.array([[1.0, 2.0]]), np.array([[3.0, 4.0]]))
    assert r[0, 0] == 3 and r[0, 1] == 8
    m = o.random_matrix(o.Rng(18), 3, 4)
    assert np.array_equal(o.hadamard(m, np.ones((3, 4))), m)
    assert np.array_equal(o.hadamard(m, np.zeros((3, 4))), np.zeros((3, 4)))
    with pytest.raises(ValueError):
        o.hadamard(m, np.ones((4, 3)))
    bad = mat2(1, np.nan, 0, 1)
    badinf = mat2(np.inf, 0, 0, 1)
    ok = np.eye(2)
    for fn in (lambda: o.khatri_rao(bad, ok), lambda: o.khatri_rao(ok, badinf), lambda: o.hadamard(bad, ok),
               lambda: o.gram(bad), lambda: o.pinv_small(badinf), lambda: o.economy_svd(bad),
               lambda: o.nnls_rowwise(ok, bad)):
        with pytest.raises(ArithmeticError):
            fn()
