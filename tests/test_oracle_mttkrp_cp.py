"""Pins the oracle's MTTKRP and CP-ALS step against the reference's own tests:
proj/tests/test_mttkrp.cpp, proj/tests/test_cp.cpp and acceptance criterion 1
(acceptance.cpp:93-141), same seeds."""
import math

import numpy as np
import pytest

from tests.helpers import rel_frob


def example():  # test_mttkrp.cpp:31-36: diag(1,2) over J=2
    return 2, 2, [np.array([[1.0, 0.0], [0.0, 2.0]])], [[0, 1]]


def proj(P):
    return P["rank"], P["n_cols"], P["blocks"], P["cols"]


def dense_y(rank, J, block, cols):
    d = np.zeros((rank, J))
    for i, c in enumerate(cols):
        d[:, c] = block[:, i]
    return d


def test_mode_kats(oracle):  # test_mttkrp.cpp:36-101
    o = oracle
    R, J, b, c = example()
    w = np.array([[3.0, 5.0]])
    assert np.array_equal(o.mttkrp(R, J, b, c, np.eye(2), np.ones((2, 2)), w, 1), [[3, 5], [6, 10]])
    assert np.array_equal(o.mttkrp(R, J, b, c, np.eye(2), np.ones((2, 2)), w, 2), [[3, 0], [0, 10]])
    m = o.mttkrp(1, 3, [np.array([[4.0]]), np.array([[7.0]])], [[0], [2]], np.array([[1.0]]), np.ones((3, 1)),
                 np.array([[1.0], [10.0]]), 2)
    assert m[0, 0] == 4 and m[1, 0] == 0 and m[2, 0] == 70
    m = o.mttkrp(R, J, b, c, np.eye(2), np.ones((2, 2)), np.ones((1, 2)), 3)
    assert m[0, 0] == 1 and m[0, 1] == 2
    m = o.mttkrp(R, J, b, c, np.array([[1.0, 2], [3, 4]]), np.ones((2, 2)), np.ones((1, 2)), 3)
    assert m[0, 0] == 7 and m[0, 1] == 10


def test_mode1_ones_and_mode3_rows(oracle):  # test_mttkrp.cpp:50-55, 103-114
    o = oracle
    rng = o.Rng(21)
    P = o.random_projected(rng, 3, 8, 5, 0.4)
    v = o.random_matrix(rng, 8, 3)
    m = o.mttkrp(*proj(P), np.eye(3), v, np.ones((5, 3)), 1)
    exp = sum(dense_y(3, 8, P["blocks"][k], P["cols"][k]) @ v for k in range(5))
    assert rel_frob(m, exp) < 1e-14
    rng = o.Rng(22)
    P = o.random_projected(rng, 2, 6, 4, 0.5)
    h = o.random_matrix(rng, 2, 2)
    v = o.random_matrix(rng, 6, 2)
    full = o.mttkrp(*proj(P), h, v, np.ones((4, 2)), 3)
    for k in range(4):
        row = o.mttkrp(2, 6, [P["blocks"][k]], [P["cols"][k]], h, v, np.ones((1, 2)), 3)
        assert np.array_equal(row[0], full[k])


def test_zero_slice_contributes_nothing(oracle):  # test_mttkrp.cpp:116-137
    o = oracle
    rng = o.Rng(23)
    v = o.random_matrix(rng, 5, 2)
    h = o.random_matrix(rng, 2, 2)
    w = o.random_matrix(rng, 2, 2)
    block = o.random_matrix(rng, 2, 3)
    for mode in (1, 2, 3):
        both = o.mttkrp(2, 5, [block, np.zeros((2, 5))], [[0, 2, 4], [0, 1, 2, 3, 4]], h, v, w, mode)
        one = o.mttkrp(2, 5, [block], [[0, 2, 4]], h, v, w[:1], mode)
        if mode == 3:
            assert np.array_equal(both[0], one[0]) and not both[1].any()
        else:
            assert np.array_equal(both, one)


def test_specialized_vs_naive(oracle):  # test_mttkrp.cpp:139-176
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
            assert rel_frob(o.mttkrp(*proj(P), h, v, w, mode), o.naive_mttkrp(*proj(P), h, v, w, mode)) < 1e-10
    R, J, b, c = example()
    m = o.naive_mttkrp(R, J, b, c, np.eye(2), np.ones((2, 2)), np.array([[3.0, 5.0]]), 1)
    assert rel_frob(m, [[3, 5], [6, 10]]) < 1e-14
    for mode in (1, 2, 3):
        assert not o.naive_mttkrp(2, 3, [np.zeros((2, 2))], [[0, 2]], np.eye(2), np.ones((3, 2)),
                                  np.ones((1, 2)), mode).any()


def test_garbage_rows_never_read(oracle):  # test_mttkrp.cpp:178-201
    o = oracle
    rng = o.Rng(25)
    blocks = [o.random_matrix(rng, 2, 2), o.random_matrix(rng, 2, 3)]
    cols = [[1, 4], [1, 5, 6]]
    h = o.random_matrix(rng, 2, 2)
    w = o.random_matrix(rng, 2, 2)
    v = o.random_matrix(rng, 9, 2)
    vg = v.copy()
    for j in (0, 2, 3, 7, 8):
        vg[j] = 1e300
        vg[j, 0] = -9.87e250
    assert np.array_equal(o.mttkrp(2, 9, blocks, cols, h, v, w, 1), o.mttkrp(2, 9, blocks, cols, h, vg, w, 1))
    assert np.array_equal(o.mttkrp(2, 9, blocks, cols, h, v, w, 3), o.mttkrp(2, 9, blocks, cols, h, vg, w, 3))


def test_thread_agreement_and_shapes(oracle):  # test_mttkrp.cpp:203-259
    o = oracle
    rng = o.Rng(26)
    P = o.random_projected(rng, 4, 20, 13, 0.3)
    h = o.random_matrix(rng, 4, 4)
    v = o.random_matrix(rng, 20, 4)
    w = o.random_matrix(rng, 13, 4)
    for mode in (1, 2, 3):
        seq = o.mttkrp(*proj(P), h, v, w, mode, 1)
        assert np.array_equal(seq, o.mttkrp(*proj(P), h, v, w, mode, 1))
        for t in (2, 3, 5):
            assert rel_frob(o.mttkrp(*proj(P), h, v, w, mode, t), seq) < 1e-12
    R, J, b, c = example()
    h, v, w = np.eye(2), np.ones((2, 2)), np.ones((1, 2))
    for args in ((np.ones((3, 2)), v, w, 1), (h, np.ones((3, 2)), w, 1), (h, v, np.ones((2, 2)), 1),
                 (h, v, np.ones((1, 3)), 1), (h, v, w, 0), (h, v, w, 4)):
        with pytest.raises(ValueError):
            o.mttkrp(R, J, b, c, *args)
    assert o.naive_mttkrp_bytes(10, 20, 3, 1) == 8 * (3 * 200 + 200 * 3 + 3 * 3)
    assert o.naive_mttkrp_bytes(10, 20, 3, 2) == 8 * (20 * 30 + 30 * 3 + 20 * 3)
    assert o.naive_mttkrp_bytes(10, 20, 3, 3) == 8 * (10 * 60 + 60 * 3 + 10 * 3)


def test_acceptance_c1(oracle):  # acceptance.cpp:93-141 (all 200 instances)
    o = oracle
    rng = o.Rng(1001)
    densities = (0.1, 0.5, 1.0)
    worst = 0.0
    for i in range(200):
        K = 1 + rng.below(20)
        J = 2 + rng.below(29)
        R = 1 + rng.below(5)
        blocks, cols = [], []
        for _ in range(K):
            rows = R + rng.below(15 - R + 1)
            X = o.random_slice_tensor(rng, rows, J, densities[i % 3])
            Q = o.random_orthonormal(rng, rows, R)
            P = o.project_slices(X, Q)
            blocks.append(P["blocks"][0])
            cols.append(P["cols"][0])
        H = o.random_matrix(rng, R, R)
        V = o.random_matrix(rng, J, R)
        W = o.random_matrix(rng, K, R)
        for mode in (1, 2, 3):
            a = o.mttkrp(R, J, blocks, cols, H, V, W, mode)
            b = o.naive_mttkrp(R, J, blocks, cols, H, V, W, mode)
            d = np.linalg.norm(b)
            worst = max(worst, np.linalg.norm(a - b) / d if d > 0 else np.linalg.norm(a - b))
    assert worst <= 1e-10


# ---------------------------------------------------------------------------
# test_cp.cpp
# ---------------------------------------------------------------------------
def normalize_into(a, b):
    n = np.linalg.norm(a, axis=0)
    return a / n, b * n


def build_from_factors(o, h, v, w):
    dense = [h @ np.diag(w[k]) @ v.T for k in range(w.shape[0])]
    blocks, cols = [], []
    for d in dense:
        c = [j for j in range(d.shape[1]) if d[:, j].any()]
        blocks.append(d[:, c])
        cols.append(c)
    return h.shape[0], v.shape[0], blocks, cols


def test_cp_fixed_point_and_rank1(oracle):  # test_cp.cpp:58-94
    o = oracle
    rng = o.Rng(31)
    h = o.random_matrix(rng, 3, 3, 0.1, 1.0)
    v = o.random_matrix(rng, 6, 3, 0.1, 1.0)
    w = o.random_matrix(rng, 5, 3, 0.2, 1.0)
    h, w = normalize_into(h, w)
    v, w = normalize_into(v, w)
    Y = build_from_factors(o, h, v, w)
    out = o.cp_als_iteration(*Y, h, v, w)
    assert o.dense_cp_objective(*Y, out["H"], out["V"], out["W"], out["lambda"]) < 1e-18
    assert np.abs(out["H"] - h).max() < 1e-12
    assert np.abs(out["V"] - v).max() < 1e-12
    assert np.abs(out["W"] - w).max() < 1e-10
    out = o.cp_als_iteration(1, 2, [np.array([[2.0, 4.0]])], [[0, 1]], np.ones((1, 1)), np.ones((2, 1)),
                             np.ones((1, 1)))
    s5 = math.sqrt(5.0)
    assert abs(out["H"][0, 0] - 1) < 1e-12
    assert abs(out["V"][0, 0] - 1 / s5) < 1e-12 and abs(out["V"][1, 0] - 2 / s5) < 1e-12
    assert abs(out["W"][0, 0] - 2 * s5) < 1e-12


def test_cp_monotone_and_unit_columns(oracle):  # test_cp.cpp:96-151
    o = oracle
    rng = o.Rng(32)
    for trial in range(50):
        rank = 1 + rng.below(4)
        n_cols = 2 + rng.below(9)
        n_slices = 1 + rng.below(8)
        P = o.random_projected(rng, rank, n_cols, n_slices, 1.0 if trial % 2 == 0 else 0.4)
        nonneg = trial % 2 == 0
        lo = 0.0 if nonneg else -1.0
        h = o.random_matrix(rng, rank, rank)
        v = o.random_matrix(rng, n_cols, rank, lo, 1.0)
        w = o.random_matrix(rng, n_slices, rank, lo, 1.0)
        lam = np.ones(rank)
        before = o.cp_objective(*proj(P), h, v, w, lam)
        assert abs(before - o.dense_cp_objective(*proj(P), h, v, w, lam)) < 1e-9 * max(1.0, before)
        out = o.cp_als_iteration(*proj(P), h, v, w, nonneg)
        after = o.cp_objective(*proj(P), out["H"], out["V"], out["W"], out["lambda"])
        direct = o.dense_cp_objective(*proj(P), out["H"], out["V"], out["W"], out["lambda"])
        assert abs(after - direct) < 1e-9 * max(1.0, direct)
        assert after <= before + 1e-9 * max(1.0, before)
        if nonneg:
            assert out["V"].min() >= 0 and out["W"].min() >= 0
    rng = o.Rng(33)
    for _ in range(10):
        rank = 1 + rng.below(3)
        P = o.random_projected(rng, rank, 7, 4, 0.6)
        out = o.cp_als_iteration(*proj(P), o.random_matrix(rng, rank, rank), o.random_matrix(rng, 7, rank, 0.0, 1.0),
                                 o.random_matrix(rng, 4, rank, 0.0, 1.0))
        for r in range(rank):
            if out["H"][:, r].any():
                assert abs(np.linalg.norm(out["H"][:, r]) - 1) < 1e-12
            if out["V"][:, r].any():
                assert abs(np.linalg.norm(out["V"][:, r]) - 1) < 1e-12
        assert np.array_equal(out["lambda"], np.ones(rank))


def test_cp_signed_h_normalize_w_m3(oracle):  # test_cp.cpp:153-206
    o = oracle
    rng = o.Rng(34)
    h = np.array([[0.8, -0.3], [-0.6, 0.9]])
    v = o.random_matrix(rng, 5, 2, 0.1, 1.0)
    w = o.random_matrix(rng, 3, 2, 0.2, 1.0)
    v, w = normalize_into(v, w)
    Y = build_from_factors(o, h, v, w)
    out = o.cp_als_iteration(*Y, h, v, w)
    assert out["H"].min() < 0 and out["V"].min() >= 0 and out["W"].min() >= 0
    assert o.dense_cp_objective(*Y, out["H"], out["V"], out["W"], out["lambda"]) < 1e-15
    rng = o.Rng(35)
    P = o.random_projected(rng, 2, 6, 5, 0.7)
    h, v, w = o.random_matrix(rng, 2, 2), o.random_matrix(rng, 6, 2, 0.0, 1.0), o.random_matrix(rng, 5, 2, 0.0, 1.0)
    a = o.cp_als_iteration(*proj(P), h, v, w, True, False)
    b = o.cp_als_iteration(*proj(P), h, v, w, True, True)
    for r in range(2):
        assert abs(b["lambda"][r] - np.linalg.norm(a["W"][:, r])) < 1e-12
        if b["lambda"][r] > 0:
            assert abs(np.linalg.norm(b["W"][:, r]) - 1) < 1e-12
    assert rel_frob(b["W"] * b["lambda"], a["W"]) < 1e-12
    rng = o.Rng(36)
    P = o.random_projected(rng, 3, 8, 6, 0.5)
    out = o.cp_als_iteration(*proj(P), o.random_matrix(rng, 3, 3), o.random_matrix(rng, 8, 3, 0.0, 1.0),
                             o.random_matrix(rng, 6, 3, 0.0, 1.0))
    assert np.array_equal(out["m3"], o.mttkrp(*proj(P), out["H"], out["V"], np.ones((6, 3)), 3))
