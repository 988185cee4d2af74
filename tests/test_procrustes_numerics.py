"""The large-R Procrustes step's numerics, restated in numpy.

k_procrustes_large_w stops its Jacobi sweeps once every scaled off-diagonal
|M'_pq| / sqrt(M'_pp M'_qq) is at most tau = 1e-4 and takes
S' = M'^{-1/2} from the second-order Daleckii-Krein expansion about
Lambda = diag(M'):  S'_pq = d_pq u_p + u_p u_q (C1 - A + P o C2)_pq with
s = sqrt(lambda), u = 1/s, P_pq = 1/(s_p + s_q), A = P o N, C1 = A diag(u) A,
C2 = A A.  These tests pin that closed form against eigh at the kernel's
tolerance, in the scaled norm that bounds the error of Q = B V' S' E'^T.
"""
import numpy as np
import pytest

TAU = 1e-4  # kTauL in paper_1703_04219_b200/csrc/k_large.cu


def second_order_inv_sqrt(M):
    lam = np.diag(M).copy()
    s = np.sqrt(lam)
    u = 1.0 / s
    N = M - np.diag(lam)
    P = 1.0 / (s[:, None] + s[None, :])
    A = P * N
    C1 = A @ np.diag(u) @ A
    C2 = A @ A
    return np.diag(u) + u[:, None] * u[None, :] * (C1 - A + P * C2)


def exact_inv_sqrt(M):
    w, U = np.linalg.eigh(M)
    return U @ np.diag(w ** -0.5) @ U.T


def scaled_err(S, Sx, lam):
    sc = np.sqrt(lam)
    return float(np.abs(sc[:, None] * (S - Sx) * sc[None, :]).max())


@pytest.mark.parametrize("R", [17, 24, 40])
def test_second_order_matches_eigh_at_tau(R):
    rng = np.random.default_rng(R)
    worst = 0.0
    for _ in range(20):
        lam = 10.0 ** rng.uniform(-3, 0, R)  # eigh is exact enough here to act as the reference
        lam[1] = lam[0] * (1 + 1e-12)        # a cluster: no eigenvalue gaps enter the formula
        N = rng.uniform(-1, 1, (R, R)) * TAU
        N = (N + N.T) / 2
        np.fill_diagonal(N, 0.0)
        s = np.sqrt(lam)
        M = np.diag(lam) + s[:, None] * N * s[None, :]
        worst = max(worst, scaled_err(second_order_inv_sqrt(M), exact_inv_sqrt(M), lam))
    assert worst <= 1e-11  # measured ~3e-12 with every scaled off-diagonal at tau


def test_second_order_is_third_order_accurate():
    """Halving the off-diagonal divides the error by ~8 (cubic truncation)."""
    rng = np.random.default_rng(7)
    R = 40
    lam = 10.0 ** rng.uniform(-2, 0, R)
    N0 = rng.uniform(-1, 1, (R, R))
    N0 = (N0 + N0.T) / 2
    np.fill_diagonal(N0, 0.0)
    s = np.sqrt(lam)
    errs = []
    for d in (4e-3, 2e-3, 1e-3):
        M = np.diag(lam) + s[:, None] * (d * N0) * s[None, :]
        errs.append(scaled_err(second_order_inv_sqrt(M), exact_inv_sqrt(M), lam))
    assert 5.0 < errs[0] / errs[1] < 11.0 and 5.0 < errs[1] / errs[2] < 11.0


def test_polar_factor_from_corrected_root():
    """Q = B E' S' E'^T from a state the sweeps stop in (every scaled
    off-diagonal <= tau) is the polar factor of B (what
    procrustes_update's economy_svd yields) and orthonormal to 1e-10."""
    rng = np.random.default_rng(3)
    I, R = 58, 40
    lam = 10.0 ** rng.uniform(-4, 0, R)  # kappa(B) = 100: the test's own eigh round-off stays below the bound
    N = rng.uniform(-1, 1, (R, R)) * TAU
    N = (N + N.T) / 2
    np.fill_diagonal(N, 0.0)
    s = np.sqrt(lam)
    Mp = np.diag(lam) + s[:, None] * N * s[None, :]           # M' = E'^T (B^T B) E'
    E, _ = np.linalg.qr(rng.standard_normal((R, R)))            # E' (the accumulated rotations)
    M = E @ Mp @ E.T
    U0, _ = np.linalg.qr(rng.standard_normal((I, R)))           # polar(B) = U0 for B = U0 M^{1/2}
    w, V = np.linalg.eigh(M)
    B = U0 @ (V @ np.diag(np.sqrt(np.clip(w, 0, None))) @ V.T)
    Q = B @ (E @ second_order_inv_sqrt(Mp) @ E.T)
    assert np.linalg.norm(Q - U0) / np.linalg.norm(U0) <= 1e-10
    assert np.linalg.norm(Q.T @ Q - np.eye(R)) <= 1e-9
