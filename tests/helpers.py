"""Test helpers: oracle import, CSR conversions, dense evaluations.

The oracle (oracle/_build/p2oracle*.so) is TEST INFRASTRUCTURE: it is used
here only as the checker.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_oracle():
    path = os.path.join(ROOT, "oracle", "_build")
    if path not in sys.path:
        sys.path.insert(0, path)
    import p2oracle  # noqa: E402

    return p2oracle


def rel_frob(a, ref):
    """helpers.hpp:48-50 — relative Frobenius distance, denominator floor 1."""
    a = np.asarray(a, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.linalg.norm(a - ref) / max(1.0, np.linalg.norm(ref)))


def rel_err(a, ref):
    """||a - b||_F / ||b||_F (acceptance.cpp:129-130), the 1e-9 parity gate."""
    a = np.asarray(a, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    d = np.linalg.norm(ref)
    return float(np.linalg.norm(a - ref) / d) if d > 0 else float(np.linalg.norm(a - ref))


def csr_from_oracle(p2g, tensor):
    J, srp, rp, ci, v = tensor.to_csr()
    return p2g.CSRTensor(int(J), srp, rp, ci, v)


def oracle_from_csr(oracle, X):
    return oracle.Tensor.from_csr(X.J, X.subj_row_ptr, X.row_ptr, X.col_idx, X.val)


def q_blocks(X, Q):
    """Packed row-major Q -> list of I_k x R blocks."""
    return [Q[X.subj_row_ptr[k]:X.subj_row_ptr[k + 1]] for k in range(X.K)]


def dense_slices(X):
    out = []
    for k in range(X.K):
        r0, r1 = X.subj_row_ptr[k], X.subj_row_ptr[k + 1]
        d = np.zeros((r1 - r0, X.J))
        for r in range(r0, r1):
            p0, p1 = X.row_ptr[r], X.row_ptr[r + 1]
            d[r - r0, X.col_idx[p0:p1]] = X.val[p0:p1]
        out.append(d)
    return out


def assert_q_close(X, Q, Qref, H, V, W, base=1e-9, eps=1e-14):
    """Per-subject Procrustes factors against the oracle's, with the polar
    factor's perturbation bound: |dQ_k| / |Q_k| <= base + eps * kappa_k, where
    kappa_k = sigma_max / sigma_r of A_k = X_k V diag(W_k) H^T over the
    singular values kept by the canonical null rule (sigma^2 > 1e-26 sigma_max^2),
    times cond(N) of the completion block for rank-deficient subjects.
    Two backward-stable polar factorisations agree to O(eps kappa); a single
    global Frobenius bound would be set by the worst-conditioned subject."""
    Q = np.asarray(Q)
    Qref = np.asarray(Qref)
    srp = np.asarray(X.subj_row_ptr)
    # per-subject relative errors, vectorised; the kappa bound is evaluated
    # only for subjects above the base tolerance
    d2 = np.add.reduceat(((Q - Qref) ** 2).sum(axis=1), srp[:-1])
    n2 = np.add.reduceat((Qref ** 2).sum(axis=1), srp[:-1])
    errs = np.sqrt(d2) / np.maximum(np.sqrt(n2), 1e-300)
    ok = errs[errs <= base]
    worst = float((ok / base).max()) if ok.size else 0.0
    for k in np.nonzero(errs > base)[0]:
        r0, r1 = X.subj_row_ptr[k], X.subj_row_ptr[k + 1]
        XV = np.zeros((r1 - r0, V.shape[1]))
        for r in range(r0, r1):
            p0, p1 = X.row_ptr[r], X.row_ptr[r + 1]
            XV[r - r0] = X.val[p0:p1] @ V[X.col_idx[p0:p1]]
        A = XV @ np.diag(W[k]) @ H.T
        U, s, Vt = np.linalg.svd(A, full_matrices=False)
        if s.size == 0 or s[0] == 0.0:
            kappa = 1.0
        else:
            rho = int(np.count_nonzero(s * s > 1e-26 * s[0] * s[0]))
            kappa = s[0] / s[rho - 1]
            if rho < A.shape[1]:  # completion polar(N), N = L E_perp - U_rho U_rho^T L E_perp
                Ep = Vt[rho:].T
                LE = np.zeros((A.shape[0], Ep.shape[1]))
                LE[:A.shape[1]] = Ep
                N = LE - U[:, :rho] @ (U[:, :rho].T @ LE)
                sn = np.linalg.svd(N, compute_uv=False)
                kappa *= sn[0] / max(sn[-1], 1e-300)
        err = np.linalg.norm(Q[r0:r1] - Qref[r0:r1]) / max(np.linalg.norm(Qref[r0:r1]), 1e-300)
        tol = base + eps * kappa
        assert err <= tol, (k, err, kappa)
        worst = max(worst, err / tol)
    return worst
