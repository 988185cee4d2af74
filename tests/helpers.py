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
