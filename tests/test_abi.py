"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/p2g.h declares, the host-side utilities are bit-exact with the
oracle, and compute entry points fail loudly (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

from tests.helpers import ROOT, oracle_from_csr


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "p2g.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(p2g_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(p2g):
    lib = ctypes.CDLL(p2g.lib_path())
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python mirror binds all of them
    assert set(syms) <= set(p2g._SIGS), set(syms) - set(p2g._SIGS)


def test_version_and_errors(p2g):
    assert b"sm_100a" in p2g.load_library().p2g_version()
    with pytest.raises(p2g.InvalidArgument):
        p2g.partition_weighted([1, 2], 1) and p2g._check(1)


def test_partition_weighted_bit_exact(p2g, oracle):
    rng = np.random.default_rng(0)
    for trial in range(200):
        n = int(rng.integers(0, 40))
        w = rng.integers(0, 5 if trial % 3 else 1000, size=n).tolist()
        chunks = int(rng.integers(1, 9))
        assert p2g.partition_weighted(w, chunks) == [tuple(x) for x in oracle.partition_weighted(w, chunks)]


def test_init_factors_follow_reference_stream(p2g, oracle):
    H, V, W = p2g.init_factors(7, 6, 5, 3)
    assert np.array_equal(H, np.eye(3))
    rng = oracle.Rng(7)
    V_ref = np.array([[0.0] * 3 for _ in range(5)])
    for r in range(3):
        for j in range(5):
            V_ref[j, r] = rng.uniform()
    W_ref = np.zeros((6, 3))
    for r in range(3):
        for k in range(6):
            W_ref[k, r] = rng.uniform()
    assert np.array_equal(V, V_ref) and np.array_equal(W, W_ref)
    # the reference's own random initialisation (solver.hpp:124-132)
    x = oracle.random_tensor(oracle.Rng(41), 4, 5, 3, 7, 0.6)
    Ho, So, Vo = oracle.initialize(x, 2, 200, 1e-8, True, "random", 7)
    H2, S2, V2 = p2g.initialize_random(7, 4, 5, 2)
    assert np.array_equal(H2, Ho) and np.array_equal(S2, So) and np.array_equal(V2, Vo)


def test_generator_cfg1_shape_and_determinism(p2g, oracle):
    X = p2g.generate_baseline(1, 5, threads=1)
    X4 = p2g.generate_baseline(1, 5, threads=4)
    for a, b in ((X.subj_row_ptr, X4.subj_row_ptr), (X.row_ptr, X4.row_ptr), (X.col_idx, X4.col_idx),
                 (X.val, X4.val)):
        assert np.array_equal(a, b)
    rows = X.rows_of()
    assert X.K == 1000 and X.J == 500
    assert rows.min() >= 5 and rows.max() <= 50            # D1 clamp to R
    per_row = np.diff(X.row_ptr)
    assert per_row.min() >= 1 and per_row.max() <= 10
    assert (X.val > 0).all() and (X.val <= 1).all()
    for r in range(0, X.n_rows, 97):                        # strictly ascending columns
        c = X.col_idx[X.row_ptr[r]:X.row_ptr[r + 1]]
        assert (np.diff(c) > 0).all()
    # first K subjects of the same stream are a prefix
    Xs = p2g.generate_baseline(1, 5, K=10)
    assert np.array_equal(Xs.col_idx, X.col_idx[:Xs.nnz])
    # the oracle sees the identical tensor
    T = oracle_from_csr(oracle, X)
    assert T.total_nnz == X.nnz and abs(T.frobenius_sq() - X.frobenius_sq()) <= 1e-12 * X.frobenius_sq()


def test_generator_cfg2_statistics(p2g):
    X = p2g.generate_baseline(2, 10, K=20000)
    rows = X.rows_of()
    assert rows.min() >= 10 and rows.max() <= 100
    assert abs(rows.mean() - 50.95) < 1.0
    assert abs(X.nnz / X.n_rows - 1.235) < 0.02             # 1 + Poisson(0.235)
    X5 = p2g.generate_baseline(5, 40, K=5000)
    r5 = X5.rows_of()
    assert r5.min() >= 40 and r5.max() <= 500
    assert set(np.unique(X5.val)) <= {1.0, 2.0, 3.0, 4.0, 5.0}
    counts = np.bincount(X5.col_idx, minlength=1500)
    assert counts[0] > counts[100] > counts[1400]           # Zipf popularity = column id


def test_compute_fails_loudly_without_gpu(p2g):
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(p2g.CudaError, match="no CUDA device"):
        p2g.Context(0)
