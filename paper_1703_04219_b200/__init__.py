"""B200-native SPARTan PARAFAC2-ALS engine — Python host mirror of the C ABI.

The product is ``lib/libp2g.so`` (CUDA sm_100a + host C++), declared in
``include/p2g.h``.  This module is a thin ctypes binding whose names and
argument meaning follow the reference's C++ entry points
(/root/reference/proj/include/parafac2):

    fit_parafac2      solver.hpp:251-321    -> Context.fit
    procrustes_update solver.hpp:173-193    -> Context.procrustes (all subjects)
    project_slices    solver.hpp:212-235    -> Context.project
    mttkrp            mttkrp.hpp:187-196    -> Context.mttkrp_packed / mttkrp_q
    cp_als_iteration  cp.hpp:99-145         -> Context.cp_als_iteration
    nnls_rowwise      kernels.hpp:194-211   -> Context.nnls_rowwise
    pinv_small / gram kernels.hpp:57-87     -> Context.pinv_small / gram
    economy_svd       kernels.hpp:89-107    -> Context.economy_svd
    partition_weighted parallel.hpp:51-79   -> partition_weighted

Errors map like the reference's exception types: ``InvalidArgument``
(std::invalid_argument), ``DataError`` (exit code 2), ``NumericalError``
(exit code 3) and ``CudaError`` (no usable GPU / CUDA / NCCL failure).
There is no CPU fallback: without the built library or a GPU every compute
call raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

__all__ = [
    "InvalidArgument", "DataError", "NumericalError", "CudaError",
    "CSRTensor", "SolverConfig", "FitResult", "Context", "lib_path", "load_library",
    "partition_weighted", "generate_baseline", "baseline_spec", "init_factors",
    "initialize_random", "FLAG_FULL_RANK", "FLAG_DEFICIENT", "FLAG_ACCURATE", "FLAG_DEGENERATE",
]

FLAG_FULL_RANK, FLAG_DEFICIENT, FLAG_ACCURATE, FLAG_DEGENERATE = 0, 1, 2, 3


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class DataError(RuntimeError):
    """parafac2::DataError (common.hpp:37-39), CLI exit code 2."""


class NumericalError(ArithmeticError):
    """parafac2::NumericalError (common.hpp:43-45), CLI exit code 3."""


class CudaError(RuntimeError):
    """CUDA / NCCL failure or no usable device (the path has no CPU fallback)."""


_ERRORS = {1: InvalidArgument, 2: DataError, 3: NumericalError, 4: CudaError}

_HERE = os.path.dirname(os.path.abspath(__file__))


def lib_path() -> str:
    return os.path.join(_HERE, "lib", "libp2g.so")


class GenSpec(ctypes.Structure):
    _fields_ = [
        ("K", ctypes.c_int64), ("J", ctypes.c_int64), ("rows_dist", ctypes.c_int32),
        ("rows_lo", ctypes.c_int64), ("rows_hi", ctypes.c_int64), ("rows_mean", ctypes.c_double),
        ("min_rows", ctypes.c_int64), ("nnz_dist", ctypes.c_int32), ("nnz_lo", ctypes.c_int64),
        ("nnz_hi", ctypes.c_int64), ("nnz_lambda", ctypes.c_double), ("col_dist", ctypes.c_int32),
        ("zipf_s", ctypes.c_double), ("val_dist", ctypes.c_int32), ("seed", ctypes.c_uint64),
        ("threads", ctypes.c_int32),
    ]


class _FitConfig(ctypes.Structure):
    _fields_ = [
        ("rank", ctypes.c_int32), ("max_iters", ctypes.c_int32), ("tol", ctypes.c_double),
        ("nonneg", ctypes.c_int32), ("init", ctypes.c_int32), ("seed", ctypes.c_uint64),
    ]


class _BenchReport(ctypes.Structure):
    _fields_ = [("K", ctypes.c_int64), ("J", ctypes.c_int64), ("R", ctypes.c_int32), ("nnz", ctypes.c_int64),
                ("reps", ctypes.c_int32), ("budget_bytes", ctypes.c_uint64),
                ("specialized_ms", ctypes.c_double * 3), ("naive_ms", ctypes.c_double * 3),
                ("naive_bytes", ctypes.c_uint64 * 3), ("naive_oom", ctypes.c_int32 * 3),
                ("specialized_sweep_ms", ctypes.c_double), ("naive_sweep_ms", ctypes.c_double),
                ("naive_sweep_oom", ctypes.c_int32), ("speedup", ctypes.c_double),
                ("specialized_device_bytes", ctypes.c_uint64), ("checksum_specialized", ctypes.c_double),
                ("checksum_naive", ctypes.c_double)]


class _FitSummary(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int32), ("converged", ctypes.c_int32),
        ("total_ms", ctypes.c_double), ("norm_x", ctypes.c_double),
    ]


_LIB = None

_P = ctypes.c_void_p
_I32, _I64, _U64, _D = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double

_SIGS = {
    "p2g_last_error": (ctypes.c_char_p, []),
    "p2g_version": (ctypes.c_char_p, []),
    "p2g_partition_weighted": (ctypes.c_int, [_P, _I64, _I32, _P, _P]),
    "p2g_gen_baseline_spec": (ctypes.c_int, [_I32, _I32, _P]),
    "p2g_gen_create": (ctypes.c_int, [_P, _P, _P, _P]),
    "p2g_gen_export": (ctypes.c_int, [_P, _P, _P, _P, _P]),
    "p2g_gen_free": (None, [_P]),
    "p2g_init_factors": (ctypes.c_int, [_U64, _I64, _I64, _I32, _P, _P, _P]),
    "p2g_initialize_random": (ctypes.c_int, [_U64, _I64, _I64, _I32, _P, _P, _P]),
    "p2g_nccl_unique_id": (ctypes.c_int, [_P]),
    "p2g_create": (ctypes.c_int, [_I32, _I32, _I32, _P, _P]),
    "p2g_destroy": (ctypes.c_int, [_P]),
    "p2g_load_csr": (ctypes.c_int, [_P, _I64, _I64, _P, _P, _P, _P]),
    "p2g_shard_info": (ctypes.c_int, [_P, _P, _P, _P, _P]),
    "p2g_fit": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "p2g_bench_iterations": (ctypes.c_int, [_P, _P, _P, _P, _P, _I32, _I32, _P, _P]),
    "p2g_kernel_times": (ctypes.c_int, [_P, _I32, _P, _P, _P, _P]),
    "p2g_launch_count": (ctypes.c_int64, []),
    "p2g_procrustes": (ctypes.c_int, [_P, _I32, _P, _P, _P, _P, _P, _P]),
    "p2g_mttkrp_q": (ctypes.c_int, [_P, _I32, _I32, _P, _P, _P, _P, _P]),
    "p2g_project": (ctypes.c_int, [_P, _I32, _P, _P, _P, _P]),
    "p2g_mttkrp_packed": (ctypes.c_int, [_P, _I32, _I64, _I64, _I32, _P, _P, _P, _P, _P, _P, _P]),
    "p2g_cp_als_iteration": (ctypes.c_int, [_P, _I64, _I64, _I32, _P, _P, _P, _P, _P, _P, _I32, _I32, _P, _P]),
    "p2g_nnls_rowwise": (ctypes.c_int, [_P, _P, _P, _I64, _I32, _I32, _P]),
    "p2g_pinv_small": (ctypes.c_int, [_P, _P, _I32, _P]),
    "p2g_economy_svd": (ctypes.c_int, [_P, _P, _I64, _I64, _P, _P, _P]),
    "p2g_gram": (ctypes.c_int, [_P, _P, _I64, _I32, _P]),
    "p2g_load_shard": (ctypes.c_int, [_P, _I64, _I64, _I64, _I64, _P, _P, _P, _P]),
    "p2g_set_host_collective": (ctypes.c_int, [_P, _P, _P]),
    "p2g_inject_fault": (ctypes.c_int, [_P, _I32, _I32]),
    "p2g_fit_phase_ms": (ctypes.c_int, [_P, _I32, _P, _P]),
    "p2g_initialize_eye": (ctypes.c_int, [_P, _I32, _P]),
    "p2g_naive_mttkrp": (ctypes.c_int, [_P, _I32, _I64, _I64, _I32, _P, _P, _P, _P, _P, _P, _P]),
    "p2g_naive_mttkrp_bytes": (ctypes.c_uint64, [_I64, _I64, _I64, _I32]),
    "p2g_bench_mttkrp": (ctypes.c_int, [_P, _I32, _I32, _U64, _U64, _P]),
    "p2g_fit_dumps": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    # ingest / export (host side)
    "p2g_coo_parse": (ctypes.c_int, [ctypes.c_char_p, _I64, _I32, _P]),
    "p2g_coo_read": (ctypes.c_int, [ctypes.c_char_p, _I32, _P]),
    "p2g_csr_info": (ctypes.c_int, [_P, _P, _P, _P, _P, _P]),
    "p2g_csr_copy": (ctypes.c_int, [_P, _P, _P, _P, _P]),
    "p2g_csr_free": (None, [_P]),
    "p2g_coo_write": (ctypes.c_int, [ctypes.c_char_p, _I64, _I64, _P, _P, _P, _P, _P, _I32]),
    "p2g_csr_cache_write": (ctypes.c_int, [ctypes.c_char_p, _I64, _I64, _P, _P, _P, _P]),
    "p2g_csr_cache_read": (ctypes.c_int, [ctypes.c_char_p, _P]),
    "p2g_matrix_write": (ctypes.c_int, [ctypes.c_char_p, _I64, _I64, _P, ctypes.c_char_p]),
    "p2g_matrix_read": (ctypes.c_int, [ctypes.c_char_p, _P, _P, _P, _I64]),
    "p2g_matrix_parse": (ctypes.c_int, [ctypes.c_char_p, _I64, _P, _P, _P, _I64]),
    "p2g_write_factors": (ctypes.c_int, [ctypes.c_char_p, _I64, _I64, _I32, _P, _P, _P, _P, _P, ctypes.c_char_p]),
    "p2g_write_trace": (ctypes.c_int, [ctypes.c_char_p, _I32, _P, _P, _P]),
}


def load_library():
    """Loads lib/libp2g.so (built by ``make -C paper_1703_04219_b200``).

    Raises ``ImportError`` loudly when the extension is missing: there is no
    Python or CPU fallback for the compute path."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = lib_path()
    if not os.path.exists(path):
        raise ImportError(f"libp2g.so not built at {path}; run __graft_entry__.build() "
                          "or `make -C paper_1703_04219_b200`")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def _check(status: int) -> None:
    if status != 0:
        msg = load_library().p2g_last_error().decode()
        raise _ERRORS.get(status, RuntimeError)(msg)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a, shape=None, order="F") -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    if shape is not None and a.shape != tuple(shape):
        if a.ndim == 1 and len(shape) == 2 and a.size == shape[0] * shape[1]:
            a = a.reshape(shape, order=order)
        else:
            raise InvalidArgument(f"expected shape {tuple(shape)}, got {a.shape}")
    return np.require(a, dtype=np.float64, requirements=[order, "A"])


# ---------------------------------------------------------------------------
# Data model
# ---------------------------------------------------------------------------
@dataclass
class CSRTensor:
    """Irregular tensor {X_k} as one flattened CSR (include/p2g.h layout).

    Equivalent to the reference's IrregularTensor (sparse.hpp:176-215): subject
    k owns rows subj_row_ptr[k]..subj_row_ptr[k+1]; columns are strictly
    ascending within a row."""

    J: int
    subj_row_ptr: np.ndarray
    row_ptr: np.ndarray
    col_idx: np.ndarray
    val: np.ndarray

    def __post_init__(self):
        self.subj_row_ptr = np.ascontiguousarray(self.subj_row_ptr, dtype=np.int64)
        self.row_ptr = np.ascontiguousarray(self.row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(self.col_idx, dtype=np.int32)
        self.val = np.ascontiguousarray(self.val, dtype=np.float64)

    @property
    def K(self) -> int:
        return len(self.subj_row_ptr) - 1

    @property
    def n_rows(self) -> int:
        return int(self.subj_row_ptr[-1])

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def rows_of(self) -> np.ndarray:
        return np.diff(self.subj_row_ptr)

    def subject_nnz(self) -> np.ndarray:
        return self.row_ptr[self.subj_row_ptr[1:]] - self.row_ptr[self.subj_row_ptr[:-1]]

    def subset(self, k0: int, k1: int) -> "CSRTensor":
        """Subjects [k0, k1) as a standalone tensor (rebased)."""
        r0, r1 = int(self.subj_row_ptr[k0]), int(self.subj_row_ptr[k1])
        p0, p1 = int(self.row_ptr[r0]), int(self.row_ptr[r1])
        return CSRTensor(self.J, self.subj_row_ptr[k0:k1 + 1] - r0, self.row_ptr[r0:r1 + 1] - p0,
                         self.col_idx[p0:p1].copy(), self.val[p0:p1].copy())

    def frobenius_sq(self) -> float:
        return float(np.dot(self.val, self.val))

    def write_coordinate(self, path: str, comments: Sequence[str] = ()) -> None:
        """write_coordinate_file (io.hpp:179-204): canonical order, %.17g values."""
        arr = (ctypes.c_char_p * max(len(comments), 1))(*[c.encode() for c in comments])
        _check(load_library().p2g_coo_write(os.fsencode(path), self.K, self.J, _ptr(self.subj_row_ptr),
                                            _ptr(self.row_ptr), _ptr(self.col_idx), _ptr(self.val),
                                            ctypes.cast(arr, ctypes.c_void_p), len(comments)))

    def write_cache(self, path: str) -> None:
        """Binary CSR cache (reloads at storage speed)."""
        _check(load_library().p2g_csr_cache_write(os.fsencode(path), self.K, self.J, _ptr(self.subj_row_ptr),
                                                  _ptr(self.row_ptr), _ptr(self.col_idx), _ptr(self.val)))


def _take_csr(handle) -> "CSRTensor":
    lib = load_library()
    try:
        K, J, nr, nz, filt = (ctypes.c_int64() for _ in range(5))
        _check(lib.p2g_csr_info(handle, ctypes.byref(K), ctypes.byref(J), ctypes.byref(nr), ctypes.byref(nz),
                                ctypes.byref(filt)))
        srp = np.empty(K.value + 1, np.int64)
        rp = np.empty(nr.value + 1, np.int64)
        ci = np.empty(nz.value, np.int32)
        val = np.empty(nz.value, np.float64)
        _check(lib.p2g_csr_copy(handle, _ptr(srp), _ptr(rp), _ptr(ci), _ptr(val)))
    finally:
        lib.p2g_csr_free(handle)
    t = CSRTensor(J.value, srp, rp, ci, val)
    t.filtered_rows = filt.value
    return t


def parse_coordinate(text, threads: int = 0) -> "CSRTensor":
    """parse_coordinate_stream (io.hpp:100-171) on a string/bytes; the result
    carries .filtered_rows (all-zero rows removed)."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    h = ctypes.c_void_p()
    _check(load_library().p2g_coo_parse(data, len(data), threads, ctypes.byref(h)))
    return _take_csr(h)


def read_coordinate(path: str, threads: int = 0) -> "CSRTensor":
    """parse_coordinate_file (io.hpp:173-177)."""
    h = ctypes.c_void_p()
    _check(load_library().p2g_coo_read(os.fsencode(path), threads, ctypes.byref(h)))
    return _take_csr(h)


def read_cache(path: str) -> "CSRTensor":
    h = ctypes.c_void_p()
    _check(load_library().p2g_csr_cache_read(os.fsencode(path), ctypes.byref(h)))
    return _take_csr(h)


def write_matrix(path: str, M, title: str) -> None:
    """write_matrix_file (io.hpp:262-268)."""
    M = _f64(M)
    _check(load_library().p2g_matrix_write(os.fsencode(path), M.shape[0], M.shape[1], _ptr(M), title.encode()))


def _matrix_from(reader, *args) -> np.ndarray:
    rows, cols = ctypes.c_int64(), ctypes.c_int64()
    _check(reader(*args, ctypes.byref(rows), ctypes.byref(cols), None, 0))
    M = np.empty((rows.value, cols.value), order="F")
    _check(reader(*args, ctypes.byref(rows), ctypes.byref(cols), _ptr(M), M.size))
    return M


def read_matrix(path: str) -> np.ndarray:
    """read_matrix_file (io.hpp:256-260)."""
    return _matrix_from(load_library().p2g_matrix_read, os.fsencode(path))


def parse_matrix(text: str) -> np.ndarray:
    """read_matrix_stream (io.hpp:218-254) on a string."""
    data = text.encode()
    return _matrix_from(load_library().p2g_matrix_parse, data, len(data))


def write_factors(out_dir: str, X: "CSRTensor", H, V, S, Q, metadata: Optional[dict] = None) -> None:
    """write_factors (io.hpp:270-305): V, S, H, U_k = Q_k H, manifest.json.
    Q is the packed row-major (sum I_k) x R array (Context.fit's Q)."""
    import json as _json
    R = np.asarray(H).shape[0]
    H, V, S = _f64(H), _f64(V), _f64(S)
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    meta = _json.dumps(metadata) if metadata else None
    _check(load_library().p2g_write_factors(os.fsencode(out_dir), X.K, X.J, R, _ptr(X.subj_row_ptr), _ptr(H),
                                            _ptr(V), _ptr(S), _ptr(Q), meta.encode() if meta else None))


def write_trace(path: str, iters, residual_sq, fit) -> None:
    """write_trace_tsv (io.hpp:307-315): deterministic fields only."""
    it = np.ascontiguousarray(iters, dtype=np.int32)
    rs = np.ascontiguousarray(residual_sq, dtype=np.float64)
    ft = np.ascontiguousarray(fit, dtype=np.float64)
    _check(load_library().p2g_write_trace(os.fsencode(path), len(it), _ptr(it), _ptr(rs), _ptr(ft)))


def format_value(v: float) -> str:
    """io.hpp:55-60: 17 significant digits (round-trips exactly)."""
    return "%.17g" % v


def rank_components(S, subject: int, top_n: int):
    """io.hpp:317-333: components of subject k by decreasing diag(S_k), ties
    toward the lower index."""
    S = np.asarray(S)
    if subject < 0 or subject >= S.shape[0]:
        raise DataError(f"subject index out of range: {subject}")
    if top_n < 0 or top_n > S.shape[1]:
        raise InvalidArgument("top_n must be between 0 and the rank")
    order = sorted(range(S.shape[1]), key=lambda r: -S[subject, r])  # stable: ties keep index order
    return [(r, float(S[subject, r])) for r in order[:top_n]]


@dataclass
class SolverConfig:
    """solver.hpp:48-58 (threads is host-only and ignored on the GPU path)."""

    rank: int = 1
    max_iters: int = 200
    tol: float = 1e-8
    nonneg: bool = True
    init: str = "random"   # "random" (solver.hpp:128-132), "eye" (solver.hpp:133-164) or explicit factors (D2)
    seed: int = 0
    threads: int = 1


@dataclass
class FitResult:
    H: np.ndarray
    V: np.ndarray
    W: np.ndarray            # this rank's rows of S (= W), shard order
    Q: Optional[np.ndarray]  # packed row-major (sum I_k) x R of this shard
    flags: Optional[np.ndarray]
    fit: np.ndarray
    residual_sq: np.ndarray
    ms: np.ndarray
    iterations: int
    converged: bool
    total_ms: float
    norm_x: float
    k_begin: int = 0
    k_end: int = 0


# ---------------------------------------------------------------------------
# Host-side utilities (no GPU needed)
# ---------------------------------------------------------------------------
def partition_weighted(weights: Sequence[int], n_chunks: int):
    """parallel.hpp:51-79, bit-exact."""
    lib = load_library()
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.uint64))
    out = np.zeros(2 * max(n_chunks, 1), dtype=np.int64)
    n = ctypes.c_int32()
    _check(lib.p2g_partition_weighted(_ptr(w), len(w), n_chunks, _ptr(out), ctypes.byref(n)))
    return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(n.value)]


def naive_mttkrp_bytes(K: int, J: int, R: int, mode: int) -> int:
    """naive_mttkrp_bytes (mttkrp.hpp:241-253)."""
    return int(load_library().p2g_naive_mttkrp_bytes(K, J, R, mode))


def baseline_spec(config_id: int, R: int) -> GenSpec:
    spec = GenSpec()
    _check(load_library().p2g_gen_baseline_spec(config_id, R, ctypes.byref(spec)))
    return spec


def generate(spec: GenSpec) -> CSRTensor:
    lib = load_library()
    g = ctypes.c_void_p()
    nr, nz = ctypes.c_int64(), ctypes.c_int64()
    _check(lib.p2g_gen_create(ctypes.byref(spec), ctypes.byref(g), ctypes.byref(nr), ctypes.byref(nz)))
    try:
        srp = np.empty(spec.K + 1, np.int64)
        rp = np.empty(nr.value + 1, np.int64)
        ci = np.empty(nz.value, np.int32)
        v = np.empty(nz.value, np.float64)
        _check(lib.p2g_gen_export(g, _ptr(srp), _ptr(rp), _ptr(ci), _ptr(v)))
    finally:
        lib.p2g_gen_free(g)
    return CSRTensor(int(spec.J), srp, rp, ci, v)


def generate_baseline(config_id: int, R: int, K: Optional[int] = None, threads: int = 0) -> CSRTensor:
    """BASELINE.json config `config_id`.  K < spec.K gives the
    first K subjects of the same stream (subject k is a pure function of k)."""
    spec = baseline_spec(config_id, R)
    if K is not None:
        spec.K = int(K)
    spec.threads = threads
    return generate(spec)


def init_factors(seed: int, K: int, J: int, R: int):
    """H = I, V then W from one Rng(seed) stream (D2).  Column-major arrays."""
    H = np.empty((R, R), order="F")
    V = np.empty((J, R), order="F")
    W = np.empty((K, R), order="F")
    _check(load_library().p2g_init_factors(seed, K, J, R, _ptr(H), _ptr(V), _ptr(W)))
    return H, V, W


def initialize_random(seed: int, K: int, J: int, R: int):
    """initialize() random branch (solver.hpp:124-132): H = I, S = ones, V."""
    H = np.empty((R, R), order="F")
    S = np.empty((K, R), order="F")
    V = np.empty((J, R), order="F")
    _check(load_library().p2g_initialize_random(seed, K, J, R, _ptr(H), _ptr(S), _ptr(V)))
    return H, S, V


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load_library().p2g_nccl_unique_id(buf))
    return buf.raw


# ---------------------------------------------------------------------------
# Device context
# ---------------------------------------------------------------------------
# int fn(double* buf, int64_t count, int32_t op, void* user): host-staged allreduce
HOST_ALLREDUCE = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_int64, ctypes.c_int32,
                                  ctypes.c_void_p)


class Context:
    """One GPU (rank).  Mirrors the reference's free functions as methods."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None):
        self._lib = load_library()
        self._h = ctypes.c_void_p()
        idbuf = None if nccl_id is None else ctypes.create_string_buffer(nccl_id, 128)
        _check(self._lib.p2g_create(device, rank, world, idbuf, ctypes.byref(self._h)))
        self.rank, self.world = rank, world
        self.tensor: Optional[CSRTensor] = None
        self._w_rows = 0  # rows of W0 / W arguments: K (full load) or the shard's subjects (load_shard)
        self._coll = None

    def close(self):
        if self._h:
            _check(self._lib.p2g_destroy(self._h))
            self._h = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- data ---------------------------------------------------------------
    def load(self, X: CSRTensor) -> None:
        _check(self._lib.p2g_load_csr(self._h, X.K, X.J, _ptr(X.subj_row_ptr), _ptr(X.row_ptr),
                                      _ptr(X.col_idx), _ptr(X.val)))
        self.tensor = X
        self._w_rows = X.K

    def load_shard(self, K: int, k_begin: int, k_end: int, shard: CSRTensor) -> None:
        """This rank's subjects [k_begin, k_end) only (`shard` rebased to the
        shard, e.g. X.subset(k_begin, k_end)); collective over the ranks."""
        _check(self._lib.p2g_load_shard(self._h, int(K), shard.J, int(k_begin), int(k_end),
                                        _ptr(shard.subj_row_ptr), _ptr(shard.row_ptr), _ptr(shard.col_idx),
                                        _ptr(shard.val)))
        self.tensor = shard
        self._w_rows = shard.K

    def set_host_collective(self, fn) -> None:
        """fn(buf: np.ndarray (float64, modified in place), op: 0 sum | 1 max)
        reduces over all ranks; replaces NCCL for this context."""
        def _cb(ptr, count, op, user):
            try:
                fn(np.ctypeslib.as_array(ptr, shape=(count,)), int(op))
                return 0
            except Exception:  # noqa: BLE001 - reported as a status to the library
                return 1
        self._coll = HOST_ALLREDUCE(_cb)
        _check(self._lib.p2g_set_host_collective(self._h, ctypes.cast(self._coll, ctypes.c_void_p), None))

    def inject_fault(self, kind: int, iteration: int) -> None:
        _check(self._lib.p2g_inject_fault(self._h, kind, iteration))

    def naive_mttkrp(self, mode: int, rank: int, J: int, blocks, cols, H, V, W):
        """naive_mttkrp (mttkrp.hpp:208-235) on the device."""
        K = len(blocks)
        ptr, cl, Y = _pack_projected(rank, blocks, cols)
        rows = {1: rank, 2: J, 3: K}.get(mode, 1)
        out = np.empty((rows, rank), order="F")
        _check(self._lib.p2g_naive_mttkrp(self._h, mode, K, J, rank, _ptr(ptr), _ptr(cl), _ptr(Y),
                                          _ptr(_f64(H, (rank, rank))), _ptr(_f64(V, (J, rank))),
                                          _ptr(_f64(W, (K, rank))), _ptr(out)))
        return out

    def bench_mttkrp(self, R: int, reps: int = 3, budget_bytes: int = 0, seed: int = 0) -> dict:
        """bench_mttkrp (bench.hpp:90-215) on the device over the loaded tensor."""
        r = _BenchReport()
        _check(self._lib.p2g_bench_mttkrp(self._h, R, reps, budget_bytes, seed, ctypes.byref(r)))
        cells = []
        for m in range(3):
            cells.append({"kernel": "specialized", "mode": m + 1, "median_ms": r.specialized_ms[m], "oom": False})
        cells.append({"kernel": "specialized", "mode": 0, "median_ms": r.specialized_sweep_ms, "oom": False})
        for m in range(3):
            cells.append({"kernel": "naive", "mode": m + 1, "median_ms": r.naive_ms[m], "oom": bool(r.naive_oom[m]),
                          "bytes_needed": int(r.naive_bytes[m])})
        cells.append({"kernel": "naive", "mode": 0, "median_ms": r.naive_sweep_ms, "oom": bool(r.naive_sweep_oom)})
        return {"subjects": r.K, "cols": r.J, "rank": r.R, "nnz": r.nnz, "reps": r.reps,
                "budget_bytes": int(r.budget_bytes), "cells": cells, "specialized_sweep_ms": r.specialized_sweep_ms,
                "naive_sweep_ms": r.naive_sweep_ms, "naive_oom": bool(r.naive_sweep_oom), "speedup": r.speedup,
                "specialized_device_bytes": int(r.specialized_device_bytes),
                "checksum_specialized": r.checksum_specialized, "checksum_naive": r.checksum_naive}

    def initialize_eye(self, R: int) -> np.ndarray:
        """initialize(..., Init::eye) V (solver.hpp:133-164), J x R."""
        V = np.empty((self.tensor.J, R), order="F")
        _check(self._lib.p2g_initialize_eye(self._h, R, _ptr(V)))
        return V

    def fit_phase_ms(self, max_iters: int = 100000) -> np.ndarray:
        """(iterations x 3) ms_procrustes, ms_project, ms_cp of the last fit."""
        out = np.zeros(3 * max(max_iters, 1))
        n = ctypes.c_int32()
        _check(self._lib.p2g_fit_phase_ms(self._h, max_iters, _ptr(out), ctypes.byref(n)))
        return out[:3 * n.value].reshape(n.value, 3)

    def fit_dumps(self, cfg: "SolverConfig", H0, V0, W0):
        """Per-iteration outputs of the loop kernels: list of dicts with m1, m2,
        m3, H, V, W (column-major arrays) and fit."""
        X = self.tensor
        R = int(cfg.rank)
        H0, V0, W0 = _f64(H0, (R, R)), _f64(V0, (X.J, R)), _f64(W0, (self._w_rows, R))
        kb, ke, _, _ = self.shard_info()
        n = max(int(cfg.max_iters), 1)
        Ks = ke - kb
        m1, H = np.zeros((n, R, R)), np.zeros((n, R, R))
        m2, V = np.zeros((n, R, X.J)), np.zeros((n, R, X.J))
        m3, W = np.zeros((n, R, Ks)), np.zeros((n, R, Ks))
        fits = np.zeros(n)
        it = ctypes.c_int32()
        c = self._cfg(cfg, True)
        _check(self._lib.p2g_fit_dumps(self._h, ctypes.byref(c), _ptr(H0), _ptr(V0), _ptr(W0), _ptr(m1), _ptr(m2),
                                       _ptr(m3), _ptr(H), _ptr(V), _ptr(W), _ptr(fits), ctypes.byref(it)))
        return [{"m1": m1[t].T, "m2": m2[t].T, "m3": m3[t].T, "H": H[t].T, "V": V[t].T, "W": W[t].T,
                 "fit": float(fits[t])} for t in range(it.value)]

    def shard_info(self):
        kb, ke, nr, nz = (ctypes.c_int64() for _ in range(4))
        _check(self._lib.p2g_shard_info(self._h, ctypes.byref(kb), ctypes.byref(ke), ctypes.byref(nr),
                                        ctypes.byref(nz)))
        return kb.value, ke.value, nr.value, nz.value

    # -- fused loop -----------------------------------------------------------
    def _cfg(self, cfg: SolverConfig, explicit: bool) -> _FitConfig:
        if explicit:
            init = 2
        elif cfg.init == "eye":
            init = 1
        elif cfg.init == "random":
            init = 0
        else:
            raise InvalidArgument(f"unknown init {cfg.init!r}")
        return _FitConfig(int(cfg.rank), int(cfg.max_iters), float(cfg.tol), 1 if cfg.nonneg else 0,
                          init, int(cfg.seed) & ((1 << 64) - 1))

    def fit(self, cfg: SolverConfig, H0=None, V0=None, W0=None, want_q: bool = True, out=None,
            q_out=None) -> FitResult:
        """fit_parafac2 (solver.hpp:251-321) on this rank's shard.  `out` may
        supply the (H, V, W) result arrays (column-major float64, e.g. views of
        pinned host memory) and `q_out` the packed row-major (rows x R) Q."""
        X = self.tensor
        if X is None:
            raise InvalidArgument("no tensor loaded")
        R = int(cfg.rank)
        explicit = H0 is not None
        if explicit:
            H0 = _f64(H0, (R, R))
            V0 = _f64(V0, (X.J, R))
            W0 = _f64(W0, (self._w_rows, R))
        kb, ke, nr, _ = self.shard_info()
        Rv = max(R, 1)
        if out is not None:
            H, V, W = out
            for a, shp in ((H, (Rv, Rv)), (V, (X.J, Rv)), (W, (ke - kb, Rv))):
                if a.shape != shp or a.dtype != np.float64 or not a.flags.f_contiguous:
                    raise InvalidArgument(f"out array must be column-major float64 of shape {shp}")
        else:
            H = np.empty((Rv, Rv), order="F")
            V = np.empty((X.J, Rv), order="F")
            W = np.empty((ke - kb, Rv), order="F")
        if q_out is not None:
            if q_out.shape != (nr, Rv) or q_out.dtype != np.float64 or not q_out.flags.c_contiguous:
                raise InvalidArgument(f"q_out must be row-major float64 of shape {(nr, Rv)}")
            Q = q_out
        else:
            Q = np.empty((nr, Rv)) if want_q else None
        flags = np.empty(ke - kb, np.int32)
        n = max(int(cfg.max_iters), 1)
        fits, res, ms = np.zeros(n), np.zeros(n), np.zeros(n)
        summ = _FitSummary()
        c = self._cfg(cfg, explicit)
        _check(self._lib.p2g_fit(self._h, ctypes.byref(c), _ptr(H0), _ptr(V0), _ptr(W0), _ptr(H), _ptr(V),
                                 _ptr(W), _ptr(Q), _ptr(flags), _ptr(fits), _ptr(res), _ptr(ms),
                                 ctypes.byref(summ)))
        it = summ.iterations
        return FitResult(H, V, W, Q, flags, fits[:it], res[:it], ms[:it], it, bool(summ.converged),
                         summ.total_ms, summ.norm_x, kb, ke)

    def bench_iterations(self, cfg: SolverConfig, iters: int, H0=None, V0=None, W0=None, reset: bool = False):
        X = self.tensor
        R = int(cfg.rank)
        explicit = H0 is not None
        if explicit:
            H0, V0, W0 = _f64(H0, (R, R)), _f64(V0, (X.J, R)), _f64(W0, (self._w_rows, R))
        ms = np.zeros(max(iters, 1))
        fits = np.zeros(max(iters, 1))
        c = self._cfg(cfg, explicit)
        _check(self._lib.p2g_bench_iterations(self._h, ctypes.byref(c), _ptr(H0), _ptr(V0), _ptr(W0),
                                              1 if reset else 0, iters, _ptr(ms), _ptr(fits)))
        return ms[:iters], fits[:iters]

    def kernel_times(self):
        n = 64
        names = ctypes.create_string_buffer(32 * n)
        ms = np.zeros(n)
        cnt = np.zeros(n, np.int64)
        got = ctypes.c_int32()
        _check(self._lib.p2g_kernel_times(self._h, n, names, _ptr(ms), _ptr(cnt), ctypes.byref(got)))
        out = {}
        for i in range(got.value):
            nm = names.raw[32 * i:32 * i + 32].split(b"\0", 1)[0].decode()
            out[nm] = (float(ms[i]), int(cnt[i]))
        return out

    # -- per-step hooks ---------------------------------------------------------
    def procrustes(self, H, V, W):
        """procrustes_update over all shard subjects + fused M1 partial.
        Returns (Q packed row-major, flags, m1)."""
        X = self.tensor
        R = np.asarray(H).shape[0]
        _, _, nr, _ = self.shard_info()
        kb, ke = self.shard_info()[:2]
        Q = np.empty((nr, R))
        flags = np.empty(ke - kb, np.int32)
        m1 = np.empty((R, R), order="F")
        _check(self._lib.p2g_procrustes(self._h, R, _ptr(_f64(H, (R, R))), _ptr(_f64(V, (X.J, R))),
                                        _ptr(_f64(W, (self._w_rows, R))), _ptr(Q), _ptr(flags), _ptr(m1)))
        return Q, flags, m1

    def mttkrp_q(self, mode: int, Q, H, V, W):
        X = self.tensor
        R = np.asarray(H).shape[0]
        kb, ke, nr, _ = self.shard_info()
        rows = {1: R, 2: X.J, 3: ke - kb}.get(mode, 1)
        out = np.empty((rows, R), order="F")
        Qc = np.ascontiguousarray(np.asarray(Q, dtype=np.float64).reshape(nr, R))
        _check(self._lib.p2g_mttkrp_q(self._h, mode, R, _ptr(Qc), _ptr(_f64(H, (R, R))),
                                      _ptr(_f64(V, (X.J, R))), _ptr(_f64(W, (self._w_rows, R))), _ptr(out)))
        return out

    def project(self, Q, R: int):
        """project_slices: returns (ycol_ptr, ycols, list of R x c_k blocks)."""
        kb, ke, nr, _ = self.shard_info()
        ptr = np.empty(ke - kb + 1, np.int64)
        _check(self._lib.p2g_project(self._h, R, None, _ptr(ptr), None, None))
        nc = int(ptr[-1])
        cols = np.empty(max(nc, 1), np.int32)
        Y = np.empty(max(nc * R, 1))
        Qc = np.ascontiguousarray(np.asarray(Q, dtype=np.float64).reshape(nr, R))
        _check(self._lib.p2g_project(self._h, R, _ptr(Qc), _ptr(ptr), _ptr(cols), _ptr(Y)))
        blocks = [Y[ptr[k] * R:ptr[k + 1] * R].reshape((R, ptr[k + 1] - ptr[k]), order="F")
                  for k in range(ke - kb)]
        return ptr, cols[:nc], blocks

    def mttkrp_packed(self, mode: int, rank: int, J: int, blocks, cols, H, V, W):
        """mttkrp(ProjectedSlices, H, V, W, mode) (mttkrp.hpp:187-196)."""
        ptr, ycols, Y = _pack_projected(rank, blocks, cols)
        K = len(blocks)
        H = _f64(H)
        V = _f64(V)
        W = _f64(W)
        R = int(rank)
        if H.shape != (R, R):
            raise InvalidArgument("mttkrp: H must be R x R")
        if V.shape != (J, R):
            raise InvalidArgument("mttkrp: V must be J x R")
        if W.shape != (K, R):
            raise InvalidArgument("mttkrp: W must be K x R")
        rows = {1: R, 2: J, 3: K}.get(mode, 1)
        out = np.empty((max(rows, 1), R), order="F")
        _check(self._lib.p2g_mttkrp_packed(self._h, mode, K, J, R, _ptr(ptr), _ptr(ycols), _ptr(Y), _ptr(H),
                                           _ptr(V), _ptr(W), _ptr(out)))
        return out[:rows]

    def cp_als_iteration(self, rank: int, J: int, blocks, cols, H, V, W, nonneg=True, normalize_w=False):
        """cp_als_iteration (cp.hpp:99-145); returns dict(H, V, W, lambda, m3)."""
        ptr, ycols, Y = _pack_projected(rank, blocks, cols)
        K = len(blocks)
        R = int(rank)
        H = np.array(_f64(H), order="F", copy=True)
        V = np.array(_f64(V), order="F", copy=True)
        W = np.array(_f64(W), order="F", copy=True)
        if H.shape != (R, R):
            raise InvalidArgument("cp factors: H must be R x R")
        if V.shape != (J, R):
            raise InvalidArgument("cp factors: V must be J x R")
        if W.shape != (K, R):
            raise InvalidArgument("cp factors: W must be K x R")
        lam = np.empty(R)
        m3 = np.empty((K, R), order="F")
        _check(self._lib.p2g_cp_als_iteration(self._h, K, J, R, _ptr(ptr), _ptr(ycols), _ptr(Y), _ptr(H), _ptr(V),
                                              _ptr(W), 1 if nonneg else 0, 1 if normalize_w else 0, _ptr(lam),
                                              _ptr(m3)))
        return {"H": H, "V": V, "W": W, "lambda": lam, "m3": m3}

    def nnls_rowwise(self, G, B, max_iter: int = 0):
        G = _f64(G)
        B = _f64(B)
        if G.ndim != 2 or G.shape[0] != G.shape[1]:
            raise InvalidArgument("nnls_rowwise: G must be square")
        if B.ndim != 2 or B.shape[1] != G.shape[0]:
            raise InvalidArgument("nnls_rowwise: B column count must match G")
        X = np.empty(B.shape, order="F")
        _check(self._lib.p2g_nnls_rowwise(self._h, _ptr(G), _ptr(B), B.shape[0], G.shape[0], max_iter, _ptr(X)))
        return X

    def pinv_small(self, G):
        G = _f64(G)
        if G.ndim != 2 or G.shape[0] != G.shape[1]:
            raise InvalidArgument("pinv_small: matrix must be square")
        out = np.empty(G.shape, order="F")
        _check(self._lib.p2g_pinv_small(self._h, _ptr(G), G.shape[0], _ptr(out)))
        return out

    def economy_svd(self, M):
        """economy_svd (kernels.hpp:95-107): (P, sigma, Z) with M = P diag(sigma) Z^T."""
        M = _f64(M)
        if M.ndim != 2 or M.shape[0] < 1 or M.shape[1] < 1:
            raise InvalidArgument("economy_svd: need a non-empty matrix")
        rho = min(M.shape)
        P = np.empty((M.shape[0], rho), order="F")
        sig = np.empty(rho)
        Z = np.empty((M.shape[1], rho), order="F")
        _check(self._lib.p2g_economy_svd(self._h, _ptr(M), M.shape[0], M.shape[1], _ptr(P), _ptr(sig), _ptr(Z)))
        return P, sig, Z

    def gram(self, A):
        A = _f64(A)
        out = np.empty((A.shape[1], A.shape[1]), order="F")
        _check(self._lib.p2g_gram(self._h, _ptr(A), A.shape[0], A.shape[1], _ptr(out)))
        return out


def _pack_projected(rank: int, blocks, cols):
    """(list of R x c_k blocks, list of column lists) -> packed C-ABI arrays."""
    K = len(blocks)
    if len(cols) != K:
        raise InvalidArgument("packed blocks and column lists differ in count")
    ptr = np.zeros(K + 1, np.int64)
    for k in range(K):
        b = np.asarray(blocks[k], dtype=np.float64)
        c = np.asarray(cols[k])
        if b.size and b.shape[0] != rank:
            raise InvalidArgument("packed block row count differs from rank")
        width = b.shape[1] if b.ndim == 2 else 0
        if width != len(c):
            raise InvalidArgument("packed block width differs from column list")
        ptr[k + 1] = ptr[k] + len(c)
    nc = int(ptr[-1])
    ycols = np.zeros(max(nc, 1), np.int32)
    Y = np.zeros(max(nc * rank, 1))
    for k in range(K):
        c = np.asarray(cols[k], dtype=np.int64)
        ycols[ptr[k]:ptr[k + 1]] = c
        if len(c):
            Y[ptr[k] * rank:ptr[k + 1] * rank] = np.asarray(blocks[k], dtype=np.float64).reshape(-1, order="F")
    return ptr, ycols, Y
