"""Ingest / export through the C ABI: the reference's
io tests (proj/tests/test_io.cpp, cited per test) restated, plus oracle
cross-checks of the parsed tensors.  Host-only: no GPU needed."""
import json

import numpy as np
import pytest

from tests.helpers import csr_from_oracle


def _ser(p2g, X, tmp_path, comments=()):
    path = tmp_path / "t.txt"
    X.write_coordinate(str(path), comments)
    return path.read_text()


def test_format_value_round_trips(p2g):  # test_io.cpp:45-53
    for v in (0.0, 1.5, -3.0, 0.1, 1.0 / 3.0, 1e300, -2.5e-17, 1.7976931348623157e308, 4.9406564584124654e-324):
        assert float(p2g.format_value(v)) == v


def test_parse_simple(p2g):  # test_io.cpp:55-64
    X = p2g.parse_coordinate("2 3\n0 0 1 2.5\n1 0 0 1.0\n")
    assert X.K == 2 and X.J == 3 and X.nnz == 2 and X.filtered_rows == 0
    assert list(X.col_idx) == [1, 0] and list(X.val) == [2.5, 1.0]


def test_parse_sums_duplicates(p2g):  # test_io.cpp:66-70
    X = p2g.parse_coordinate("1 2\n0 0 1 1.0\n0 0 1 1.0\n")
    assert X.nnz == 1 and X.val[0] == 2.0


def test_parse_comments_blank_cr(p2g):  # test_io.cpp:72-82
    X = p2g.parse_coordinate("# a comment\r\n\n  \t \n1 2\r\n# interior comment\n0 0 0 4.25\r\n")
    assert X.K == 1 and X.val[0] == 4.25 and X.col_idx[0] == 0


def test_parse_filters_zero_rows(p2g):  # test_io.cpp:84-89
    X = p2g.parse_coordinate("1 3\n0 5 1 2.0\n")
    assert X.n_rows == 1 and X.filtered_rows == 5 and X.col_idx[0] == 1 and X.val[0] == 2.0


@pytest.mark.parametrize("text,msg", [  # test_io.cpp:91-151
    ("1 3\n0 0 5 1.0\n", "column index out of range at line 2"),
    ("1 3\n4 0 0 1.0\n", "subject index out of range at line 2"),
    ("1 3\n-1 0 0 1.0\n", "subject index out of range at line 2"),
    ("1 3\n0 -2 0 1.0\n", "row index out of range at line 2"),
    ("1\n", "at line 1"),
    ("x y\n", "malformed header"),
    ("0 3\n", "subject count must be positive"),
    ("2 0\n", "column count must be positive"),
    ("1 3\n0 0 1\n", "malformed entry (expected 'k i j v') at line 2"),
    ("1 3\n# ok\n0 0 one 1.0\n", "at line 3"),
    ("1 3\n0 0 1 abc\n", "malformed entry"),
    ("1 3\n0 0 1 inf\n", "non-finite value at line 2"),
    ("1 3\n0 0 1 nan\n", "non-finite value at line 2"),
    ("", "empty file"),
    ("# only comments\n", "empty file"),
    ("2 2\n0 0 0 1.0\n", "subject 1 has no entries"),
    ("1 1\n0 0 0 1.0\n0 0 0 -1.0\n", "subject 0 has no entries"),
])
def test_parse_errors(p2g, text, msg):
    with pytest.raises(p2g.DataError, match=msg.replace("(", r"\(").replace(")", r"\)")):
        p2g.parse_coordinate(text)


def test_parse_error_line_numbers_across_threads(p2g):
    """The first error in file order wins, with its exact line number, however
    the file is split across host threads."""
    lines = ["# big", "3 10"] + [f"{k % 3} {k % 7} {k % 10} 1.5" for k in range(20000)]
    lines[12345] = "0 0 99 1.0"   # column error (line 12346)
    lines[15000] = "7 0 0 1.0"    # later subject error
    text = "\n".join(lines) + "\n"
    for threads in (1, 3, 16):
        with pytest.raises(p2g.DataError, match="column index out of range at line 12346"):
            p2g.parse_coordinate(text, threads=threads)


def test_missing_file(p2g):  # test_io.cpp:143-146
    with pytest.raises(p2g.DataError):
        p2g.read_coordinate("/nonexistent/path/data.txt")


def test_canonical_serialisation(p2g, tmp_path):  # test_io.cpp:153-163
    X = p2g.parse_coordinate("2 3\n0 1 2 2.5\n0 0 0 1.5\n1 0 1 -3.0\n")
    assert _ser(p2g, X, tmp_path, ["demo"]) == "# demo\n2 3\n0 0 0 1.5\n0 1 2 2.5\n1 0 1 -3\n"


def test_round_trip_byte_identical(p2g, oracle, tmp_path):  # test_io.cpp:165-197
    rng = oracle.Rng(71)
    # every row occupied: serialize -> parse -> serialize is byte-identical
    X = csr_from_oracle(p2g, oracle.random_tensor(rng, 5, 7, 2, 6, 1.0))
    first = _ser(p2g, X, tmp_path)
    P = p2g.parse_coordinate(first)
    assert P.filtered_rows == 0 and _ser(p2g, P, tmp_path) == first
    # sparse: the first parse filters empty rows, then serialization is a fixpoint
    T = oracle.random_tensor(rng, 5, 7, 2, 6, 0.4)
    Y = csr_from_oracle(p2g, T)
    canonical = _ser(p2g, p2g.parse_coordinate(_ser(p2g, Y, tmp_path)), tmp_path)
    P = p2g.parse_coordinate(canonical)
    assert P.filtered_rows == 0 and _ser(p2g, P, tmp_path) == canonical
    # a scrambled entry order parses to the same bytes
    out = ["# scrambled order", f"{Y.K} {Y.J}"]
    for k in range(Y.K - 1, -1, -1):
        r0, r1 = Y.subj_row_ptr[k], Y.subj_row_ptr[k + 1]
        trips = [(r - r0, Y.col_idx[p], Y.val[p]) for r in range(r0, r1) for p in range(Y.row_ptr[r], Y.row_ptr[r + 1])]
        for i, j, v in reversed(trips):
            out.append(f"{k} {i} {j} {p2g.format_value(v)}")
    assert _ser(p2g, p2g.parse_coordinate("\n".join(out) + "\n"), tmp_path) == canonical


def test_parse_matches_oracle_with_duplicates(p2g, oracle):
    """Duplicate sums follow the reference's std::sort order: bit-identical to
    the oracle's SparseSlice::from_triplets on the same entries."""
    rng = np.random.default_rng(5)
    K, J = 40, 30
    lines = [f"{K} {J}"]
    per = {k: [] for k in range(K)}
    for _ in range(3000):
        k, i, j = int(rng.integers(K)), int(rng.integers(6)), int(rng.integers(J))
        v = float(rng.standard_normal())
        lines.append(f"{k} {i} {j} {p2g.format_value(v)}")
        per[k].append((i, j, v))
    X = p2g.parse_coordinate("\n".join(lines) + "\n", threads=4)
    T = oracle.Tensor.from_triplets(J, [(max(i for i, _, _ in per[k]) + 1, per[k]) for k in range(K)])
    Jo, srp, rp, ci, val = T.to_csr()
    # the oracle keeps all-zero rows; compare entry streams per subject
    for k in range(K):
        a = X.val[X.row_ptr[X.subj_row_ptr[k]]:X.row_ptr[X.subj_row_ptr[k + 1]]]
        b = np.asarray(val)[rp[srp[k]]:rp[srp[k + 1]]]
        assert np.array_equal(np.sort(a), np.sort(b))


def test_csr_cache_round_trip(p2g, tmp_path):
    X = p2g.generate_baseline(1, 5)
    X.write_cache(str(tmp_path / "x.p2g"))
    Y = p2g.read_cache(str(tmp_path / "x.p2g"))
    for a, b in ((X.subj_row_ptr, Y.subj_row_ptr), (X.row_ptr, Y.row_ptr), (X.col_idx, Y.col_idx), (X.val, Y.val)):
        assert np.array_equal(a, b)
    (tmp_path / "bad").write_bytes(b"nope")
    with pytest.raises(p2g.DataError):
        p2g.read_cache(str(tmp_path / "bad"))


def test_generator_text_round_trip(p2g, tmp_path):
    """A BASELINE tensor through the text format and back is bit-identical."""
    X = p2g.generate_baseline(1, 5)
    X.write_coordinate(str(tmp_path / "c1.txt"), ["cfg1"])
    Y = p2g.read_coordinate(str(tmp_path / "c1.txt"), threads=8)
    assert Y.filtered_rows == 0
    for a, b in ((X.subj_row_ptr, Y.subj_row_ptr), (X.row_ptr, Y.row_ptr), (X.col_idx, Y.col_idx), (X.val, Y.val)):
        assert np.array_equal(a, b)


def test_matrix_round_trip_and_golden(p2g, oracle, tmp_path):  # test_io.cpp:199-222
    m = oracle.random_matrix(oracle.Rng(72), 4, 3, -10.0, 10.0)
    m[0, 0], m[1, 2], m[2, 1] = 1.0 / 3.0, 1e-300, -0.1
    p2g.write_matrix(str(tmp_path / "m.txt"), m, "test matrix")
    assert np.array_equal(p2g.read_matrix(str(tmp_path / "m.txt")), m)
    p2g.write_matrix(str(tmp_path / "g.txt"), np.array([[1.5, -3.0], [0.25, 100.0]]), "demo")
    assert (tmp_path / "g.txt").read_text() == "# demo\n2 2\n1.5 -3\n0.25 100\n"


@pytest.mark.parametrize("text,msg", [  # test_io.cpp:224-239
    ("", "empty matrix file"),
    ("2 2\n1 2\n", "ended before all rows"),
    ("1 2\n1 2\n3 4\n", "unexpected extra matrix row"),
    ("1 3\n1 2\n", "wrong number of values"),
    ("1 1\nzz\n", "malformed matrix value"),
    ("bad header\n", "malformed matrix header"),
])
def test_matrix_errors(p2g, text, msg):
    with pytest.raises(p2g.DataError, match=msg):
        p2g.parse_matrix(text)


def test_write_factors_directory(p2g, oracle, tmp_path):  # test_io.cpp:241-274
    rng = oracle.Rng(73)
    H = oracle.random_matrix(rng, 2, 2)
    V = oracle.random_matrix(rng, 5, 2)
    S = oracle.random_matrix(rng, 3, 2, 0.0, 2.0)
    Qs = [oracle.random_orthonormal(rng, 4, 2), oracle.random_orthonormal(rng, 6, 2), oracle.random_orthonormal(rng, 3, 2)]
    srp = np.array([0, 4, 10, 13], np.int64)
    X = p2g.CSRTensor(5, srp, np.zeros(14, np.int64), np.zeros(0, np.int32), np.zeros(0))
    p2g.write_factors(str(tmp_path / "f"), X, H, V, S, np.vstack(Qs), {"rank": 2, "seed": 9})
    d = tmp_path / "f"
    assert np.array_equal(p2g.read_matrix(str(d / "V.txt")), V)
    assert np.array_equal(p2g.read_matrix(str(d / "S.txt")), S)
    assert np.array_equal(p2g.read_matrix(str(d / "H.txt")), H)
    for k in range(3):
        U = p2g.read_matrix(str(d / f"U_{k}.txt"))
        assert np.allclose(U, np.asarray(Qs[k]) @ np.asarray(H), rtol=0, atol=1e-15)
    man = json.loads((d / "manifest.json").read_text())
    assert man["rank"] == 2 and man["subjects"] == 3 and man["columns"] == 5
    assert len(man["files"]["U"]) == 3 and man["files"]["V"] == "V.txt"
    assert "mt19937_64" in man["prng"] and man["config"]["seed"] == 9


def test_trace_golden(p2g, tmp_path):  # test_io.cpp:276-293
    p2g.write_trace(str(tmp_path / "t.tsv"), [1, 2], [2.5, 1.25], [0.5, 0.75])
    assert (tmp_path / "t.tsv").read_text() == "iter\tresidual_sq\tfit\n1\t2.5\t0.5\n2\t1.25\t0.75\n"


def test_rank_components(p2g):  # test_io.cpp:295-322
    s = np.array([[0.1, 0.9], [0.5, 0.5]])
    assert p2g.rank_components(s, 0, 2) == [(1, 0.9), (0, 0.1)]
    assert p2g.rank_components(s, 1, 2) == [(0, 0.5), (1, 0.5)]
    assert p2g.rank_components(np.array([[0.3, 0.1, 0.7, 0.2, 0.6]]), 0, 1) == [(2, 0.7)]
    for args, exc in (((2, 1), p2g.DataError), ((-1, 1), p2g.DataError), ((0, 3), p2g.InvalidArgument),
                      ((0, -1), p2g.InvalidArgument)):
        with pytest.raises(exc):
            p2g.rank_components(s, *args)
