"""The oracle-side BASELINE generator (oracle/baseline_gen.hpp, used by the
CPU arms of bench.py so they never map libp2g) against libp2g's
p2g_gen_create: bit-identical CSR arrays and initial factors (SURVEY.md 8d,
decisions D1/D2/D10/D11).  CPU only."""
import numpy as np
import pytest

CASES = [(1, 5, None), (1, 40, 300), (2, 10, 3000), (3, 40, 1500), (4, 40, 1500), (5, 40, 1500), (5, 24, 800)]


@pytest.mark.parametrize("cfg,R,K", CASES)
def test_oracle_generator_matches_libp2g(oracle, p2g, cfg, R, K):
    X = p2g.generate_baseline(cfg, R, K=K)
    J, srp, rp, ci, v = oracle.baseline_generate(cfg, R, K or 0, 3)
    assert J == X.J
    np.testing.assert_array_equal(srp, X.subj_row_ptr)
    np.testing.assert_array_equal(rp, X.row_ptr)
    np.testing.assert_array_equal(ci, X.col_idx)
    assert np.array_equal(v.view(np.uint64), X.val.view(np.uint64))
    # D1: every subject has at least R rows
    assert np.diff(srp).min() >= R


@pytest.mark.parametrize("cfg,R", [(1, 5), (4, 40)])
def test_oracle_init_factors_match_libp2g(oracle, p2g, cfg, R):
    spec = oracle.baseline_spec(cfg, R)
    K, J, seed = spec["K"], spec["J"], spec["seed"]
    H, V, W = p2g.init_factors(seed, K, J, R)
    Ho, Vo, Wo = oracle.baseline_init(seed, K, J, R)
    for a, b in ((H, Ho), (V, Vo), (W, Wo)):
        assert np.array_equal(np.asarray(a).view(np.uint64), np.ascontiguousarray(b).view(np.uint64)) or \
            np.array_equal(a, b)
    # a prefix of W is the same stream's first K_use rows (the CPU arms' bounded samples)
    _, _, Wp = oracle.baseline_init(seed, K, J, R, 123)
    np.testing.assert_array_equal(Wp, Wo[:123])


def test_subject_prefix_is_a_prefix(oracle):
    _, srp_a, rp_a, ci_a, v_a = oracle.baseline_generate(2, 10, 500, 2)
    _, srp_b, rp_b, ci_b, v_b = oracle.baseline_generate(2, 10, 200, 1)
    np.testing.assert_array_equal(srp_a[:201], srp_b)
    n = rp_b[-1]
    np.testing.assert_array_equal(ci_a[:n], ci_b)
    np.testing.assert_array_equal(v_a[:n], v_b)
