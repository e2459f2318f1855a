"""The CPU oracle is pinned against outputs of the real reference
(tests/golden/*.npz, produced by tests/golden/make_golden.py in the build
container) and against the reference's own known-answer tests."""

import os

import numpy as np
import pytest
from numpy.testing import assert_allclose, assert_array_equal

import oracle
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_larfg_worked_example():
    # test_densecore.py:119-123
    tau, beta, ess = oracle.larfg(3.0, np.array([4.0]))
    assert beta == -5.0 and tau == 1.6
    assert_array_equal(ess, [0.5])


def test_larfg_zero_tail_is_identity():
    tau, beta, ess = oracle.larfg(-2.0, np.zeros(3))
    assert tau == 0.0 and beta == -2.0


def test_givens_worked_example():
    # test_densecore.py:168-172
    c, s, r = oracle.lartg(3.0, 4.0)
    assert_allclose((c, s, r), (0.6, 0.8, 5.0), rtol=1e-15)
    assert oracle.lartg(0.0, 0.0) == (1.0, 0.0, 0.0)


def test_tinv_worked_example():
    # test_qrblock.py:69-79
    y = np.array([[1.0, 0.0], [1.0, 1.0], [0.0, 1.0]])
    assert_allclose(oracle.cwy_tinv(y, np.array([1.0, 2.0])), [[1.0, 1.0], [0.0, 0.5]])


def test_split_four_row_example():
    # test_bdc.py:127-138
    left, right, alpha, beta = oracle.split_rows(oracle.Bidiag([1.0, 2.0, 3.0, 4.0], [5.0, 6.0, 7.0]))
    assert left.n == 1 and left.bordered and right.n == 2 and not right.bordered
    assert (alpha, beta) == (2.0, 6.0)


def test_deflation_examples():
    # test_bdc.py:208-252
    out = oracle.deflate_entries([0.0, 1.0, 1.0], [1.0, 0.6, 0.8])
    assert_array_equal(out["z"], [1.0, 1.0, 0.0])
    assert_array_equal(out["kept"], [0, 1])
    assert_array_equal(out["dvals"], [1.0])
    out = oracle.deflate_entries([0.0, 1.0, 2.0], [1.0, 1e-20, 1.0])
    assert_array_equal(out["kept"], [0, 2])
    out = oracle.deflate_entries([0.0, 1.0], [0.0, 1.0])
    assert out["zs"][0] != 0.0 and abs(out["zs"][0]) <= 16 * np.finfo(float).eps
    out = oracle.deflate_entries([0.0, 1e-18, 1.0], [0.6, 0.8, 1.0])
    assert_array_equal(out["dvals"], [0.0])


def test_secular_golden(golden):
    # test_bdc.py:284-291: d=[0,1], z=[1,1] -> omega^2 = (3 -+ sqrt 5)/2
    om, anc, mu = oracle.secular_roots(np.array([0.0, 1.0]), np.array([1.0, 1.0]))
    assert_allclose(om ** 2, [(3 - np.sqrt(5)) / 2, (3 + np.sqrt(5)) / 2], rtol=1e-14)
    assert_array_equal(om, golden["kat_secular_omega"])
    assert_array_equal(mu, golden["kat_secular_mu"])


def test_leaf_single_negative():
    # test_bdc.py:62-66
    r = oracle.leaf_svd(oracle.Bidiag([-3.0], np.zeros(0)))
    assert_array_equal(r.vals, [3.0])
    assert_array_equal(r.W, [[-1.0]])


def test_philox_stream_pins():
    # test_harness.py:24-40 first uniform is 0.011546754286331617
    u = oracle.philox_uniforms(0, 4)
    assert u[0] == 0.011546754286331617


def test_gesdd_matches_reference_bitwise(golden):
    for i in range(int(golden["svd_count"])):
        a = golden[f"svd{i}_a"]
        s, u, vt = oracle.svd(a)
        assert_array_equal(s, golden[f"svd{i}_sigma"])
        assert_array_equal(u, golden[f"svd{i}_u"])
        assert_array_equal(vt, golden[f"svd{i}_vt"])
        s2, _, _ = oracle.svd(a, want_vectors=False)
        assert_array_equal(s2, golden[f"svd{i}_sigma_values_only"])


def test_generator_matches_reference_inputs(golden):
    for i in range(int(golden["svd_count"])):
        m, n, cond, seed = golden[f"svd{i}_spec"]
        kind = str(golden[f"svd{i}_kind"])
        a = oracle.make_matrix(kind, int(m), int(n), float(cond), int(seed))
        assert_array_equal(a, golden[f"svd{i}_a"])


def test_gebrd_matches_reference_bitwise(golden):
    for i in range(int(golden["gebrd_count"])):
        a = golden[f"gebrd{i}_a"].copy(order="F")
        d, e, tq, tp = oracle.gebrd(a, int(golden[f"gebrd{i}_block"]))
        assert_array_equal(a, golden[f"gebrd{i}_packed"])
        for name, v in (("d", d), ("e", e), ("tauq", tq), ("taup", tp)):
            assert_array_equal(v, golden[f"gebrd{i}_{name}"])


def test_qr_matches_reference_bitwise(golden):
    for i in range(int(golden["qr_count"])):
        a = golden[f"qr{i}_a"].copy(order="F")
        b, ob = golden[f"qr{i}_blocks"]
        tau = oracle.geqrf(a, int(b))
        assert_array_equal(a, golden[f"qr{i}_packed"])
        assert_array_equal(tau, golden[f"qr{i}_tau"])
        assert_array_equal(oracle.orgqr(a, tau, a.shape[1], int(ob)), golden[f"qr{i}_q"])


def test_bdsdc_matches_reference_bitwise(golden):
    for i in range(int(golden["bdc_count"])):
        bord, leaf = (int(x) for x in golden[f"bdc{i}_meta"])
        r = oracle.bdc(oracle.Bidiag(golden[f"bdc{i}_d"], golden[f"bdc{i}_e"], bool(bord)), leaf=leaf)
        assert_array_equal(r.vals, golden[f"bdc{i}_vals"])
        assert_array_equal(r.W, golden[f"bdc{i}_w"])
        assert_array_equal(r.Q, golden[f"bdc{i}_q"])
        assert_array_equal(r.edge, golden[f"bdc{i}_edge"])


def test_values_only_bitwise():
    rng = np.random.default_rng(3)
    b = oracle.Bidiag(rng.standard_normal(70), rng.standard_normal(69))
    assert_array_equal(oracle.bdc(b, True, 8).vals, oracle.bdc(b, False, 8).vals)


@pytest.mark.slow
def test_c1_sigma_matches_reference():
    ref = np.load(os.path.join(GOLDEN, "c1_sigma.npz"))
    a = oracle.make_matrix("random", 1024, 1024, seed=1)
    s, _, _ = oracle.svd(a, want_vectors=False)
    assert_array_equal(s, ref["sigma"])
