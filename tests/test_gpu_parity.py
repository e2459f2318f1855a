"""GPU parity: every hot-path entry point on the B200 vs the CPU oracle
(pinned to the reference by tests/test_oracle_golden.py) and vs the golden
reference outputs, with the north-star tolerances:

  max|sigma - sigma_ref| / sigma_max        <= 1e-12 * n
  ||A - U S Vt||_F / (||A||_F * n)          <= 1e-14
  ||U^T U - I||_F / n, ||V V^T - I||_F / n  <= 1e-14

Intermediate factors (bidiagonal, reflectors, QR) are compared with a
relative tolerance scaled by ||A|| (floating point, different summation
order than OpenBLAS)."""

import os

import numpy as np
import pytest
import torch
from numpy.testing import assert_array_equal

import oracle
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

pytestmark = pytest.mark.gpu

SIG_TOL = 1e-12
RES_TOL = 1e-14
ORTH_TOL = 1e-14


def _g():
    import paper_2508_11467_b200 as g

    return g


def _lib_handle():
    from paper_2508_11467_b200 import _lib

    return _lib.load_library()


def check_svd(a, sigma, u, vt, sigma_ref):
    m, n = a.shape
    k = min(m, n)
    nn = max(m, n)
    smax = max(float(np.max(np.abs(sigma_ref))), np.finfo(float).tiny)
    assert np.all(np.diff(sigma) <= 0.0) and np.all(sigma >= 0.0)
    assert np.max(np.abs(sigma - sigma_ref)) / smax <= SIG_TOL * nn
    if u is not None:
        na = np.linalg.norm(a)
        assert np.linalg.norm(a - (u * sigma) @ vt) / (na if na > 0 else 1.0) / nn <= RES_TOL
        assert np.linalg.norm(u.T @ u - np.eye(k)) / k <= ORTH_TOL
        assert np.linalg.norm(vt @ vt.T - np.eye(k)) / k <= ORTH_TOL


def test_native_library_is_loaded(cuda):
    g = _g()
    g.gesdd(np.eye(4))
    maps = open("/proc/self/maps").read()
    assert "libdcsvd_b200.so" in maps
    assert g.launch_count() > 0


def test_gesdd_golden_shapes_and_kinds(cuda, golden):
    g = _g()
    for i in range(int(golden["svd_count"])):
        a = golden[f"svd{i}_a"]
        r = g.gesdd(a)
        check_svd(a, r.sigma, r.u, r.vt, golden[f"svd{i}_sigma"])
        v = g.gesdd(a, g.SVDOptions(want_vectors=False))
        assert v.u is None and v.vt is None
        assert_array_equal(v.sigma, r.sigma)  # values-only bitwise == vector mode


def test_gesdd_input_not_modified(cuda):
    g = _g()
    a = oracle.make_matrix("random", 50, 40, seed=3)
    a0 = a.copy()
    g.gesdd(a)
    assert_array_equal(a, a0)


def test_gesdd_deterministic(cuda):
    g = _g()
    a = oracle.make_matrix("logrand", 300, 200, 1e6, seed=9)
    r1, r2 = g.gesdd(a), g.gesdd(a)
    assert_array_equal(r1.sigma, r2.sigma)
    assert_array_equal(r1.u, r2.u)
    assert_array_equal(r1.vt, r2.vt)


@pytest.mark.parametrize("shape", [(1, 1), (2, 1), (1, 5), (33, 33), (64, 1), (129, 65), (65, 129), (257, 128),
                                   (500, 100), (100, 500), (600, 64)])
def test_gesdd_vs_oracle_shapes(cuda, shape):
    g = _g()
    m, n = shape
    a = oracle.make_matrix("random", m, n, seed=m * 7 + n)
    s, _, _ = oracle.svd(a, want_vectors=False)
    r = g.gesdd(a)
    check_svd(a, r.sigma, r.u, r.vt, s)


def test_gesdd_rank_deficient_and_zero(cuda):
    g = _g()
    rng = np.random.default_rng(4)
    a = rng.standard_normal((80, 5)) @ rng.standard_normal((5, 60))
    r = g.gesdd(a)
    check_svd(a, r.sigma, r.u, r.vt, np.linalg.svd(a, compute_uv=False))
    z = np.zeros((20, 10))
    r = g.gesdd(z)
    assert_array_equal(r.sigma, np.zeros(10))
    assert np.linalg.norm(r.u.T @ r.u - np.eye(10)) <= 1e-13


def test_gesdd_options_paths(cuda):
    g = _g()
    a = oracle.make_matrix("geo", 256, 96, 1e10, seed=5)
    s, _, _ = oracle.svd(a, want_vectors=False)
    for opts in (g.SVDOptions(), g.SVDOptions(ts_crossover=100.0), g.SVDOptions(leaf_size=4, bidiag_block=8),
                 g.SVDOptions(apply_block=16, orgqr_block=32, qr_block=8), g.SVDOptions(deflation_multiple=64.0)):
        r = g.gesdd(a, opts)
        check_svd(a, r.sigma, r.u, r.vt, s)


def test_gesdd_torch_device_path(cuda):
    g = _g()
    a = oracle.make_matrix("random", 300, 200, seed=21)
    t = torch.from_numpy(a).to(cuda)
    r = g.gesdd(t)
    assert r.sigma.is_cuda and r.u.is_cuda and r.vt.is_cuda
    check_svd(a, r.sigma.cpu().numpy(), r.u.cpu().numpy(), r.vt.cpu().numpy(), oracle.svd(a, want_vectors=False)[0])


def test_c1_against_reference_sigma(cuda):
    g = _g()
    ref = np.load(os.path.join(GOLDEN, "c1_sigma.npz"))
    a = oracle.make_matrix("random", 1024, 1024, seed=1)
    r = g.gesdd(a)
    check_svd(a, r.sigma, r.u, r.vt, ref["sigma"])


def test_gebrd_vs_golden(cuda, golden):
    g = _g()
    for i in range(int(golden["gebrd_count"])):
        a = golden[f"gebrd{i}_a"].copy(order="F")
        f = g.gebrd_blocked(a, int(golden[f"gebrd{i}_block"]))
        scale = np.linalg.norm(golden[f"gebrd{i}_a"])
        # entries of B are backward- but not forward-stable: error ~ eps * n * ||A||
        tol = 1e-13 * a.shape[1] * scale
        for name in ("d", "e"):
            assert np.max(np.abs(getattr(f, name) - golden[f"gebrd{i}_{name}"])) <= tol
        for name in ("tauq", "taup"):
            assert np.max(np.abs(getattr(f, name) - golden[f"gebrd{i}_{name}"])) <= 1e-12 * a.shape[1]
        assert np.max(np.abs(a - golden[f"gebrd{i}_packed"])) <= tol
        assert f.packed is a  # in place, like bidiag.py:204
        # B's singular values equal A's
        n = a.shape[1]
        b = np.diag(f.d) + np.diag(f.e, 1)
        sa = np.linalg.svd(golden[f"gebrd{i}_a"], compute_uv=False)
        assert np.max(np.abs(np.linalg.svd(b, compute_uv=False) - sa)) <= 1e-12 * n * sa[0]


@pytest.mark.parametrize("mode", [0, 8, 1])
def test_gebrd_cluster_tail_modes(cuda, golden, mode):
    """The GEBRD tail on a thread-block cluster (16 CTAs by default, 8 forced)
    and the panel-only path give the golden factorization (70^2, 64^2 and
    129x100 run entirely in the cluster kernel; 300x260 switches mid-way)."""
    g = _g()
    lib = _lib_handle()
    lib.dcsvd_debug_gebd2_cluster(mode)
    try:
        for i in range(int(golden["gebrd_count"])):
            a = golden[f"gebrd{i}_a"].copy(order="F")
            f = g.gebrd_blocked(a, int(golden[f"gebrd{i}_block"]))
            tol = 1e-13 * a.shape[1] * np.linalg.norm(golden[f"gebrd{i}_a"])
            assert np.max(np.abs(f.d - golden[f"gebrd{i}_d"])) <= tol
            assert np.max(np.abs(f.e - golden[f"gebrd{i}_e"])) <= tol
            assert np.max(np.abs(a - golden[f"gebrd{i}_packed"])) <= tol
        rng = np.random.default_rng(11)
        a0 = np.asfortranarray(rng.standard_normal((600, 560)))
        a = a0.copy(order="F")
        f = g.gebrd_blocked(a, 32)
        d, e, tq, tp = oracle.gebd2(a0.copy(order="F"))
        sc = np.linalg.norm(a0)
        assert np.max(np.abs(np.abs(f.d) - np.abs(d))) <= 1e-12 * sc
        assert np.max(np.abs(np.abs(f.e) - np.abs(e))) <= 1e-12 * sc
        b = np.diag(f.d) + np.diag(f.e, 1)
        sa = np.linalg.svd(a0, compute_uv=False)
        assert np.max(np.abs(np.linalg.svd(b, compute_uv=False) - sa)) <= 1e-12 * 560 * sa[0]
    finally:
        lib.dcsvd_debug_gebd2_cluster(1)


def test_gebrd_halfwidth_panels(cuda):
    """Mid-size views take 16-wide panels so the two-phase LABRD kernel runs
    (gebrd.cu labrd_panel_width): same factorization as 32-wide panels up to
    rounding (the panel width only regroups the trailing updates), and the
    same singular values through gesdd."""
    g = _g()
    lib = _lib_handle()
    a = g.generate_matrix(g.MatrixSpec("random", 3072, 3000, seed=5), device=True)
    out = {}
    try:
        for mode in (0, 1):
            lib.dcsvd_debug_labrd_halfwidth(mode, 0)
            f = g.gebrd_blocked(a.clone())
            s = g.gesdd(a, g.SVDOptions(want_vectors=False)).sigma
            s = s.cpu().numpy() if isinstance(s, torch.Tensor) else np.asarray(s)
            out[mode] = (f.d.abs().cpu().numpy(), f.e.abs().cpu().numpy(), s)
    finally:
        lib.dcsvd_debug_labrd_halfwidth(1, 0)
    sc = float(torch.linalg.norm(a))
    for i in range(2):
        assert np.max(np.abs(out[1][i] - out[0][i])) <= 1e-12 * sc
    assert np.max(np.abs(out[1][2] - out[0][2])) <= SIG_TOL * 3072 * out[0][2][0]


def test_ormbr_batched_t_matches_per_block(cuda):
    """ORMBR with op(T) of all full CWY blocks precomputed in batched launches
    (qr.cu ormbr_run) gives the per-block result up to rounding: 700^2 has five
    full 128-wide blocks per side plus a partial one."""
    g = _g()
    lib = _lib_handle()
    a = g.generate_matrix(g.MatrixSpec("random", 700, 700, seed=4), device=True)
    out = {}
    try:
        for pre in (0, 1):
            lib.dcsvd_debug_ormbr_pre(pre)
            r = g.gesdd(a)
            out[pre] = (r.sigma.clone(), r.u.clone(), r.vt.clone())
    finally:
        lib.dcsvd_debug_ormbr_pre(1)
    assert torch.equal(out[0][0], out[1][0])  # sigma does not depend on the back-transform
    assert float((out[0][1] - out[1][1]).abs().max()) <= 1e-13
    assert float((out[0][2] - out[1][2]).abs().max()) <= 1e-13


@pytest.mark.parametrize("rpl", [2, 4, 8])
def test_labrd2_geometries_agree(cuda, rpl):
    """The two-phase LABRD kernel gives the same bidiagonal for every block
    geometry it can take (rows per lane forced through the debug knob; the
    default prefers 4), within rounding of the different reduction trees."""
    g = _g()
    lib = _lib_handle()
    a = g.generate_matrix(g.MatrixSpec("random", 1536, 1400, seed=6), device=True)
    ref = g.gebrd_blocked(a.clone())
    try:
        lib.dcsvd_debug_labrd2_rpl(rpl)
        f = g.gebrd_blocked(a.clone())
    finally:
        lib.dcsvd_debug_labrd2_rpl(0)
    sc = float(torch.linalg.norm(a))
    assert float((f.d.abs() - ref.d.abs()).abs().max()) <= 1e-12 * sc
    assert float((f.e.abs() - ref.e.abs()).abs().max()) <= 1e-12 * sc


def test_gebrd_unblocked_and_panel(cuda):
    g = _g()
    rng = np.random.default_rng(6)
    a = np.asfortranarray(rng.standard_normal((40, 30)))
    a2 = a.copy(order="F")
    f = g.gebrd_unblocked(a)
    d, e, tq, tp = oracle.gebd2(a2)
    assert np.max(np.abs(f.d - d)) <= 1e-12 * np.linalg.norm(a2)
    # one LABRD panel vs the oracle panel
    b = np.asfortranarray(rng.standard_normal((90, 70)))
    b2 = b.copy(order="F")
    work = g.PanelWorkspace.allocate(90, 70, 8)
    dd, ee, t1, t2 = (np.zeros(8) for _ in range(4))
    p, q = g.labrd_panel(b, 8, work, dd, ee, t1, t2)
    od, oe, o1, o2 = (np.zeros(8) for _ in range(4))
    P, Q = oracle.labrd(b2, 8, od, oe, o1, o2)
    sc = np.linalg.norm(b2)
    assert np.max(np.abs(dd - od)) <= 1e-12 * sc and np.max(np.abs(ee - oe)) <= 1e-12 * sc
    assert np.max(np.abs(p - P)) <= 1e-11 * sc and np.max(np.abs(q - Q)) <= 1e-11 * sc
    assert np.max(np.abs(b - b2)) <= 1e-11 * sc


def test_qr_vs_golden(cuda, golden):
    g = _g()
    for i in range(int(golden["qr_count"])):
        a = golden[f"qr{i}_a"].copy(order="F")
        b, ob = (int(x) for x in golden[f"qr{i}_blocks"])
        f = g.geqrf_blocked(a, b)
        sc = np.linalg.norm(golden[f"qr{i}_a"])
        assert np.max(np.abs(a - golden[f"qr{i}_packed"])) <= 1e-12 * sc
        assert np.max(np.abs(f.tau - golden[f"qr{i}_tau"])) <= 1e-12
        q = g.orgqr(f, a.shape[1], ob)
        assert np.max(np.abs(q - golden[f"qr{i}_q"])) <= 1e-12


def test_ormbr_vs_oracle(cuda):
    g = _g()
    rng = np.random.default_rng(8)
    for m, n in ((70, 70), (100, 60), (200, 129)):
        a = np.asfortranarray(rng.standard_normal((m, n)))
        d, e, tq, tp = oracle.gebrd(a, 32)
        f = g.BidiagonalFactorization(a, d, e, tq, tp)
        for trans in (False, True):
            c = np.asfortranarray(rng.standard_normal((m, 37)))
            c2 = c.copy(order="F")
            g.ormqr_like(g.column_reflectors(f), c, transpose=trans)
            oracle.apply_u1(a, tq, c2, 64, trans=trans)
            assert np.max(np.abs(c - c2)) <= 1e-12 * np.linalg.norm(c2)
            v = np.asfortranarray(rng.standard_normal((41, n)))
            v2 = v.copy(order="F")
            g.ormlq_like(g.row_reflectors(f), v, transpose=trans)
            oracle.apply_v1t(a, tp, v2, 64, trans=trans)
            assert np.max(np.abs(v - v2)) <= 1e-12 * np.linalg.norm(v2)


def _bdc_check(g, d, e, bord, leaf, ref_vals=None):
    prob = g.BidiagonalProblem(d, e, bordered=bord)
    r = g.bdsdc(prob, leaf=leaf)
    n = prob.n
    o = oracle.bdc(oracle.Bidiag(d, e, bord), leaf=leaf)
    ref = o.vals if ref_vals is None else ref_vals
    scale = max(float(ref[0]) if n else 1.0, 1.0)
    if n:
        assert np.max(np.abs(r.dvals - ref)) <= SIG_TOL * max(n, 1) * scale
        b = prob.dense()
        assert np.linalg.norm(b - (r.w * r.dvals) @ r.qfull[:, :n].T) <= 1e-13 * n * scale
        assert np.linalg.norm(r.w.T @ r.w - np.eye(n)) <= 1e-13 * n
    assert np.linalg.norm(r.qfull.T @ r.qfull - np.eye(prob.ncols)) <= 1e-13 * max(n, 1)
    v = g.bdsdc(prob, want_vectors=False, leaf=leaf)
    assert v.w is None and v.qfull is None
    assert_array_equal(v.dvals, r.dvals)  # values-only bitwise (bdc.py:14-21)
    assert_array_equal(v.edge_rows, r.edge_rows)
    return r


def test_bdsdc_vs_golden(cuda, golden):
    g = _g()
    for i in range(int(golden["bdc_count"])):
        bord, leaf = (int(x) for x in golden[f"bdc{i}_meta"])
        _bdc_check(g, golden[f"bdc{i}_d"], golden[f"bdc{i}_e"], bool(bord), leaf, golden[f"bdc{i}_vals"])


@pytest.mark.parametrize("leaf", [1, 2, 4, 32])
@pytest.mark.parametrize("bordered", [False, True])
def test_bdsdc_sizes(cuda, leaf, bordered):
    g = _g()
    rng = np.random.default_rng(57)
    for n in (0, 1, 2, 3, 5, 9, 21, 40, 100):
        if n == 0 and not bordered:
            continue
        d = rng.standard_normal(n)
        e = rng.standard_normal(n if bordered else max(n - 1, 0))
        _bdc_check(g, d, e, bordered, leaf)


def test_bdsdc_deflation_stress(cuda):
    g = _g()
    n = 300
    _bdc_check(g, np.ones(n), np.zeros(n - 1), False, 8)                          # all duplicates
    _bdc_check(g, np.repeat([1.0, 2.0, 3.0], 100), np.full(n - 1, 1e-9), False, 32)  # clusters
    dg = np.float_power(10.0, -np.arange(40, dtype=float))
    _bdc_check(g, dg, 0.5 * dg[:-1], False, 4)                                    # graded
    c4 = np.load(os.path.join(GOLDEN, "c4_n1024.npz"))
    r = _bdc_check(g, c4["d"], c4["e"], False, 32, c4["sigma_ref"])
    assert np.max(np.abs(r.dvals - c4["sigma_prescribed"])) <= 1e-12 * 1024 * 2


def test_bdsdc_diagonal_signed_permutation(cuda):
    g = _g()
    r = g.bdsdc(g.BidiagonalProblem([3.0, -1.0, 2.0], np.zeros(2)), leaf=1)
    np.testing.assert_allclose(r.dvals, [3.0, 2.0, 1.0], rtol=1e-15)
    np.testing.assert_allclose(np.abs(r.w), np.abs(r.qfull), atol=1e-15)


def test_errors_map_to_reference_exceptions(cuda):
    g = _g()
    with pytest.raises(ValueError):
        g.gesdd(np.zeros((0, 3)))
    with pytest.raises(ValueError):
        g.gebrd_blocked(np.zeros((3, 5)))
    with pytest.raises(ValueError):
        g.bdsdc(g.BidiagonalProblem([1.0], np.zeros(0)), leaf=0)
    with pytest.raises(ValueError):
        g.geqrf_blocked(np.zeros((3, 5)))


def test_matmul_accumulate(cuda):
    g = _g()
    rng = np.random.default_rng(1)
    for (m, n, k, ta, tb) in ((100, 70, 50, False, False), (130, 257, 64, False, True),
                              (64, 300, 1000, True, False), (33, 17, 9, True, True)):
        a = rng.standard_normal((k, m) if ta else (m, k))
        b = rng.standard_normal((n, k) if tb else (k, n))
        c = np.asfortranarray(rng.standard_normal((m, n)))
        ref = 0.5 * c + 2.0 * ((a.T if ta else a) @ (b.T if tb else b))
        g.matmul_accumulate(2.0, a, ta, b, tb, 0.5, c)
        assert np.max(np.abs(c - ref)) <= 1e-13 * k * np.max(np.abs(ref))
    c = np.full((4, 4), np.nan, order="F")
    g.matmul_accumulate(1.0, np.eye(4), False, np.eye(4), False, 0.0, c)  # beta = 0 never reads C
    assert_array_equal(c, np.eye(4))


def test_matvec_accumulate(cuda):
    """densecore.py:96-111 through dcsvd_dgemv: random shapes and both
    transposes against numpy (test_densecore.py:94-106), beta = 0 never reads
    y (:108-111), shape mismatch raises (:113-116), plus a long GEMV."""
    g = _g()
    rng = np.random.default_rng(7)
    for _ in range(20):
        trans_a = bool(rng.integers(0, 2))
        m, k = (int(v) for v in rng.integers(1, 9, size=2))
        a = rng.standard_normal((k, m) if trans_a else (m, k))
        x = rng.standard_normal(k)
        y = rng.standard_normal(m)
        alpha, beta = rng.standard_normal(2)
        expect = beta * y + alpha * ((a.T if trans_a else a) @ x)
        g.matvec_accumulate(alpha, a, trans_a, x, beta, y)
        np.testing.assert_allclose(y, expect, rtol=1e-13, atol=1e-13)
    y = np.full(2, np.nan)
    g.matvec_accumulate(1.0, np.eye(2), False, np.ones(2), 0.0, y)
    assert_array_equal(y, np.ones(2))
    with pytest.raises(ValueError):
        g.matvec_accumulate(1.0, np.eye(2), False, np.zeros(3), 0.0, np.zeros(2))
    for trans_a in (False, True):
        a = np.asfortranarray(rng.standard_normal((3000, 700)))
        x = rng.standard_normal(3000 if trans_a else 700)
        y = rng.standard_normal(700 if trans_a else 3000)
        expect = 0.25 * y - 1.5 * ((a.T if trans_a else a) @ x)
        g.matvec_accumulate(-1.5, a, trans_a, x, 0.25, y)
        assert np.max(np.abs(y - expect)) <= 1e-13 * 3000 * np.max(np.abs(expect))


def test_gesdd_batched(cuda):
    g = _g()
    mats = [oracle.make_matrix("random", 128, 128, seed=1000 + i) for i in range(5)]
    res = g.gesdd_batched(mats)
    for a, r in zip(mats, res):
        check_svd(a, r.sigma, r.u, r.vt, np.linalg.svd(a, compute_uv=False))


@pytest.mark.slow
def test_c4_fixture_heavy_deflation(cuda):
    """BASELINE config 4: n = 16384 bidiagonal with 8 singular-value clusters
    (tests/golden/c4_n16384.npz, sigma_ref from the reference bdsdc)."""
    g = _g()
    z = np.load(os.path.join(GOLDEN, "c4_n16384.npz"))
    n = z["d"].size
    prob = g.BidiagonalProblem(torch.from_numpy(z["d"]).cuda(), torch.from_numpy(z["e"]).cuda())
    r = g.bdsdc(prob)
    vals = r.dvals.cpu().numpy()
    assert np.max(np.abs(vals - z["sigma_ref"])) / z["sigma_ref"][0] <= SIG_TOL * n
    assert np.max(np.abs(vals - z["sigma_prescribed"])) <= 1e-12 * n
    eye = torch.eye(n, dtype=torch.float64, device=r.w.device)
    assert torch.linalg.matrix_norm(r.w.t() @ r.w - eye).item() / n <= ORTH_TOL
    assert torch.linalg.matrix_norm(r.qfull.t() @ r.qfull - eye).item() / n <= ORTH_TOL
    # B = W diag(s) Q^T, checked through B Q = W diag(s) on the device
    d = prob.d
    e = prob.e
    BQ = d[:, None] * r.qfull
    BQ[:-1] += e[:-1, None] * r.qfull[1:]
    resid = torch.linalg.matrix_norm(BQ - r.w * r.dvals).item()
    assert resid / (float(vals[0]) * n) <= RES_TOL
    v = g.bdsdc(prob, want_vectors=False)
    assert torch.equal(v.dvals, r.dvals)


def _sigma_fixture(tag):
    """Reference sigma on the same input bytes (tests/golden/make_large_sigma.py:
    the real reference's gesdd values-only on MatrixSpec('random', ...))."""
    p = os.path.join(GOLDEN, f"{tag}_sigma.npz")
    if not os.path.exists(p):
        pytest.skip(f"{tag}_sigma.npz not generated")
    return np.load(p)


@pytest.mark.slow
def test_c2_scale_square_8192(cuda):
    """Headline config C2 at full size on the exact reference input
    (MatrixSpec('random', 8192, 8192, seed=2), bit-identical GPU Philox):
    sigma against the REAL reference's sigma on the same bytes
    (tests/golden/c2_sigma.npz) within 1e-12 n, residual / orthogonality on
    the device, values-only sigma bitwise equal to vector-mode sigma."""
    g = _g()
    n = 8192
    fx = _sigma_fixture("c2")
    a = g.generate_matrix(g.MatrixSpec("random", n, n, seed=2), device=True)
    r = g.gesdd(a)
    _check_report(g, a, r, fx["sigma"], n)
    v = g.gesdd(a, g.SVDOptions(want_vectors=False))
    assert torch.equal(v.sigma, r.sigma)


@pytest.mark.parametrize("k", [1, 37, 64, 100, 128])
@pytest.mark.parametrize("tb", [False, True])
@pytest.mark.parametrize("m", [2000, 2001])
@pytest.mark.parametrize("ab", [(-1.0, 0.75), (-1.0, 1.0), (1.0, 1.0)])
def test_rank_k_update_kernel(cuda, k, tb, m, ab):
    """Large rank-k updates take the streaming kernel (K <= 64) or the
    warp-specialized TMA tensor-map kernel (K > 64; gemm.cu); compare with a
    plain torch fp64 product.  m = 2001 leaves an odd-row last tile (cp.async
    fallback / TMA zero fill).  (alpha, beta) = (+-1, 1) takes the folded
    accumulator path of the TMA kernel, others its general epilogue."""
    g = _g()
    alpha, beta = ab
    torch.manual_seed(k)
    n = 1500
    a = torch.randn(m, k, dtype=torch.float64, device=cuda)
    b = torch.randn(n, k, dtype=torch.float64, device=cuda) if tb else torch.randn(k, n, dtype=torch.float64, device=cuda)
    c = torch.randn(n, m, dtype=torch.float64, device=cuda).t()  # column-major m x n
    ref = beta * c + alpha * (a @ (b.t() if tb else b))
    a_cm = a.t().contiguous().t()
    b_cm = b.t().contiguous().t()
    g.matmul_accumulate(alpha, a_cm, False, b_cm, tb, beta, c)
    assert (c - ref).abs().max().item() <= 1e-12 * max(k, 1)


@pytest.mark.parametrize("ws", [(1, 1), (3, 1), (0, 1), (0, 0)])
def test_rank_k_kernels_agree_on_pipeline_shapes(cuda, ws):
    """The ORMBR-shaped rank-128 update (8192 x 4096, C -= Y X) through the
    persistent TMA tile kernel with C staged in shared memory (default), its
    register-prefetch variant (3), the 3-group TMA kernel (dgemm_ws 0) and the
    cp.async streaming kernel (both off), against torch."""
    g = _g()
    lib = _lib_handle()
    torch.manual_seed(5)
    m, n, k = 8192, 4096, 128
    a = torch.randn(k, m, dtype=torch.float64, device=cuda).t()
    b = torch.randn(n, k, dtype=torch.float64, device=cuda).t()
    c = torch.randn(n, m, dtype=torch.float64, device=cuda).t()
    ref = c - a @ b
    lib.dcsvd_debug_dgemm_ws(ws[0])
    lib.dcsvd_debug_rankk_ws(ws[1])
    try:
        g.matmul_accumulate(-1.0, a, False, b, False, 1.0, c)
    finally:
        lib.dcsvd_debug_dgemm_ws(1)
        lib.dcsvd_debug_rankk_ws(1)
    assert (c - ref).abs().max().item() <= 1e-12 * k


def test_gesdd_batched_high_concurrency(cuda):
    """12 concurrent sub-contexts: each LABRD grid has ~12 CTAs, which takes
    the global-memory path for the P/Q slice caches.  Inputs are C5 items
    (seeds 1000..1011); sigma against the real reference's on the same bytes."""
    g = _g()
    fx = _sigma_fixture("c5")
    mats = [g.generate_matrix(g.MatrixSpec("random", 2048, 2048, seed=1000 + i), device=True) for i in range(12)]
    res = g.gesdd_batched(mats, concurrency=12)
    for i, (a, r) in enumerate(zip(mats, res)):
        _check_report(g, a, r, fx["sigma"][i], 2048)


# ---- stage pieces of the reference API (KATs from pkg/tests, oracle parity) ----

def test_householder_and_givens_kats(cuda):
    g = _g()
    r = g.householder_generate(3.0, np.array([4.0]))      # test_densecore.py:119-123
    assert r.pivot_value == -5.0 and abs(r.tau - 1.6) <= 1e-15
    np.testing.assert_allclose(r.essential, [0.5], rtol=1e-15)
    r0 = g.householder_generate(-2.0, np.zeros(3))         # zero tail: identity
    assert r0.tau == 0.0 and r0.pivot_value == -2.0
    rot, rr = g.givens_generate(3.0, 4.0)                  # test_densecore.py:168-172
    np.testing.assert_allclose((rot.c, rot.s, rr), (0.6, 0.8, 5.0), rtol=1e-15)
    rot, rr = g.givens_generate(0.0, 0.0)
    assert (rot.c, rot.s, rr) == (1.0, 0.0, 0.0)
    rng = np.random.default_rng(3)
    x = rng.standard_normal(300)
    r = g.householder_generate(0.7, x)
    tau, beta, ess = oracle.larfg(0.7, x)
    assert abs(r.tau - tau) <= 1e-14 and abs(r.pivot_value - beta) <= 1e-13
    assert np.max(np.abs(r.essential - ess)) <= 1e-14


@pytest.mark.parametrize("side", ["left", "right"])
@pytest.mark.parametrize("trans", [False, True])
def test_triangular_solve(cuda, side, trans):
    g = _g()
    rng = np.random.default_rng(5)
    t = np.triu(rng.standard_normal((40, 40))) + 5.0 * np.eye(40)
    b = np.asfortranarray(rng.standard_normal((40, 17) if side == "left" else (17, 40)))
    ref = b.copy()
    g.triangular_solve(t, b, side=side, trans=trans)
    tt = t.T if trans else t
    back = tt @ b if side == "left" else b @ tt
    assert np.max(np.abs(back - ref)) <= 1e-12
    with pytest.raises(np.linalg.LinAlgError):
        tz = t.copy()
        tz[3, 3] = 0.0
        g.triangular_solve(tz, b.copy(order="F"), side=side)


def test_tinv_and_block_reflectors(cuda):
    g = _g()
    y = np.array([[1.0, 0.0], [1.0, 1.0], [0.0, 1.0]])    # test_qrblock.py:69-79
    np.testing.assert_allclose(g.build_tinv(y, np.array([1.0, 2.0])), [[1.0, 1.0], [0.0, 0.5]], atol=1e-15)
    rng = np.random.default_rng(9)
    a = np.asfortranarray(rng.standard_normal((90, 7)))
    tau = oracle.geqrf(a, 7)
    y = oracle.cwy_y(a, tau)
    tinv = g.build_tinv(y, tau)
    np.testing.assert_allclose(tinv, oracle.cwy_tinv(y, tau), atol=1e-13)
    blk = g.CompactWYBlock(y, tinv)
    for trans in (False, True):
        c = np.asfortranarray(rng.standard_normal((90, 33)))
        c2 = c.copy(order="F")
        g.apply_block_reflector_left(blk, c, transpose=trans)
        oracle.cwy_apply_left(y, oracle.cwy_tinv(y, tau), c2, trans)
        assert np.max(np.abs(c - c2)) <= 1e-13 * np.linalg.norm(c2)
        c = np.asfortranarray(rng.standard_normal((21, 90)))
        c2 = c.copy(order="F")
        g.apply_block_reflector_right(blk, c, transpose=trans)
        oracle.cwy_apply_right(y, oracle.cwy_tinv(y, tau), c2, trans)
        assert np.max(np.abs(c - c2)) <= 1e-13 * np.linalg.norm(c2)


def test_geqrf_panel(cuda):
    g = _g()
    rng = np.random.default_rng(12)
    a = np.asfortranarray(rng.standard_normal((500, 24)))
    a2 = a.copy(order="F")
    tau = np.zeros(24)
    g.geqrf_panel(a, tau)
    tau2 = np.zeros(24)
    oracle.geqr2(a2, tau2)
    assert np.max(np.abs(a - a2)) <= 1e-12 * np.linalg.norm(a2)
    assert np.max(np.abs(tau - tau2)) <= 1e-13


def _secular_system(rng, n):
    d = np.concatenate(([0.0], np.sort(rng.uniform(0.05, 3.0, n - 1))))
    z = rng.standard_normal(n)
    z[np.abs(z) < 0.02] = 0.1
    return d, z


def test_secular_pieces_vs_oracle(cuda):
    g = _g()
    # golden ratio (test_bdc.py:284-303)
    sysg = g.SecularSystem(np.array([0.0, 1.0]), np.array([1.0, 1.0]), np.sqrt(3.0))
    roots = g.solve_all_roots(sysg)
    np.testing.assert_allclose(roots.omega ** 2, [(3 - np.sqrt(5)) / 2, (3 + np.sqrt(5)) / 2], rtol=1e-14)
    zt = g.recompute_z(sysg, roots)
    _, vmat = g.secular_vectors(sysg, roots, zt)
    direction = np.array([-2.618034, 1.618034]) / np.linalg.norm([-2.618034, 1.618034])
    np.testing.assert_allclose(vmat[:, 0] * np.sign(vmat[0, 0] * direction[0]), direction, rtol=1e-6)
    rng = np.random.default_rng(51)
    for n in (1, 2, 5, 17, 64, 300):
        d, z = _secular_system(rng, n)
        s = g.SecularSystem(d, z, float(np.sqrt(d[-1] ** 2 + z @ z)))
        r = g.solve_all_roots(s)
        om, anc, mu = oracle.secular_roots(d, z)
        assert np.max(np.abs(r.omega - om)) <= 1e-13 * max(om.max(), 1.0)
        for i in range(n):
            a, m = int(r.anchor[i]), r.mu[i]
            den = (d - d[a]) * (d + d[a]) - m
            terms = z ** 2 / den
            assert abs(1.0 + terms.sum()) <= 1e-12 * (1.0 + np.abs(terms).sum())
        if n >= 3:
            assert g.solve_secular(s, 2) == (float(r.omega[2]), int(r.anchor[2]), float(r.mu[2]))
        zt = g.recompute_z(s, r)
        zt2 = oracle.loewner_z(d, z, r.anchor, r.mu)
        assert np.max(np.abs(zt - zt2)) <= 1e-12 * np.max(np.abs(zt2))
        u, v = g.secular_vectors(s, r, zt)
        assert np.linalg.norm(u.T @ u - np.eye(n)) <= 1e-13 * n
        assert np.linalg.norm(v.T @ v - np.eye(n)) <= 1e-13 * n


def test_split_and_leaf(cuda):
    g = _g()
    left, right, alpha, beta = g.split(g.BidiagonalProblem([1.0, 2.0, 3.0, 4.0], [5.0, 6.0, 7.0]))
    assert left.n == 1 and left.bordered and right.n == 2 and not right.bordered and (alpha, beta) == (2.0, 6.0)
    r = g.bdsqr_base(g.BidiagonalProblem([-3.0], np.zeros(0)))     # test_bdc.py:62-66
    assert_array_equal(r.dvals, [3.0])
    assert_array_equal(r.w, [[-1.0]])
    rng = np.random.default_rng(43)
    for bordered in (False, True):
        p = g.BidiagonalProblem(rng.standard_normal(11), rng.standard_normal(11 if bordered else 10), bordered)
        r = g.bdsqr_base(p)
        o = oracle.leaf_svd(oracle.Bidiag(p.d, p.e, bordered))
        assert np.all(np.diff(r.dvals) >= 0.0)
        assert np.max(np.abs(r.dvals - o.vals)) <= 1e-13 * max(o.vals.max(), 1.0)
        assert_array_equal(r.edge_rows[0], r.qfull[0, :])
        assert_array_equal(r.edge_rows[1], r.qfull[-1, :])


# ---------------------------------------------------------------------------
# standalone merge stages: build_z, deflate, merge_vectors (bdc.py:382-747)

def test_deflate_kats(cuda):
    g = _g()
    out = g.deflate([0.0, 1.0, 1.0], [1.0, 0.6, 0.8])          # test_bdc.py:208-222
    assert_array_equal(out.z, [1.0, 1.0, 0.0])
    assert_array_equal(out.kept, [0, 1])
    assert_array_equal(out.deflated, [2])
    assert_array_equal(out.deflated_values, [1.0])
    (i, j, rot), = out.applied_rotations
    assert (i, j) == (1, 2)
    np.testing.assert_allclose((rot.c, rot.s), (0.6, 0.8), rtol=1e-15)
    assert_array_equal(out.system.d, [0.0, 1.0])
    assert_array_equal(out.system.z, [1.0, 1.0])
    out = g.deflate([0.0, 3.0, 1.0, 2.0], [1.0, 0.5, 0.5, 0.5])
    assert_array_equal(out.d, [0.0, 1.0, 2.0, 3.0])
    assert_array_equal(out.permutation, [0, 2, 3, 1])
    out = g.deflate([0.0, 1.0, 2.0], [1.0, 1e-20, 1.0])        # tiny z
    assert_array_equal(out.kept, [0, 2])
    assert_array_equal(out.deflated, [1])
    out = g.deflate([0.0, 1.0], [0.0, 1.0])                     # z0 clamp
    assert 0 in out.kept and out.system.z[0] != 0.0 and abs(out.system.z[0]) <= 16.0 * np.finfo(float).eps
    rng = np.random.default_rng(48)                              # pair with the zero entry
    right = np.asfortranarray(rng.standard_normal((3, 3)))
    left = np.asfortranarray(rng.standard_normal((3, 3)))
    left0, right0 = left.copy(), right.copy()
    out = g.deflate([0.0, 1e-18, 1.0], [0.6, 0.8, 1.0], left, right)
    assert_array_equal(out.deflated_values, [0.0])
    np.testing.assert_allclose(out.z[0], 1.0, rtol=1e-15)
    assert_array_equal(left, left0)
    assert not np.array_equal(right, right0)
    d = np.array([0.0, 1.0, 1.0])
    z = np.array([1.0, 0.6, 0.8])
    g.deflate(d, z)
    assert_array_equal(d, [0.0, 1.0, 1.0])
    with pytest.raises(ValueError):
        g.deflate([1.0, 2.0], [1.0, 1.0])


def _merge_case(rng, n, clustered):
    d = np.concatenate(([0.0], rng.uniform(0.1, 2.0, n - 1)))
    if clustered:
        d[1:] = np.round(d[1:] * 4) / 4                          # exact duplicates -> Givens deflation
    z = rng.standard_normal(n)
    z[rng.random(n) < 0.2] = 1e-19                               # tiny z -> outright deflation
    perm = rng.permutation(n - 1) + 1
    d[1:], z[1:] = d[perm], z[perm]
    lcls = rng.integers(0, 4, n).astype(np.int64)
    rcls = rng.integers(1, 4, n).astype(np.int64)
    return d, z, lcls, rcls


@pytest.mark.parametrize("n", [2, 7, 40, 300])
@pytest.mark.parametrize("clustered", [False, True])
def test_deflate_vs_oracle(cuda, n, clustered):
    g = _g()
    rng = np.random.default_rng(1000 + n + clustered)
    d, z, lcls, rcls = _merge_case(rng, n, clustered)
    L = np.asfortranarray(rng.standard_normal((n, n)))
    R = np.asfortranarray(rng.standard_normal((n + 1, n)))
    E = np.asfortranarray(rng.standard_normal((2, n)))
    L2, R2, E2, lc2, rc2 = L.copy(order="F"), R.copy(order="F"), E.copy(order="F"), lcls.copy(), rcls.copy()
    out = g.deflate(d, z, L, R, edge_rows=E, left_classes=lcls, right_classes=rcls)
    ref = oracle.deflate_entries(d, z, L2, R2, E2, lc2, rc2)
    assert_array_equal(out.permutation, ref["perm"])
    assert_array_equal(out.kept, ref["kept"])
    assert_array_equal(out.deflated, ref["deflated"])
    assert [(i, j) for i, j, _ in out.applied_rotations] == [(p, q) for p, q, _, _ in ref["rotations"]]
    np.testing.assert_allclose(out.deflated_values, ref["dvals"], rtol=0, atol=0)
    np.testing.assert_allclose(out.d, ref["d"], rtol=0, atol=0)
    np.testing.assert_allclose(out.z, ref["z"], rtol=1e-15, atol=0)
    assert_array_equal(lcls, lc2)
    assert_array_equal(rcls, rc2)
    for a, b in ((L, L2), (R, R2), (E, E2)):
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-15 * np.abs(b).max())
    assert out.system.n == ref["kept"].size


def test_build_z_and_merge_vectors_vs_oracle(cuda):
    g = _g()
    rng = np.random.default_rng(45)
    for n, bordered in ((9, False), (12, True), (40, True)):
        prob = g.BidiagonalProblem(rng.standard_normal(n), rng.standard_normal(n if bordered else n - 1), bordered)
        lp, rp, _, _ = g.split(prob)
        left, right = g.bdsqr_base(lp), g.bdsqr_base(rp)
        d, z, coupling = g.build_z(prob, left, right)
        OL = oracle.NodeSVD(left.dvals, left.w, left.qfull, left.edge_rows)
        OR = oracle.NodeSVD(right.dvals, right.w, right.qfull, right.edge_rows)
        od, oz, ocp = oracle.merge_inputs(oracle.Bidiag(prob.d, prob.e, bordered), OL, OR)
        assert_array_equal(d, od)
        np.testing.assert_allclose(z, oz, rtol=1e-15, atol=0)
        assert (coupling is None) == (ocp is None)
        if bordered:
            np.testing.assert_allclose((coupling.c, coupling.s), ocp, rtol=1e-15)
    for rows, K, nout in ((30, 12, 12), (257, 100, 90)):
        cols = np.asfortranarray(rng.standard_normal((rows, K + 5)))
        cls = rng.integers(0, 4, K + 5)
        cls[cls == 0] = 1
        cls[3] = 0                                                # one unit column
        kept = np.sort(rng.choice(K + 5, K, replace=False))
        small = np.asfortranarray(rng.standard_normal((K, nout)))
        mid = rows // 2
        out = g.dc._structured_product(torch.from_numpy(cols).cuda(), cls, kept,
                                       torch.from_numpy(np.ascontiguousarray(small.T)).cuda().t(), mid, mid + 1, mid)
        ref = oracle.dc_ref._blocked_product(cols, cls, kept, small, mid, mid + 1, mid)
        np.testing.assert_allclose(out.cpu().numpy(), ref, rtol=0, atol=1e-13 * np.abs(ref).max())


def test_merge_from_standalone_stages(cuda):
    """One merge assembled from build_z -> deflate -> roots -> z~ -> vectors ->
    merge_vectors reproduces the node's singular values and vectors."""
    g = _g()
    rng = np.random.default_rng(49)
    for n, bordered in ((17, False), (33, True)):
        prob = g.BidiagonalProblem(rng.standard_normal(n), rng.standard_normal(n if bordered else n - 1), bordered)
        lp, rp, _, _ = g.split(prob)
        left, right = g.bdsqr_base(lp), g.bdsqr_base(rp)
        nl, nr = left.n, right.n
        d, z, cp = g.build_z(prob, left, right)
        ncols = prob.ncols
        lpre = np.zeros((n, n), order="F")
        lpre[nl, 0] = 1.0
        lpre[:nl, 1:1 + nl] = left.w
        lpre[nl + 1:, 1 + nl:] = right.w
        rpre = np.zeros((ncols, n), order="F")
        q1 = np.zeros(ncols)
        q1[:nl + 1] = left.qfull[:, nl]
        if bordered:
            q2 = np.zeros(ncols)
            q2[nl + 1:] = right.qfull[:, nr]
            rpre[:, 0] = cp.c * q1 + cp.s * q2
        else:
            rpre[:, 0] = q1
        rpre[:nl + 1, 1:1 + nl] = left.qfull[:, :nl]
        rpre[nl + 1:, 1 + nl:] = right.qfull[:, :nr]
        rcls = np.full(n, 3 if bordered else 1)
        rcls[1:1 + nl], rcls[1 + nl:] = 1, 2
        lcls = np.zeros(n, dtype=np.int64)
        lcls[1:1 + nl], lcls[1 + nl:] = 1, 2
        out = g.deflate(d, z, lpre, rpre, left_classes=lcls, right_classes=rcls)
        roots = g.solve_all_roots(out.system)
        zt = g.recompute_z(out.system, roots)
        umat, vmat = g.secular_vectors(out.system, roots, zt)
        w_cols, q_cols = g.merge_vectors(out, umat, vmat, lpre, rpre, lcls, rcls, nl)
        vals = np.concatenate([roots.omega, out.deflated_values])
        B = prob.dense()
        ref = np.linalg.svd(B, compute_uv=False)
        np.testing.assert_allclose(np.sort(vals)[::-1], ref, rtol=0, atol=1e-13 * ref[0])
        # B q_i = sigma_i w_i for every assembled column pair
        np.testing.assert_allclose(B @ q_cols[:, :], w_cols * vals, rtol=0, atol=1e-12 * ref[0])


# ---------------------------------------------------------------------------
# harness on the GPU: Philox stream, generators, accuracy, CLI (harness.py:69-343)

def test_philox_stream_bitwise(cuda):
    from paper_2508_11467_b200 import harness as hz

    u = hz.philox_stream(0, 4).cpu().numpy()                     # test_harness.py:24-37 pin
    assert_array_equal(u, [0.011546754286331617, 0.24154919656271817, 0.11142585551493828, 0.56441462160713374])
    for seed in (1, 7, 2**40 + 3, 2**64 + 11):
        for off, cnt in ((0, 1), (0, 4099), (3, 1000), (5, 17)):
            ref = np.random.Philox(key=seed).random_raw(off + cnt)[off:]
            ref_u = ((ref >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0 ** -53
            assert_array_equal(hz.philox_stream(seed, cnt, off).cpu().numpy(), ref_u)
    z = hz.philox_stream(0, 2, normal=True).cpu().numpy()        # test_harness.py:39-41 pin
    np.testing.assert_allclose(z, [0.15853383451844044, 2.9828792826170751], rtol=4e-16)
    for seed, cnt, off in ((5, 3, 0), (11, 200001, 0), (3, 1001, 7)):
        ref = oracle.gen_ref.WordStream(seed)
        if off:
            ref.uniforms(off)
        np.testing.assert_allclose(hz.philox_stream(seed, cnt, off, normal=True).cpu().numpy(), ref.normals(cnt),
                                   rtol=0, atol=4e-15)


def test_generate_matrix_vs_oracle(cuda):
    g = _g()
    a = g.generate_matrix(g.MatrixSpec("random", 5, 3, seed=4))  # test_harness.py:73-79
    assert a.flags.f_contiguous and a.shape == (5, 3)
    assert_array_equal(a, oracle.make_matrix("random", 5, 3, seed=4))
    assert_array_equal(g.generate_matrix(g.MatrixSpec("random", 300, 257, seed=2)),
                       oracle.make_matrix("random", 300, 257, seed=2))
    for kind, m, n, cond, seed in (("logrand", 40, 30, 1e8, 3), ("arith", 33, 33, 1e2, 1), ("geo", 20, 45, 1e10, 9),
                                   ("logrand", 200, 130, 1e6, 0)):
        a = g.generate_matrix(g.MatrixSpec(kind, m, n, cond, seed))
        ref = oracle.make_matrix(kind, m, n, cond, seed)
        assert np.max(np.abs(a - ref)) <= 1e-13
        s = g.prescribed_singular_values(kind, min(m, n), cond, seed)
        ref_s = oracle.gen_ref._spectrum(kind, min(m, n), cond, oracle.gen_ref.WordStream(seed))
        np.testing.assert_allclose(s, ref_s, rtol=1e-14)
        np.testing.assert_allclose(np.linalg.svd(a, compute_uv=False), s, rtol=0, atol=1e-13)


def test_accuracy_report_vs_oracle(cuda):
    g = _g()
    a = oracle.make_matrix("random", 70, 50, seed=3)
    r = g.gesdd(a)
    rep = g.accuracy(a, r, reference_sigma=np.linalg.svd(a, compute_uv=False))
    ref = oracle.accuracy_metrics(a, r.sigma, r.u, r.vt, np.linalg.svd(a, compute_uv=False))
    for k in ("e_sigma", "e_svd", "orth_u", "orth_v"):
        assert abs(getattr(rep, k) - ref[k]) <= 1e-15 + 1e-3 * ref[k], k
    r0 = g.gesdd(a, g.SVDOptions(want_vectors=False))
    rep0 = g.accuracy(a, r0)
    assert rep0.e_sigma is None and rep0.e_svd is None and rep0.orth_u is None and rep0.orth_v is None
    with pytest.raises(ValueError):
        g.accuracy(a, r, reference_sigma=np.ones(3))


def test_cli_end_to_end(cuda, tmp_path, capsys):
    g = _g()
    p = str(tmp_path / "a.dsvd")
    assert g.cli_main(["gen", "--kind", "geo", "--m", "60", "--n", "40", "--cond", "1e4", "--seed", "2",
                       "--out", p]) == 0
    a = g.read_matrix(p)
    assert np.max(np.abs(a - oracle.make_matrix("geo", 60, 40, 1e4, 2))) <= 1e-13
    capsys.readouterr()
    assert g.cli_main(["run", "--input", p, "--out-s", str(tmp_path / "s.dsvd"), "--out-u", str(tmp_path / "u.dsvd"),
                       "--out-vt", str(tmp_path / "vt.dsvd")]) == 0
    printed = np.array([float(x) for x in capsys.readouterr().out.split()])
    s = g.read_matrix(str(tmp_path / "s.dsvd"))[:, 0]
    assert_array_equal(printed, s)
    np.testing.assert_allclose(s, g.prescribed_singular_values("geo", 40, 1e4), rtol=0, atol=1e-13)
    u, vt = g.read_matrix(str(tmp_path / "u.dsvd")), g.read_matrix(str(tmp_path / "vt.dsvd"))
    assert np.linalg.norm(a - (u * s) @ vt) <= 1e-13 * np.linalg.norm(a)
    assert g.cli_main(["run", "--input", p, "--jobz", "n", "--out-u", str(tmp_path / "x")]) == 2
    assert g.cli_main(["verify", "--input", p]) == 0
    assert "[ok]" in capsys.readouterr().out
    assert g.cli_main(["verify", "--input", p, "--tol", "1e-30"]) == 1
    csv = tmp_path / "p.csv"
    assert g.cli_main(["profile", "--input", p, "--csv", str(csv)]) == 0
    lines = csv.read_text().splitlines()
    assert lines[0] == "phase,seconds" and [l.split(",")[0] for l in lines[1:]] == list(g.PHASE_NAMES)


# ---------------------------------------------------------------------------
# spectrum sweeps on GPU-generated inputs (harness kinds, acceptance criterion 1 style)

def _check_report(g, a_dev, r, sigma_ref, scale_n):
    rep = g.accuracy(a_dev, r)
    assert rep.e_svd / scale_n <= RES_TOL
    k = r.sigma.numel() if isinstance(r.sigma, torch.Tensor) else r.sigma.size
    assert rep.orth_u / k <= ORTH_TOL and rep.orth_v / k <= ORTH_TOL
    if sigma_ref is not None:
        s = r.sigma.cpu().numpy() if isinstance(r.sigma, torch.Tensor) else r.sigma
        assert np.max(np.abs(s - sigma_ref)) / sigma_ref[0] <= SIG_TOL * scale_n


@pytest.mark.parametrize("kind", ["logrand", "arith", "geo"])
@pytest.mark.parametrize("cond", [1e2, 1e6, 1e10])
@pytest.mark.parametrize("shape", [(700, 700), (1500, 300), (300, 900)])
def test_spectrum_sweep_gpu_generated(cuda, kind, cond, shape):
    g = _g()
    m, n = shape
    spec = g.MatrixSpec(kind, m, n, cond, seed=m + n)
    a = g.generate_matrix(spec, device=True)
    s_ref = g.prescribed_singular_values(kind, min(m, n), cond, seed=m + n)
    r = g.gesdd(a)
    _check_report(g, a, r, s_ref, max(m, n))
    v = g.gesdd(a, g.SVDOptions(want_vectors=False))
    assert torch.equal(v.sigma, r.sigma)


@pytest.mark.slow
def test_c3_scale_tall_skinny(cuda):
    """Config C3 shape at full size: 65536 x 1024 (GEQRF pre-step path), the
    reference's own tall-skinny stress kind (logrand, cond 1e8), sigma against
    the prescribed spectrum, residual / orthogonality on the device."""
    g = _g()
    m, n = 65536, 1024
    a = g.generate_matrix(g.MatrixSpec("logrand", m, n, 1e8, seed=3), device=True)
    s_ref = g.prescribed_singular_values("logrand", n, 1e8, seed=3)
    r = g.gesdd(a)
    _check_report(g, a, r, s_ref, m)
    # the 'random' C3 input itself (bitwise the reference's MatrixSpec('random', 65536, 1024, seed=3)):
    # sigma against the REAL reference's on the same bytes, tolerance 1e-12 n (n = 1024)
    a = g.generate_matrix(g.MatrixSpec("random", m, n, seed=3), device=True)
    r = g.gesdd(a)
    _check_report(g, a, r, None, m)
    s = r.sigma.cpu().numpy()
    ref = _sigma_fixture("c3")["sigma"]
    assert np.max(np.abs(s - ref)) / ref[0] <= SIG_TOL * n


@pytest.mark.parametrize("shape", [(400000, 40), (200000, 96), (48, 300000)])
def test_panels_taller_than_shared_memory(cuda, shape):
    """Tall-skinny inputs whose QR panel slab per CTA exceeds shared memory
    (R1 x 32 doubles > 200 KB): the panel kernel keeps the slab in global
    memory; same accuracy bar as every other shape."""
    g = _g()
    m, n = shape
    spec = g.MatrixSpec("logrand", m, n, 1e6, seed=7)
    a = g.generate_matrix(spec, device=True)
    s_ref = g.prescribed_singular_values("logrand", min(m, n), 1e6, seed=7)
    r = g.gesdd(a)
    _check_report(g, a, r, s_ref, max(m, n))


def test_c5_shaped_batch(cuda):
    """Config C5 shape (2048^2) batch on the concurrent sub-context path."""
    g = _g()
    fx = _sigma_fixture("c5")
    mats = [g.generate_matrix(g.MatrixSpec("random", 2048, 2048, seed=1000 + i), device=True) for i in range(6)]
    res = g.gesdd_batched(mats)
    for i, (a, r) in enumerate(zip(mats, res)):
        _check_report(g, a, r, fx["sigma"][i], 2048)
    # a sub-context runs its panels on sms/concurrency CTAs (different partial-sum
    # grouping than a whole-GPU call): equal to rounding, bitwise reproducible per mode
    one = g.gesdd(mats[3])
    assert (one.sigma - res[3].sigma).abs().max().item() <= 1e-13 * one.sigma[0].item()
    again = g.gesdd_batched(mats)
    assert all(torch.equal(x.sigma, y.sigma) for x, y in zip(res, again))


def test_bdsdc_trivial_sizes(cuda):
    """n = 0 and n = 1 problems return the reference's shapes/values
    (bdc.py:754-765, 861-880)."""
    g = _g()
    r = g.bdsdc(g.BidiagonalProblem(np.zeros(0), np.zeros(0)))
    assert r.dvals.shape == (0,) and r.w.shape == (0, 0) and r.qfull.shape == (0, 0)
    r = g.bdsdc(g.BidiagonalProblem(np.array([2.0]), np.zeros(0)))
    assert_array_equal(r.dvals, [2.0])
    assert_array_equal(r.w, [[1.0]])
    assert_array_equal(r.qfull, [[1.0]])
    assert_array_equal(r.edge_rows, [[1.0], [1.0]])
    r = g.bdsdc(g.BidiagonalProblem(np.array([-2.0]), np.zeros(0)))
    assert_array_equal(r.dvals, [2.0])
    assert_array_equal(r.w, [[-1.0]])
    with pytest.raises(ValueError):
        g.gesdd(np.zeros((0, 5)))


def test_wide_options_and_partial_sequences(cuda):
    """Block/leaf widths above the GPU kernels' limits are accepted like the
    reference (same factorization up to rounding); left reflector sequences
    with count < ncols apply the first `count` reflectors (backtransform.py:60-72)."""
    g = _g()
    a = oracle.make_matrix("random", 150, 120, seed=12)
    s, _, _ = oracle.svd(a, want_vectors=False)
    for opts in (g.SVDOptions(bidiag_block=64, leaf_size=64, qr_block=100, orgqr_block=300, apply_block=256),
                 g.SVDOptions(bidiag_block=200, ts_crossover=1.0)):
        r = g.gesdd(a, opts)
        check_svd(a, r.sigma, r.u, r.vt, s)
    f1 = g.gebrd_blocked(np.asfortranarray(a.copy()), 64)
    f2 = g.gebrd_blocked(np.asfortranarray(a.copy()), 32)
    np.testing.assert_allclose(f1.d, f2.d, rtol=0, atol=1e-12 * np.abs(f2.d).max())
    prob = g.BidiagonalProblem(f2.d, f2.e[:119])
    np.testing.assert_allclose(g.bdsdc(prob, leaf=100).dvals, g.bdsdc(prob).dvals, rtol=0, atol=1e-13 * s[0])
    r = g.bdsqr_base(g.BidiagonalProblem(np.linspace(1, 2, 50), np.full(49, 0.1)))
    assert np.all(np.diff(r.dvals) >= 0)
    # partial left sequence vs the oracle's reflector-by-reflector product
    fact = g.gebrd_blocked(np.asfortranarray(oracle.make_matrix("random", 60, 40, seed=3)), 8)
    seq = g.column_reflectors(fact)
    seq = g.ReflectorSequence(seq.packed, seq.tau, "left", 0, 17)
    c = np.asfortranarray(np.random.default_rng(0).standard_normal((60, 25)))
    ref = c.copy()
    for i in reversed(range(17)):                     # U1 C = H_0 (H_1 (... H_16 C))
        v = np.concatenate(([1.0], fact.packed[i + 1:, i]))
        ref[i:] -= fact.tauq[i] * np.outer(v, v @ ref[i:])
    out = g.ormqr_like(seq, c.copy(order="F"))
    np.testing.assert_allclose(out, ref, rtol=0, atol=1e-13)


@pytest.mark.parametrize("k,tb", [(64, True), (128, False), (37, True)])
def test_rank_k_bulk_matches_cp_async(cuda, k, tb):
    """The streaming kernel's A tiles by TMA bulk copies and by per-thread
    cp.async hold the same bytes, so C is bitwise identical; an A view at an
    odd element offset (not 16-byte aligned) takes the 8-byte cp.async path."""
    g = _g()
    from paper_2508_11467_b200 import _lib
    lib = _lib.load_library()
    torch.manual_seed(3)
    m, n = 3001, 2999
    a = torch.randn(k, m, dtype=torch.float64, device=cuda).t()
    b = (torch.randn(k, n, dtype=torch.float64, device=cuda).t() if tb
         else torch.randn(n, k, dtype=torch.float64, device=cuda).t())
    c0 = torch.randn(n, m, dtype=torch.float64, device=cuda).t()
    out = []
    try:
        for bulk in (1, 0):
            lib.dcsvd_debug_rankk_bulk(bulk)
            c = c0.clone()
            g.matmul_accumulate(-1.0, a, False, b, tb, 1.0, c)
            out.append(c)
    finally:
        lib.dcsvd_debug_rankk_bulk(1)
    assert torch.equal(out[0], out[1])
    ref = c0 - a @ (b.t() if tb else b)
    assert (out[0] - ref).abs().max().item() <= 1e-12 * k
    store = torch.randn(k * (m + 1) + 1, dtype=torch.float64, device=cuda)
    a_odd = store[1:1 + k * (m + 1)].view(k, m + 1).t()[:m]  # base at an odd element, ld = m + 1
    a_odd.copy_(a)
    c = c0.clone()
    g.matmul_accumulate(-1.0, a_odd, False, b, tb, 1.0, c)
    assert (c - ref).abs().max().item() <= 1e-12 * k


# ---- error paths through the device status word (bdc.py:309-312, 636-639, 669-672) ----

@pytest.mark.parametrize("budget", [0, 1])
def test_secular_budget_raises_convergence_error(cuda, budget):
    """A secular root not converged within max_iterations -> the kernel's
    status word -> ConvergenceError, as the reference's _secular_roots
    (bdc.py:589, 636-639) on the same system."""
    g = _g()
    s = g.SecularSystem(np.array([0.0, 1.0, 2.0]), np.array([1.0, 1.0, 1.0]), np.sqrt(3.0))
    with pytest.raises(g.ConvergenceError):
        g.solve_all_roots(s, max_iterations=budget)
    # the handle is usable afterwards (status word reset) and the default budget converges
    r = g.solve_all_roots(s)
    np.testing.assert_allclose(r.omega, [0.59518794, 1.41421356, 2.37607898], rtol=1e-8)
    r2 = g.solve_all_roots(s, max_iterations=100)
    assert np.array_equal(r.omega, r2.omega)


@pytest.mark.parametrize("case", [([1, 1, 2], [1.0, 1.0, 1.64575131]), ([0, 0, 2], [0.35424869, 0.35424869, 1.64575131]),
                                  ([0, 1, 2], [0.35424869, -0.5, 1.64575131])])
def test_loewner_nonpositive_radicand_raises_arithmetic_error(cuda, case):
    """Roots that violate interlacing give a non-positive radicand in the
    Loewner z update -> ArithmeticError (bdc.py:669-672); the same inputs
    raise in the oracle (and in the reference, checked when the cases were
    chosen)."""
    g = _g()
    d = np.array([0.0, 1.0, 2.0])
    z = np.array([1.0, 1.0, 1.0])
    anc, mu = np.array(case[0], dtype=np.intp), np.array(case[1])
    s = g.SecularSystem(d, z, np.sqrt(3.0))
    bad = g.SecularRoots(np.sqrt(d[anc] ** 2 + mu), anc, mu)
    with pytest.raises(ArithmeticError):
        oracle.loewner_z(d, z, anc, mu)
    with pytest.raises(ArithmeticError):
        g.recompute_z(s, bad)
    good = g.solve_all_roots(s)
    zt = g.recompute_z(s, good)
    np.testing.assert_allclose(zt, oracle.loewner_z(d, z, good.anchor, good.mu), rtol=1e-13)


def test_secular_vectors_match_oracle(cuda):
    """secular_vectors (bdc.py:676-694) against oracle.secular_vecs on a
    random system (round 1 checked only orthonormality)."""
    g = _g()
    rng = np.random.default_rng(77)
    n = 40
    d = np.concatenate([[0.0], np.sort(rng.uniform(0.1, 3.0, n - 1))])
    z = rng.standard_normal(n)
    s = g.SecularSystem(d, z, float(np.linalg.norm(z)))
    roots = g.solve_all_roots(s)
    zt = g.recompute_z(s, roots)
    u, v = g.secular_vectors(s, roots, zt)
    ou, ov = oracle.secular_vecs(d, roots.anchor, roots.mu, oracle.loewner_z(d, z, roots.anchor, roots.mu))
    np.testing.assert_allclose(np.asarray(u), ou, rtol=0, atol=1e-12)
    np.testing.assert_allclose(np.asarray(v), ov, rtol=0, atol=1e-12)


@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("tb", [False, True])
@pytest.mark.parametrize("shape", [(1000, 2000, 300), (1537, 1029, 97), (128, 9000, 4000), (8, 9600, 300), (9600, 8, 300), (300, 9600, 3)])
def test_tma_gemm_matches_torch(cuda, ta, tb, shape):
    """General GEMMs large enough for the warp-specialized TMA kernel
    (dgemm_ws_kernel: >= 148 output tiles, 16-byte-aligned operands), every
    transpose combination, K not a multiple of the 32-wide stage (TMA zero
    fill), beta != 0; against torch fp64, and against the cp.async kernel."""
    g = _g()
    lib = _lib_handle()
    m, n, k = shape
    torch.manual_seed(m + n + k)
    a = torch.randn(k, m, dtype=torch.float64, device=cuda).t() if not ta else torch.randn(m, k, dtype=torch.float64, device=cuda).t()
    b = torch.randn(n, k, dtype=torch.float64, device=cuda).t() if not tb else torch.randn(k, n, dtype=torch.float64, device=cuda).t()
    c0 = torch.randn(n, m, dtype=torch.float64, device=cuda).t()
    ref = 0.5 * c0 + 1.25 * ((a.t() if ta else a) @ (b.t() if tb else b))
    outs = []
    for ws in (1, 0):
        lib.dcsvd_debug_dgemm_ws(ws)
        try:
            c = c0.clone()
            g.matmul_accumulate(1.25, a, ta, b, tb, 0.5, c)
        finally:
            lib.dcsvd_debug_dgemm_ws(1)
        assert (c - ref).abs().max().item() <= 1e-12 * k * ref.abs().max().item()
        outs.append(c)
    assert (outs[0] - outs[1]).abs().max().item() <= 1e-13 * k * ref.abs().max().item()


@pytest.mark.parametrize("n", [1000, 2048])
def test_bdc_merge_products_tma_vs_cpasync(cuda, n):
    """BDC merge products on the TMA gather GEMM (workspace stack, gather4
    A columns, odd row offsets loaded one row early) are bitwise equal to the
    cp.async gather kernel's (same k order per output)."""
    g = _g()
    lib = _lib_handle()
    a = g.generate_matrix(g.MatrixSpec("random", n, n, seed=9), device=True)
    f = g.gebrd_blocked(a)
    prob = g.BidiagonalProblem(f.d, f.e)
    r1 = g.bdsdc(prob)
    lib.dcsvd_debug_dgemm_ws(0)
    try:
        r0 = g.bdsdc(prob)
    finally:
        lib.dcsvd_debug_dgemm_ws(1)
    assert torch.equal(r0.dvals, r1.dvals)
    assert torch.equal(r0.w, r1.w) and torch.equal(r0.qfull, r1.qfull)


@pytest.mark.parametrize("shape", [(700, 700), (1536, 1024), (4000, 600)])
def test_gesdd_c_abi_odd_leading_dimensions(cuda, shape):
    """dcsvd_gesdd through the C ABI with caller buffers whose leading
    dimensions are odd (ld = rows + 1): the TMA kernels cannot map such
    operands and must fall back (rank-k updates on U / V^T, TS recombination)
    with the same accuracy."""
    import ctypes
    from paper_2508_11467_b200 import _lib
    g = _g()
    m, n = shape
    k = min(m, n)
    a = g.generate_matrix(g.MatrixSpec("random", m, n, seed=m + n), device=True)
    lda, ldu, ldvt = m + 1, m + 1, k + 1
    A = torch.zeros(n, lda, dtype=torch.float64, device=cuda)
    A[:, :m] = a.t()
    U = torch.zeros(k, ldu, dtype=torch.float64, device=cuda)
    VT = torch.zeros(n, ldvt, dtype=torch.float64, device=cuda)
    S = torch.zeros(k, dtype=torch.float64, device=cuda)
    lib = _lib.load_library()
    h = _lib.handle()
    rc = lib.dcsvd_gesdd(h, m, n, _lib.ptr(A), lda, _lib.ptr(S), _lib.ptr(U), ldu, _lib.ptr(VT), ldvt, None, None,
                         _lib.stream_ptr())
    _lib.check(rc, h)
    u = U[:, :m].t()
    vt = VT[:, :k].t()
    ref = g.gesdd(a)
    assert (S - ref.sigma).abs().max().item() <= SIG_TOL * max(m, n) * ref.sigma[0].item()
    eye = torch.eye(k, dtype=torch.float64, device=cuda)
    assert torch.linalg.matrix_norm(a - (u * S) @ vt).item() / torch.linalg.matrix_norm(a).item() / max(m, n) <= RES_TOL
    assert torch.linalg.matrix_norm(u.t() @ u - eye).item() / k <= ORTH_TOL
    assert torch.linalg.matrix_norm(vt @ vt.t() - eye).item() / k <= ORTH_TOL


@pytest.mark.parametrize("shape", [(300000, 1, 64, False), (256, 1100, 128, True), (262144, 2, 5, False), (1000, 300, 128, True)])
def test_rank_k_degenerate_shapes(cuda, shape):
    """Rank-k updates at the edges of the TMA tile kernel's routing (one or two
    output columns, the minimum 256 rows, K = 5): zero-filled boxes past the
    tensor, short tiles; against torch fp64."""
    g = _g()
    m, n, k, tb = shape
    torch.manual_seed(m + n + k)
    a = torch.randn(k, m, dtype=torch.float64, device=cuda).t()
    b = torch.randn(k, n, dtype=torch.float64, device=cuda).t() if tb else torch.randn(n, k, dtype=torch.float64, device=cuda).t()
    c = torch.randn(n, m, dtype=torch.float64, device=cuda).t()
    ref = c - a @ (b.t() if tb else b)
    g.matmul_accumulate(-1.0, a, False, b, tb, 1.0, c)
    assert (c - ref).abs().max().item() <= 1e-12 * max(k, 1) * max(1.0, ref.abs().max().item())
