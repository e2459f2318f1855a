"""Generate golden vectors by running the REAL reference (/root/reference,
dcsvd 0.1.0, pure Python) in the build container.

The GPU box has no /root/reference, so the outputs are committed as
``tests/golden/golden.npz`` (+ ``c1_sigma.npz``) and the tests read only
those files.  Re-run with:

    PYTHONDONTWRITEBYTECODE=1 OPENBLAS_NUM_THREADS=1 \
        python tests/golden/make_golden.py
"""

import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import dcsvd  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    g = {}
    # -- gesdd over shapes x kinds (driver.py:147); inputs regenerated from the
    #    Philox MatrixSpec so only the spec is needed to rebuild them.
    specs = [
        ("random", 1, 1, 1.0, 11), ("random", 5, 3, 1.0, 12), ("random", 3, 5, 1.0, 13),
        ("random", 64, 64, 1.0, 14), ("random", 100, 37, 1.0, 15), ("random", 37, 100, 1.0, 16),
        ("random", 130, 130, 1.0, 17), ("random", 200, 40, 1.0, 18), ("random", 96, 64, 1.0, 19),
        ("logrand", 80, 80, 1e6, 20), ("geo", 72, 72, 1e10, 21), ("arith", 90, 60, 1e2, 22),
        ("logrand", 160, 48, 1e8, 23), ("random", 257, 257, 1.0, 24),
    ]
    for idx, (kind, m, n, cond, seed) in enumerate(specs):
        a = dcsvd.generate_matrix(dcsvd.MatrixSpec(kind, m, n, cond, seed))
        r = dcsvd.gesdd(a)
        g[f"svd{idx}_spec"] = np.array([m, n, cond, seed], dtype=np.float64)
        g[f"svd{idx}_kind"] = np.array(kind)
        g[f"svd{idx}_a"] = a
        g[f"svd{idx}_sigma"] = r.sigma
        g[f"svd{idx}_u"] = r.u
        g[f"svd{idx}_vt"] = r.vt
        vo = dcsvd.gesdd(a, dcsvd.SVDOptions(want_vectors=False))
        g[f"svd{idx}_sigma_values_only"] = vo.sigma
    g["svd_count"] = np.array(len(specs))

    # -- gebrd_blocked (bidiag.py:168) for several shapes / block widths
    rng = np.random.default_rng(100)
    cases = [(70, 70, 32), (90, 50, 8), (64, 64, 3), (33, 33, 32), (129, 100, 16)]
    for idx, (m, n, b) in enumerate(cases):
        a = np.asfortranarray(rng.standard_normal((m, n)))
        g[f"gebrd{idx}_a"] = a.copy(order="F")
        f = dcsvd.gebrd_blocked(a, b)
        g[f"gebrd{idx}_block"] = np.array(b)
        for k in ("packed", "d", "e", "tauq", "taup"):
            g[f"gebrd{idx}_{k}"] = getattr(f, k)
    g["gebrd_count"] = np.array(len(cases))

    # -- geqrf_blocked / orgqr (qrblock.py:122,147)
    cases = [(200, 40, 32, 64), (65, 65, 7, 16), (300, 96, 32, 64)]
    for idx, (m, n, b, ob) in enumerate(cases):
        a = np.asfortranarray(rng.standard_normal((m, n)))
        g[f"qr{idx}_a"] = a.copy(order="F")
        f = dcsvd.geqrf_blocked(a, b)
        g[f"qr{idx}_packed"] = f.packed
        g[f"qr{idx}_tau"] = f.tau
        g[f"qr{idx}_q"] = dcsvd.orgqr(f, n, ob)
        g[f"qr{idx}_blocks"] = np.array([b, ob])
    g["qr_count"] = np.array(len(cases))

    # -- bdsdc (bdc.py:861) incl. bordered, small leaves and deflation stress
    bcases = []
    for n, leaf, bord in ((40, 4, False), (40, 4, True), (90, 32, False), (70, 1, True),
                          (33, 2, False), (200, 32, False), (129, 8, True)):
        d = rng.standard_normal(n)
        e = rng.standard_normal(n if bord else n - 1)
        bcases.append((d, e, bord, leaf))
    bcases.append((np.ones(48), np.zeros(47), False, 4))                       # identity: full deflation
    dg = np.float_power(10.0, -np.arange(30, dtype=float))
    bcases.append((dg, 0.5 * dg[:-1], False, 4))                              # graded
    bcases.append((np.repeat([1.0, 2.0, 3.0], 30), np.full(89, 1e-9), False, 8))  # clustered, tiny e
    c4 = np.load(os.path.join(HERE, "c4_n1024.npz"))
    bcases.append((c4["d"][:256], c4["e"][:255], False, 32))
    for idx, (d, e, bord, leaf) in enumerate(bcases):
        prob = dcsvd.BidiagonalProblem(d, e, bordered=bord)
        r = dcsvd.bdsdc(prob, leaf=leaf)
        g[f"bdc{idx}_d"] = d
        g[f"bdc{idx}_e"] = e
        g[f"bdc{idx}_meta"] = np.array([int(bord), leaf])
        g[f"bdc{idx}_vals"] = r.dvals
        g[f"bdc{idx}_w"] = r.w
        g[f"bdc{idx}_q"] = r.qfull
        g[f"bdc{idx}_edge"] = r.edge_rows
    g["bdc_count"] = np.array(len(bcases))

    # -- secular / deflation KATs (test_bdc.py:208-303)
    sysd = dcsvd.SecularSystem(np.array([0.0, 1.0]), np.array([1.0, 1.0]), np.sqrt(3.0))
    roots = dcsvd.solve_all_roots(sysd)
    g["kat_secular_omega"] = roots.omega
    g["kat_secular_mu"] = roots.mu
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **g)

    # -- C1: 1024^2 random seed=1 (BASELINE config 1) sigma from the reference
    a = dcsvd.generate_matrix(dcsvd.MatrixSpec("random", 1024, 1024, seed=1))
    t0 = time.perf_counter()
    r = dcsvd.gesdd(a)
    t = time.perf_counter() - t0
    acc = dcsvd.accuracy(a, r)
    np.savez_compressed(os.path.join(HERE, "c1_sigma.npz"), sigma=r.sigma, seconds=np.array(t),
                        e_svd=np.array(acc.e_svd), orth_u=np.array(acc.orth_u), orth_v=np.array(acc.orth_v))
    print(f"C1 reference gesdd {t:.2f}s e_svd={acc.e_svd:.3e} orth_u={acc.orth_u:.3e}")


if __name__ == "__main__":
    main()
