"""Quick stage-by-stage GPU check against the oracle (dev tool)."""
import sys, time, traceback, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_11467_b200 as g
import oracle

rng = np.random.default_rng(0)
def stage(name, fn):
    t0 = time.time()
    try:
        fn(); print(f"[ok] {name} {time.time()-t0:.2f}s", flush=True)
    except Exception:
        print(f"[FAIL] {name}", flush=True); traceback.print_exc()

def t_gemm():
    for (m, n, k, ta, tb) in [(100, 70, 50, False, False), (130, 257, 64, False, True), (64, 300, 1000, True, False), (33, 17, 9, True, True)]:
        a = rng.standard_normal((k, m) if ta else (m, k)); b = rng.standard_normal((n, k) if tb else (k, n)); c = rng.standard_normal((m, n))
        ref = 0.5 * c + 2.0 * ((a.T if ta else a) @ (b.T if tb else b))
        g.matmul_accumulate(2.0, a, ta, b, tb, 0.5, c)
        print("  gemm", m, n, k, ta, tb, np.max(np.abs(c - ref)))
def t_gebrd():
    for (m, n, nb) in [(70, 70, 32), (90, 50, 8), (300, 300, 32), (129, 100, 16), (40, 40, 64)]:
        a = rng.standard_normal((m, n)); a1 = np.asfortranarray(a.copy()); a2 = np.asfortranarray(a.copy())
        f = g.gebrd_blocked(a1, nb); d, e, tq, tp = oracle.gebrd(a2, min(nb, max(n,1)) if nb < n else nb)
        print("  gebrd", m, n, nb, np.max(np.abs(f.d - d)), np.max(np.abs(f.e - e)), np.max(np.abs(f.tauq - tq)), np.max(np.abs(f.taup - tp)), np.max(np.abs(a1 - a2)))
def t_bdc():
    for n, leaf, bord in [(5, 32, False), (40, 4, False), (40, 4, True), (90, 32, False), (70, 1, True), (200, 32, False), (1, 32, False), (0, 32, True)]:
        d = rng.standard_normal(n); e = rng.standard_normal(n)
        ee = e if bord else e[:max(n-1,0)]
        R = g.bdsdc(g.BidiagonalProblem(d, ee, bord), leaf=leaf)
        O = oracle.bdc(oracle.Bidiag(d, ee, bord), leaf=leaf)
        errs = [np.max(np.abs(R.dvals - O.vals)) if n else 0.0]
        if n:
            B = g.BidiagonalProblem(d, ee, bord).dense()
            rec = (R.w * R.dvals) @ R.qfull[:, :n].T
            errs += [np.linalg.norm(B - rec), np.linalg.norm(R.w.T @ R.w - np.eye(n)), np.linalg.norm(R.qfull.T @ R.qfull - np.eye(n + bord)), np.max(np.abs(R.edge_rows - O.edge))]
        V = g.bdsdc(g.BidiagonalProblem(d, ee, bord), want_vectors=False, leaf=leaf)
        errs.append(bool(np.array_equal(V.dvals, R.dvals)))
        print("  bdc", n, leaf, bord, errs)
def t_qr():
    for (m, n, b, ob) in [(200, 40, 32, 64), (65, 65, 7, 16), (300, 96, 32, 64)]:
        a = rng.standard_normal((m, n)); a1 = np.asfortranarray(a.copy()); a2 = np.asfortranarray(a.copy())
        f = g.geqrf_blocked(a1, b); tau = oracle.geqrf(a2, b)
        q = g.orgqr(f, n, ob); q2 = oracle.orgqr(a2, tau, n, ob)
        print("  qr", m, n, np.max(np.abs(a1 - a2)), np.max(np.abs(f.tau - tau)), np.max(np.abs(q - q2)))
def t_ormbr():
    for (m, n) in [(70, 70), (100, 60)]:
        a = np.asfortranarray(rng.standard_normal((m, n)))
        a2 = a.copy(order="F"); d, e, tq, tp = oracle.gebrd(a2, 32)
        f = g.BidiagonalFactorization(a2, d, e, tq, tp)
        c = np.asfortranarray(rng.standard_normal((m, n))); c2 = c.copy(order="F")
        g.ormqr_like(g.column_reflectors(f), c, transpose=False); oracle.apply_u1(a2, tq, c2, 64, trans=False)
        v = np.asfortranarray(rng.standard_normal((n, n))); v2 = v.copy(order="F")
        g.ormlq_like(g.row_reflectors(f), v, transpose=True); oracle.apply_v1t(a2, tp, v2, 64, trans=True)
        print("  ormbr", m, n, np.max(np.abs(c - c2)), np.max(np.abs(v - v2)))
def t_gesdd():
    for (m, n) in [(64, 64), (100, 37), (37, 100), (130, 130), (200, 40), (300, 300), (1024, 1024)]:
        a = oracle.make_matrix("random", m, n, seed=5)
        r = g.gesdd(a); s, u, vt = oracle.svd(a) if m * n < 200000 else (np.linalg.svd(a, compute_uv=False), None, None)
        k = min(m, n)
        res = np.linalg.norm(a - (r.u * r.sigma) @ r.vt) / np.linalg.norm(a) / max(m, n)
        ou = np.linalg.norm(r.u.T @ r.u - np.eye(k)) / k; ov = np.linalg.norm(r.vt @ r.vt.T - np.eye(k)) / k
        print("  gesdd", m, n, np.max(np.abs(r.sigma - s)) / s[0], res, ou, ov)
    a = oracle.make_matrix("random", 2048, 2048, seed=7)
    torch.cuda.synchronize(); t0 = time.time(); p = g.phase_profile(a); print("  profile 2048", p, time.time() - t0)
for name, fn in [("gemm", t_gemm), ("gebrd", t_gebrd), ("bdc", t_bdc), ("qr", t_qr), ("ormbr", t_ormbr), ("gesdd", t_gesdd)]:
    if len(sys.argv) > 1 and name not in sys.argv[1:]: continue
    stage(name, fn)
