"""Build the C4 heavy-deflation bidiagonal fixture.

Recipe (independent of the engine under test): normals from the harness
Philox stream (seed 4) filled column-major; U = Q of LAPACK QR with columns
sign-fixed by diag(R); V likewise from the continuing stream; A = (U*sigma)V^T
with sigma = 1 + j/8 (j = 0..7, multiplicity n/8 each); then LAPACK dgebrd
(ctypes, LAPACKE from scipy's bundled OpenBLAS).  Stores (d, e) as a .npz and
prints its SHA-256.  Optionally runs the reference bdsdc on it (values-only)
to store the golden sigma.  Runs on CPU in the build container; the output
file is committed, so the GPU box never rebuilds it.

usage: python tools/make_c4_fixture.py N OUT.npz [--ref]
"""
import ctypes, glob, hashlib, os, sys, time
import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from oracle.gen_ref import WordStream  # noqa: E402


def lapack_dgebrd(a):
    import scipy
    libs = glob.glob(os.path.join(os.path.dirname(scipy.__file__), "..", "scipy.libs", "libscipy_openblas*.so"))
    lib = ctypes.CDLL(libs[0])
    f = lib.scipy_LAPACKE_dgebrd
    m, n = a.shape
    k = min(m, n)
    d = np.zeros(k); e = np.zeros(max(k - 1, 1)); tq = np.zeros(k); tp = np.zeros(k)
    P = ctypes.POINTER(ctypes.c_double)
    f.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, P, ctypes.c_int, P, P, P, P]
    f.restype = ctypes.c_int
    a = np.asfortranarray(a)
    info = f(102, m, n, a.ctypes.data_as(P), m, d.ctypes.data_as(P), e.ctypes.data_as(P),
             tq.ctypes.data_as(P), tp.ctypes.data_as(P))
    assert info == 0, info
    return d, e[: k - 1]


def haar(ws, n):
    g = np.asfortranarray(ws.normals(n * n).reshape((n, n), order="F"))
    q, r = np.linalg.qr(g)
    sgn = np.sign(np.diag(r)); sgn[sgn == 0] = 1.0
    return np.asfortranarray(q * sgn)


def main():
    n = int(sys.argv[1]); out = sys.argv[2]
    t0 = time.time()
    ws = WordStream(4)
    sigma = 1.0 + np.repeat(np.arange(8), n // 8) / 8.0
    u = haar(ws, n)
    v = haar(ws, n)
    a = np.asfortranarray((u * sigma) @ v.T)
    del u, v
    t1 = time.time()
    d, e = lapack_dgebrd(a)
    t2 = time.time()
    extra = {}
    if "--ref" in sys.argv:
        sys.path.insert(0, "/root/reference/pkg/src")
        import dcsvd
        t3 = time.time()
        res = dcsvd.bdsdc(dcsvd.BidiagonalProblem(d, e), want_vectors=False)
        extra["sigma_ref"] = res.dvals
        extra["ref_seconds_values_only"] = np.array(time.time() - t3)
    np.savez(out, d=d, e=e, sigma_prescribed=np.sort(sigma)[::-1], **extra)
    h = hashlib.sha256(np.concatenate([d, e]).tobytes()).hexdigest()
    print(f"n={n} build A {t1-t0:.1f}s dgebrd {t2-t1:.1f}s sha256(d|e)={h}", flush=True)


if __name__ == "__main__":
    main()
