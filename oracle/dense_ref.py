"""Dense stages of the oracle: reflector/rotation generation, one-stage
bidiagonalization, blocked Householder QR, compact-WY block reflectors and the
back-transformations.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

All matrices are float64 column-major numpy arrays; functions that the
reference runs in place run in place here too.
"""

import numpy as np

_F = "F"


def larfg(alpha, x):
    """Householder generation, no safmin rescaling.

    Follows pkg/src/dcsvd/densecore.py:114-128: tail norm 0 -> (tau 0, beta
    alpha, essential unchanged); else beta = -copysign(hypot(alpha, |x|),
    alpha), tau = (beta-alpha)/beta, essential = x/(alpha-beta).
    Returns (tau, beta, essential).
    """
    x = np.asarray(x, dtype=np.float64)
    xnorm = np.linalg.norm(x)
    if xnorm == 0.0:
        return 0.0, float(alpha), x.copy()
    beta = -np.copysign(np.hypot(alpha, xnorm), alpha)
    return float((beta - alpha) / beta), float(beta), x / (alpha - beta)


def lartg(f, g):
    """Plane rotation (c, s, r), r = hypot(f, g) >= 0; (0, 0) -> identity.

    Follows pkg/src/dcsvd/densecore.py:131-140.
    """
    r = np.hypot(f, g)
    if r == 0.0:
        return 1.0, 0.0, 0.0
    return f / r, g / r, float(r)


# ---------------------------------------------------------------------------
# bidiagonalization (pkg/src/dcsvd/bidiag.py)


def gebd2(a):
    """Unblocked rank-2-per-step reduction in place (bidiag.py:75-110).

    Returns (d, e, tauq, taup) with e of length n-1 and taup[n-1] = 0.
    """
    m, n = a.shape
    d = np.zeros(n)
    e = np.zeros(max(n - 1, 0))
    tq = np.zeros(n)
    tp = np.zeros(n)
    for k in range(n):
        tau, beta, ess = larfg(a[k, k], a[k + 1:, k])
        tq[k], d[k] = tau, beta
        a[k, k] = beta
        a[k + 1:, k] = ess
        if tau != 0.0 and k + 1 < n:
            v = np.concatenate(([1.0], ess))
            blk = a[k:, k + 1:]
            blk -= tau * np.outer(v, v @ blk)
        if k + 1 < n:
            tau, beta, ess = larfg(a[k, k + 1], a[k, k + 2:])
            tp[k], e[k] = tau, beta
            a[k, k + 1] = beta
            a[k, k + 2:] = ess
            if tau != 0.0:
                u = np.concatenate(([1.0], ess))
                blk = a[k + 1:, k + 1:]
                blk -= tau * np.outer(blk @ u, u)
    return d, e, tq, tp


def labrd(a, nb, d, e, tq, tp):
    """Merged rank-(2 nb) panel of the view ``a`` (bidiag.py:113-165).

    P = [v_0, x_0, v_1, x_1, ...] (m' x 2nb), Q = [y_0, u_0, ...] (n' x 2nb),
    full height with zeros above the pivots; tau/pi folded into y/x.  Only
    panel rows/columns of ``a`` change; returns (P, Q).
    """
    m, n = a.shape
    if not 1 <= nb < n <= m:
        raise ValueError(f"panel {nb} needs nb < ncols <= nrows, got {m}x{n}")
    P = np.zeros((m, 2 * nb), order=_F)
    Q = np.zeros((n, 2 * nb), order=_F)
    for k in range(nb):
        c0, c1 = 2 * k, 2 * k + 1
        if k:
            a[k:, k] -= P[k:, :c0] @ Q[k, :c0]
        tau, beta, ess = larfg(a[k, k], a[k + 1:, k])
        tq[k], d[k] = tau, beta
        a[k, k] = beta
        a[k + 1:, k] = ess
        P[k, c0] = 1.0
        P[k + 1:, c0] = ess
        if tau != 0.0:
            v = P[k:, c0]
            y = a[k:, k + 1:].T @ v
            if k:
                y -= Q[k + 1:, :c0] @ (P[k:, :c0].T @ v)
            Q[k + 1:, c0] = tau * y
        a[k, k + 1:] -= Q[k + 1:, :c1] @ P[k, :c1]
        tau, beta, ess = larfg(a[k, k + 1], a[k, k + 2:])
        tp[k], e[k] = tau, beta
        a[k, k + 1] = beta
        a[k, k + 2:] = ess
        Q[k + 1, c1] = 1.0
        Q[k + 2:, c1] = ess
        if tau != 0.0:
            u = Q[k + 1:, c1]
            x = a[k + 1:, k + 1:] @ u
            x -= P[k + 1:, :c1] @ (Q[k + 1:, :c1].T @ u)
            P[k + 1:, c1] = tau * x
    return P, Q


def gebrd(a, nb=32):
    """Blocked one-stage bidiagonalization in place (bidiag.py:168-204).

    Panels of ``nb`` columns while more than ``nb`` columns remain, each
    followed by the single trailing update A -= P Q^T; the remainder goes
    through :func:`gebd2`.  Returns (d, e, tauq, taup).
    """
    m, n = a.shape
    if n < 1 or m < n:
        raise ValueError(f"gebrd needs m >= n >= 1, got {m}x{n}")
    if nb < 1:
        raise ValueError("block must be >= 1")
    d = np.zeros(n)
    e = np.zeros(max(n - 1, 0))
    tq = np.zeros(n)
    tp = np.zeros(n)
    j = 0
    while n - j > nb:
        sl = slice(j, j + nb)
        P, Q = labrd(a[j:, j:], nb, d[sl], e[sl], tq[sl], tp[sl])
        a[j + nb:, j + nb:] -= P[nb:, :] @ Q[nb:, :].T
        j += nb
    td, te, tt, ts = gebd2(a[j:, j:])
    d[j:], e[j:], tq[j:], tp[j:] = td, te, tt, ts
    return d, e, tq, tp


# ---------------------------------------------------------------------------
# compact WY with inverse triangular factor (pkg/src/dcsvd/qrblock.py)


def cwy_y(packed_cols, taus):
    """Unit-lower-trapezoidal Y from packed essentials (qrblock.py:74-87);
    columns with tau == 0 are all-zero."""
    rows, w = packed_cols.shape
    y = np.zeros((rows, w), order=_F)
    for j in range(w):
        if taus[j] != 0.0:
            y[j, j] = 1.0
            y[j + 1:, j] = packed_cols[j + 1:, j]
    return y


def cwy_tinv(y, taus):
    """Tinv = strict-upper(Y^T Y) + diag(1/tau) (1 where tau == 0)
    (qrblock.py:90-100)."""
    t = np.triu(y.T @ y, 1)
    w = y.shape[1]
    for j in range(w):
        t[j, j] = 1.0 / taus[j] if taus[j] != 0.0 else 1.0
    return np.asfortranarray(t)


def _tri_solve_upper(t, b, trans):
    import scipy.linalg as sl

    return sl.solve_triangular(t, b, lower=False, trans=1 if trans else 0)


def cwy_apply_left(y, tinv, c, trans=False):
    """C <- (I - Y T Y^T) C, T = Tinv^-1 (or the transposed block)
    (qrblock.py:103-111)."""
    if np.any(np.diag(tinv) == 0.0):
        raise np.linalg.LinAlgError("zero diagonal in Tinv")
    z = _tri_solve_upper(tinv, y.T @ c, trans)
    c -= y @ z
    return c


def cwy_apply_right(y, tinv, c, trans=False):
    """C <- C (I - Y T Y^T) (or transposed block) (qrblock.py:114-119):
    Z = C Y, X = Z T (or Z T^T), C -= X Y^T."""
    if np.any(np.diag(tinv) == 0.0):
        raise np.linalg.LinAlgError("zero diagonal in Tinv")
    z = c @ y
    # Z Tinv^-1 = (Tinv^-T Z^T)^T ; Z Tinv^-T = (Tinv^-1 Z^T)^T
    x = _tri_solve_upper(tinv, z.T, not trans).T
    c -= x @ y.T
    return c


def geqr2(a, tau):
    """Unblocked Householder QR of a panel in place (qrblock.py:51-71)."""
    m, n = a.shape
    for j in range(n):
        t, beta, ess = larfg(a[j, j], a[j + 1:, j])
        tau[j] = t
        a[j, j] = beta
        a[j + 1:, j] = ess
        if t != 0.0 and j + 1 < n:
            v = np.concatenate(([1.0], ess))
            blk = a[j:, j + 1:]
            blk -= t * np.outer(v, v @ blk)
    return a


def geqrf(a, nb=32):
    """Blocked QR in place (qrblock.py:122-144): panel by :func:`geqr2`, the
    trailing columns take the transposed block reflector.  Returns tau."""
    m, n = a.shape
    if n < 1 or m < n:
        raise ValueError(f"geqrf needs m >= n >= 1, got {m}x{n}")
    tau = np.zeros(n)
    for j in range(0, n, nb):
        w = min(nb, n - j)
        geqr2(a[j:, j:j + w], tau[j:j + w])
        if j + w < n:
            y = cwy_y(a[j:, j:j + w], tau[j:j + w])
            cwy_apply_left(y, cwy_tinv(y, tau[j:j + w]), a[j:, j + w:], trans=True)
    return tau


def orgqr(packed, tau, k, nb=64):
    """First k columns of Q = H_1...H_n, blocks back to front onto an identity
    slab (qrblock.py:147-164)."""
    m, n = packed.shape
    q = np.zeros((m, k), order=_F)
    q[np.arange(min(m, k)), np.arange(min(m, k))] = 1.0
    for j in reversed(range(0, n, nb)):
        w = min(nb, n - j)
        y = cwy_y(packed[j:, j:j + w], tau[j:j + w])
        cwy_apply_left(y, cwy_tinv(y, tau[j:j + w]), q[j:, :], trans=False)
    return q


# ---------------------------------------------------------------------------
# back-transformation (pkg/src/dcsvd/backtransform.py)


def apply_u1(packed, tauq, c, nb=64, trans=False):
    """C <- U1 C (back to front) or U1^T C (front to back, transposed blocks)
    with U1 = H_0...H_{n-1} the column reflectors (backtransform.py:90-109)."""
    m, n = packed.shape
    starts = list(range(0, n, nb))
    for j in (starts if trans else reversed(starts)):
        w = min(nb, n - j)
        y = np.zeros((m - j, w), order=_F)
        for t in range(w):
            if tauq[j + t] != 0.0:
                y[t, t] = 1.0
                y[t + 1:, t] = packed[j + t + 1:, j + t]
        cwy_apply_left(y, cwy_tinv(y, tauq[j:j + w]), c[j:, :], trans=trans)
    return c


def apply_v1t(packed, taup, c, nb=64, trans=True):
    """C <- C V1^T (trans, blocks back to front) or C V1 (front to back) with
    the row reflectors G_0...G_{n-2} acting on columns >= off+1
    (backtransform.py:112-131, row blocks :75-87)."""
    n = packed.shape[1]
    count = max(n - 1, 0)
    starts = list(range(0, count, nb))
    for j in (reversed(starts) if trans else starts):
        w = min(nb, count - j)
        y = np.zeros((n - j - 1, w), order=_F)
        for t in range(w):
            i = j + t
            if taup[i] != 0.0:
                y[t, t] = 1.0
                y[t + 1:, t] = packed[i, i + 2:]
        cwy_apply_right(y, cwy_tinv(y, taup[j:j + w]), c[:, j + 1:], trans=trans)
    return c
