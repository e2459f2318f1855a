"""Bidiagonal divide and conquer, oracle restatement of
pkg/src/dcsvd/bdc.py.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Conventions kept from the reference (they decide branches, so they matter):
values ascending inside the tree and descending only at the top
(bdc.py:861-880); edge rows (first/last row of the right basis) propagated in
both modes so values-only runs are bitwise equal (bdc.py:14-21); LAPACK
dlasd2-style column classes (bdc.py:173-177).
"""

from dataclasses import dataclass

import numpy as np

from .dense_ref import lartg

EPS = np.finfo(np.float64).eps
TINY = np.finfo(np.float64).tiny

UNIT, FIRST, SECOND, MIXED = 0, 1, 2, 3


class SolverBudgetError(RuntimeError):
    """Iteration budget exceeded (maps to dcsvd.ConvergenceError)."""


@dataclass
class Bidiag:
    """Upper bidiagonal d (n), e (n; e[n-1] used only when bordered).
    (bdc.py:56-96)"""

    d: np.ndarray
    e: np.ndarray
    bordered: bool = False

    def __post_init__(self):
        self.d = np.atleast_1d(np.asarray(self.d, dtype=np.float64)).copy()
        e = np.atleast_1d(np.asarray(self.e, dtype=np.float64)).copy()
        if self.d.size and e.size == self.d.size - 1:
            e = np.append(e, 0.0)
        if e.size != self.d.size:
            raise ValueError("superdiagonal length mismatch")
        self.e = e

    @property
    def n(self):
        return self.d.size

    @property
    def ncols(self):
        return self.n + int(self.bordered)

    def dense(self):
        b = np.zeros((self.n, self.ncols))
        for i in range(self.n):
            b[i, i] = self.d[i]
            if i + 1 < self.ncols:
                b[i, i + 1] = self.e[i]
        return b


@dataclass
class NodeSVD:
    """B = W diag(vals) Q[:, :n]^T; ``edge`` = rows 0 and ncols-1 of Q
    (bdc.py:99-117)."""

    vals: np.ndarray
    W: np.ndarray | None
    Q: np.ndarray | None
    edge: np.ndarray


def _rot_cols(mats, p, q, c, s):
    # [[c, s], [-s, c]] on columns (p, q)  (bdc.py:180-187)
    for m in mats:
        if m is None:
            continue
        cp = m[:, p].copy()
        cq = m[:, q].copy()
        m[:, p] = c * cp + s * cq
        m[:, q] = c * cq - s * cp


# ---------------------------------------------------------------------------
# leaf: implicit-shift QR iteration (bdc.py:201-359)


def _small(x, a, b, bnorm):
    return abs(x) <= EPS * (abs(a) + abs(b)) or abs(x) <= EPS * bnorm * 1e-3


def _shift(d, e, lo, hi):
    # Wilkinson shift of the trailing 2x2 of B^T B (bdc.py:205-215)
    ep = e[hi - 2] if hi - 2 >= lo else 0.0
    a11 = d[hi - 1] * d[hi - 1] + ep * ep
    a12 = d[hi - 1] * e[hi - 1]
    a22 = d[hi] * d[hi] + e[hi - 1] * e[hi - 1]
    h = 0.5 * (a11 - a22)
    den = h + np.copysign(np.hypot(h, a12), h if h != 0.0 else 1.0)
    return a22 if den == 0.0 else a22 - a12 * a12 / den


def _sweep(d, e, lo, hi, lmats, rmats):
    # one bulge chase on [lo, hi] (bdc.py:218-244)
    mu = _shift(d, e, lo, hi)
    f = d[lo] * d[lo] - mu
    g = d[lo] * e[lo]
    for k in range(lo, hi):
        c, s, r = lartg(f, g)
        if k > lo:
            e[k - 1] = r
        f = c * d[k] + s * e[k]
        e[k] = c * e[k] - s * d[k]
        g = s * d[k + 1]
        d[k + 1] = c * d[k + 1]
        _rot_cols(rmats, k, k + 1, c, s)
        c, s, r = lartg(f, g)
        d[k] = r
        f = c * e[k] + s * d[k + 1]
        d[k + 1] = c * d[k + 1] - s * e[k]
        if k < hi - 1:
            g = s * e[k + 1]
            e[k + 1] = c * e[k + 1]
        _rot_cols(lmats, k, k + 1, c, s)
    e[hi - 1] = f


def _zero_diag_row(d, e, k, hi, lmats):
    # bdc.py:247-257
    f = e[k]
    e[k] = 0.0
    for j in range(k + 1, hi + 1):
        c, s, r = lartg(d[j], f)
        d[j] = r
        if j < hi:
            f = -s * e[j]
            e[j] = c * e[j]
        _rot_cols(lmats, j, k, c, s)


def _zero_diag_last(d, e, hi, lo, rmats):
    # bdc.py:260-270
    f = e[hi - 1]
    e[hi - 1] = 0.0
    for j in range(hi - 1, lo - 1, -1):
        c, s, r = lartg(d[j], f)
        d[j] = r
        if j > lo:
            f = -s * e[j - 1]
            e[j - 1] = c * e[j - 1]
        _rot_cols(rmats, j, hi, c, s)


def qr_diagonalize(d, e, lmats, rmats):
    """Square bidiagonal QR iteration in place (bdc.py:273-312)."""
    n = d.size
    if n == 0:
        return
    bnorm = max(np.max(np.abs(d)), np.max(np.abs(e)) if e.size else 0.0)
    if bnorm == 0.0:
        return
    limit = 60 * n * max(n, 4)
    used = 0
    hi = n - 1
    while hi > 0:
        if _small(e[hi - 1], d[hi - 1], d[hi], bnorm):
            e[hi - 1] = 0.0
            hi -= 1
            continue
        lo = hi - 1
        while lo > 0 and not _small(e[lo - 1], d[lo - 1], d[lo], bnorm):
            lo -= 1
        if lo > 0:
            e[lo - 1] = 0.0
        hit = -1
        for k in range(lo, hi + 1):
            if abs(d[k]) <= EPS * bnorm * 1e-3:
                hit = k
                break
        if hit >= 0:
            d[hit] = 0.0
            if hit < hi:
                _zero_diag_row(d, e, hit, hi, lmats)
            else:
                _zero_diag_last(d, e, hi, lo, rmats)
            continue
        _sweep(d, e, lo, hi, lmats, rmats)
        used += hi - lo
        if used > limit:
            raise SolverBudgetError(f"QR iteration exceeded {limit} rotations (n={n})")


def leaf_svd(prob, vectors=True):
    """Leaf SVD (bdc.py:315-359): bordered column chased in, QR iteration,
    sign fixes into W, stable ascending sort."""
    n, nc = prob.n, prob.ncols
    edge = np.zeros((2, nc))
    if nc:
        edge[0, 0] = 1.0
        edge[1, nc - 1] = 1.0
    W = np.eye(n, order="F") if vectors else None
    Q = np.eye(nc, order="F") if vectors else None
    if n == 0:
        return NodeSVD(np.zeros(0), W, Q, edge)
    d = prob.d.copy()
    e = prob.e[: n - 1].copy()
    lm = [W] if vectors else []
    rm = [Q, edge] if vectors else [edge]
    if prob.bordered:
        f = prob.e[n - 1]
        for i in range(n - 1, -1, -1):
            c, s, r = lartg(d[i], f)
            d[i] = r
            if i > 0:
                f = -s * e[i - 1]
                e[i - 1] = c * e[i - 1]
            _rot_cols(rm, i, n, c, s)
            if s == 0.0:
                break
    qr_diagonalize(d, e, lm, rm)
    neg = d < 0.0
    d[neg] = -d[neg]
    if vectors:
        W[:, neg] = -W[:, neg]
    order = np.argsort(d, kind="stable")
    if vectors:
        W[:, :] = W[:, order]
    for m in rm:
        m[:, :n] = m[:, order]
    return NodeSVD(d[order], W, Q, edge)


# ---------------------------------------------------------------------------
# divide / merge (bdc.py:366-847)


def split_rows(prob):
    """k = n//2: bordered left child of k-1 rows, right child n-k rows
    bordered iff the parent is; alpha = d[k-1], beta = e[k-1] (bdc.py:366-379)."""
    n = prob.n
    if n < 2:
        raise ValueError("cannot split fewer than 2 rows")
    k = n // 2
    left = Bidiag(prob.d[: k - 1], prob.e[: k - 1], True)
    right = Bidiag(prob.d[k:], prob.e[k:], prob.bordered)
    return left, right, float(prob.d[k - 1]), float(prob.e[k - 1])


def merge_inputs(prob, L, R):
    """Pre-sort (d, z) and the bordered coupling (bdc.py:382-412)."""
    nl, nr = L.vals.size, R.vals.size
    alpha = float(prob.d[nl])
    beta = float(prob.e[nl])
    last1 = L.edge[1]
    first2 = R.edge[0]
    d = np.concatenate(([0.0], L.vals, R.vals))
    z = np.empty(d.size)
    z[1:1 + nl] = alpha * last1[:nl]
    z[1 + nl:] = beta * first2[:nr]
    if prob.bordered:
        c, s, r = lartg(alpha * last1[nl], beta * first2[nr])
        z[0] = r
        return d, z, (c, s)
    z[0] = alpha * last1[nl]
    return d, z, None


def deflate_entries(d, z, lcols=None, rcols=None, edge=None, lcls=None, rcls=None, tol_mult=8.0):
    """Sort + deflation (bdc.py:423-508).  Rotations go straight into the
    supplied column sets.  Returns dict with kept, deflated, dvals (deflated
    values), perm, d, z, rotations, and the surviving system (ds, zs)."""
    d = np.array(d, dtype=np.float64)
    z = np.array(z, dtype=np.float64)
    n = d.size
    perm = np.argsort(d, kind="stable")
    d, z = d[perm], z[perm]
    if d[0] != 0.0:
        raise ValueError("deflation needs the zero border entry")
    for m in (lcols, rcols, edge):
        if m is not None:
            m[:, :n] = m[:, perm]
    for cl in (lcls, rcls):
        if cl is not None:
            cl[:n] = cl[perm]
    tol = tol_mult * EPS * max(np.max(np.abs(d)), np.max(np.abs(z)), 0.0)
    if abs(z[0]) <= tol:
        z[0] = np.copysign(max(tol, TINY), z[0] if z[0] != 0.0 else 1.0)
    kept = [0]
    defl, dval, rots = [], [], []
    for j in range(1, n):
        if abs(z[j]) <= tol:
            z[j] = 0.0
            defl.append(j)
            dval.append(d[j])
            continue
        p = kept[-1]
        if d[j] - d[p] <= tol:
            c, s, r = lartg(z[p], z[j])
            z[p], z[j] = r, 0.0
            rots.append((p, j, c, s))
            if p == 0:
                _rot_cols([rcols, edge], p, j, c, s)
                if rcls is not None:
                    rcls[p] = rcls[j] = rcls[p] if rcls[p] == rcls[j] else MIXED
                dval.append(0.0)
            else:
                d[p] = d[j]
                _rot_cols([lcols, rcols, edge], p, j, c, s)
                for cl in (lcls, rcls):
                    if cl is not None:
                        cl[p] = cl[j] = cl[p] if cl[p] == cl[j] else MIXED
                dval.append(d[j])
            defl.append(j)
        else:
            kept.append(j)
    kept = np.asarray(kept, dtype=np.intp)
    return dict(
        kept=kept,
        deflated=np.asarray(defl, dtype=np.intp),
        dvals=np.asarray(dval, dtype=np.float64),
        perm=perm,
        d=d,
        z=z,
        rotations=rots,
        ds=d[kept],
        zs=z[kept],
    )


def secular_roots(d, z, lanes=None, max_iter=100):
    """Frozen-lane rational-interpolation secular solver in the offset
    variable mu (bdc.py:541-641).  Returns (omega, anchor, mu)."""
    d = np.asarray(d, dtype=np.float64)
    z = np.asarray(z, dtype=np.float64)
    n = d.size
    ii = np.arange(n) if lanes is None else np.asarray(lanes)
    z2 = z * z
    zz = float(np.sum(z2))
    if n == 1:
        w = np.sqrt(zz)
        return np.full(ii.size, w), np.zeros(ii.size, dtype=np.intp), np.full(ii.size, zz)
    top = ii == n - 1
    lo_i = ii
    hi_i = np.where(top, n - 1, np.minimum(ii + 1, n - 1))
    dl, dh = d[lo_i], d[hi_i]
    width = np.where(top, zz, (dh - dl) * (dh + dl))
    with np.errstate(all="ignore"):
        fmid = 1.0 + np.sum(z2[None, :] / ((d[None, :] - dl[:, None]) * (d[None, :] + dl[:, None]) - 0.5 * width[:, None]), axis=1)
    lower = fmid > 0.0
    anc = np.where(lower | top, lo_i, hi_i)
    da = d[anc]
    off = (d[None, :] - da[:, None]) * (d[None, :] + da[:, None])
    gl = off[np.arange(ii.size), lo_i]
    gh = np.where(top, gl + zz, off[np.arange(ii.size), hi_i])
    lo = np.where(lower, 0.0, np.where(top, 0.5 * width, -0.5 * width))
    hi = np.where(lower, 0.5 * width, np.where(top, width, 0.0))
    mu = 0.5 * (lo + hi)
    left_mask = np.arange(n)[None, :] <= ii[:, None]
    live = np.ones(ii.size, dtype=bool)
    ftol = 8.0 * n * EPS
    for _ in range(max_iter):
        with np.errstate(all="ignore"):
            den = off - mu[:, None]
            t = z2[None, :] / den
            f = 1.0 + t.sum(axis=1)
            sa = 1.0 + np.abs(t).sum(axis=1)
            narrow = (hi - lo) <= 8.0 * EPS * np.maximum(np.abs(lo), np.abs(hi))
            live &= ~((np.abs(f) <= ftol * sa) | narrow | ~np.isfinite(f))
            if not live.any():
                break
            neg = live & (f < 0.0)
            pos = live & ~(f < 0.0)
            lo = np.where(neg, mu, lo)
            hi = np.where(pos, mu, hi)
            t2 = t / den
            psi = np.where(left_mask, t, 0.0).sum(axis=1)
            phi = np.where(left_mask, 0.0, t).sum(axis=1)
            dpsi = np.where(left_mask, t2, 0.0).sum(axis=1)
            dphi = np.where(left_mask, 0.0, t2).sum(axis=1)
            a_ = gl - mu
            b_ = gh - mu
            S = dpsi * a_ * a_
            R = dphi * b_ * b_
            s0 = 1.0 + (psi - dpsi * a_) + (phi - dphi * b_)
            qb = -(s0 * (a_ + b_) + S + R)
            qc = s0 * a_ * b_ + S * b_ + R * a_
            sq = np.sqrt(np.maximum(qb * qb - 4.0 * s0 * qc, 0.0))
            qq = -0.5 * (qb + np.where(qb >= 0.0, sq, -sq))
            e1 = qq / s0
            e2 = qc / qq
            c1, c2 = mu + e1, mu + e2
            ok1 = np.isfinite(c1) & (c1 > lo) & (c1 < hi)
            ok2 = np.isfinite(c2) & (c2 > lo) & (c2 < hi)
            take1 = ok1 & (~ok2 | (np.abs(e1) <= np.abs(e2)))
            mu = np.where(live, np.where(take1, c1, np.where(ok2, c2, 0.5 * (lo + hi))), mu)
    if live.any():
        raise SolverBudgetError(f"secular solver: {int(live.sum())} roots did not converge")
    return np.sqrt(np.maximum(da * da + mu, 0.0)), anc.astype(np.intp), mu


def loewner_z(d, z, anc, mu):
    """Gu-Eisenstat z recomputation from the roots (bdc.py:644-673)."""
    n = d.size
    da = d[anc]
    num = (da[None, :] - d[:, None]) * (da[None, :] + d[:, None]) + mu[None, :]
    if n == 1:
        rad = num[:, 0]
    else:
        dlo = (d[None, :-1] - d[:, None]) * (d[None, :-1] + d[:, None])
        dhi = (d[None, 1:] - d[:, None]) * (d[None, 1:] + d[:, None])
        below = np.arange(n - 1)[None, :] < np.arange(n)[:, None]
        rad = num[:, n - 1] * np.prod(num[:, : n - 1] / np.where(below, dlo, dhi), axis=1)
    if not np.all(rad > 0.0):
        raise ArithmeticError("interlacing violated in z recomputation")
    return np.copysign(np.sqrt(rad), z)


def secular_vecs(d, anc, mu, zt):
    """Middle-matrix singular vectors (bdc.py:676-694)."""
    da = d[anc]
    den = (d[None, :] - da[:, None]) * (d[None, :] + da[:, None]) - mu[:, None]
    v = (zt[None, :] / den).T
    u = d[:, None] * v
    u[0, :] = -1.0
    return np.asfortranarray(u / np.linalg.norm(u, axis=0)), np.asfortranarray(v / np.linalg.norm(v, axis=0))


def _blocked_product(cols, cls, kept, small, top, bottom, unit_row=None):
    # class-structured cols[:, kept] @ small (bdc.py:701-728)
    out = np.zeros((cols.shape[0], small.shape[1]), order="F")
    kc = cls[kept]
    for c, rows in ((MIXED, slice(None)), (FIRST, slice(0, top)), (SECOND, slice(bottom, None))):
        g = np.flatnonzero(kc == c)
        if g.size:
            out[rows, :] += cols[rows, kept[g]] @ small[g, :]
    g = np.flatnonzero(kc == UNIT)
    if g.size:
        out[unit_row, :] += small[g[0], :]
    return out


def merge_node(prob, L, R, vectors, tol_mult):
    """One merge (bdc.py:768-847)."""
    nl, nr = L.vals.size, R.vals.size
    n = prob.n
    nc = prob.ncols
    bord = prob.bordered
    d0, z0, cs = merge_inputs(prob, L, R)
    f1, l2 = L.edge[0], R.edge[1]
    edge = np.zeros((2, n))
    edge[0, 1:1 + nl] = f1[:nl]
    edge[1, 1 + nl:] = l2[:nr]
    if bord:
        c, s = cs
        edge[0, 0] = c * f1[nl]
        edge[1, 0] = s * l2[nr]
        null_edge = np.array([-s * f1[nl], c * l2[nr]])
    else:
        edge[0, 0] = f1[nl]
        null_edge = None
    rcls = np.full(n, MIXED if bord else FIRST)
    rcls[1:1 + nl] = FIRST
    rcls[1 + nl:] = SECOND
    lcls = np.full(n, UNIT)
    lcls[1:1 + nl] = FIRST
    lcls[1 + nl:] = SECOND
    lpre = rpre = null_col = None
    if vectors:
        lpre = np.zeros((n, n), order="F")
        lpre[nl, 0] = 1.0
        lpre[:nl, 1:1 + nl] = L.W
        lpre[nl + 1:, 1 + nl:] = R.W
        rpre = np.zeros((nc, n), order="F")
        q1 = np.zeros(nc)
        q1[: nl + 1] = L.Q[:, nl]
        if bord:
            c, s = cs
            q2 = np.zeros(nc)
            q2[nl + 1:] = R.Q[:, nr]
            rpre[:, 0] = c * q1 + s * q2
            null_col = -s * q1 + c * q2
        else:
            rpre[:, 0] = q1
        rpre[: nl + 1, 1:1 + nl] = L.Q[:, :nl]
        rpre[nl + 1:, 1 + nl:] = R.Q[:, :nr]
    out = deflate_entries(d0, z0, lpre, rpre, edge, lcls, rcls, tol_mult)
    om, anc, mu = secular_roots(out["ds"], out["zs"])
    zt = loewner_z(out["ds"], out["zs"], anc, mu)
    umat, vmat = secular_vecs(out["ds"], anc, mu, zt)
    kept, defl = out["kept"], out["deflated"]
    vals = np.concatenate([om, out["dvals"]])
    ecols = np.hstack([edge[:, kept] @ vmat, edge[:, defl]])
    order = np.argsort(vals, kind="stable")
    new_edge = np.empty((2, nc))
    new_edge[:, :n] = ecols[:, order]
    if bord:
        new_edge[:, n] = null_edge
    if not vectors:
        return NodeSVD(vals[order], None, None, new_edge)
    wk = _blocked_product(lpre, lcls, kept, umat, nl, nl + 1, unit_row=nl)
    qk = _blocked_product(rpre, rcls, kept, vmat, nl + 1, nl + 1)
    Wn = np.asfortranarray(np.hstack([wk, lpre[:, defl]])[:, order])
    Qn = np.zeros((nc, nc), order="F")
    Qn[:, :n] = np.hstack([qk, rpre[:, defl]])[:, order]
    if bord:
        Qn[:, n] = null_col
    return NodeSVD(vals[order], Wn, Qn, new_edge)


def _empty(prob, vectors):
    nc = prob.ncols
    edge = np.zeros((2, nc))
    if nc:
        edge[0, 0] = 1.0
        edge[1, nc - 1] = 1.0
    return NodeSVD(np.zeros(0), np.zeros((0, 0)) if vectors else None,
                   np.eye(nc, order="F") if vectors else None, edge)


def _solve(prob, vectors, leaf, tol_mult):
    # depth-first recursion (bdc.py:850-858)
    if prob.n == 0:
        return _empty(prob, vectors)
    if prob.n <= leaf:
        return leaf_svd(prob, vectors)
    lp, rp, _, _ = split_rows(prob)
    return merge_node(prob, _solve(lp, vectors, leaf, tol_mult),
                      _solve(rp, vectors, leaf, tol_mult), vectors, tol_mult)


def bdc(prob, vectors=True, leaf=32, tol_mult=8.0):
    """Bidiagonal SVD by divide and conquer, values descending
    (bdc.py:861-880)."""
    if leaf < 1:
        raise ValueError("leaf must be >= 1")
    res = _solve(prob, vectors, leaf, tol_mult)
    n = res.vals.size
    rev = np.arange(n)[::-1]
    edge = res.edge.copy()
    edge[:, :n] = edge[:, rev]
    W = Q = None
    if vectors:
        W = np.asfortranarray(res.W[:, rev])
        Q = res.Q.copy(order="F")
        Q[:, :n] = Q[:, rev]
    return NodeSVD(res.vals[rev].copy(), W, Q, edge)
