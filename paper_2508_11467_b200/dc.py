"""GPU bidiagonal divide and conquer with the reference API of
pkg/src/dcsvd/bdc.py (``BidiagonalProblem`` :56-96, ``SubproblemSVD`` :99-117,
``bdsdc`` :861-880).  The whole recursion -- leaves, deflation, secular
roots, Loewner vectors, merge GEMMs -- runs on the device (csrc/bdc.cu)."""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


@dataclass
class BidiagonalProblem:
    """Upper bidiagonal d (n), e (n-1 or n; e[n-1] is the border entry when
    ``bordered``)."""

    d: object
    e: object
    bordered: bool = False

    def __post_init__(self):
        self._torch = isinstance(self.d, torch.Tensor)
        if self._torch:
            self.d = self.d.to(torch.float64).reshape(-1)
            e = torch.as_tensor(self.e, dtype=torch.float64, device=self.d.device).reshape(-1)
            n = self.d.numel()
            if n and e.numel() == n - 1:
                e = torch.cat([e, e.new_zeros(1)])
            if e.numel() != n:
                raise ValueError(f"superdiagonal must have {max(n - 1, 0)} or {n} entries, got {e.numel()}")
            self.e = e
            return
        self.d = np.atleast_1d(np.asarray(self.d, dtype=np.float64))
        e = np.atleast_1d(np.asarray(self.e, dtype=np.float64))
        n = self.d.size
        if n and e.size == n - 1:
            e = np.append(e, 0.0)
        if e.size != n:
            raise ValueError(f"superdiagonal must have {max(n - 1, 0)} or {n} entries, got {e.size}")
        self.e = e

    @property
    def n(self):
        return int(self.d.numel() if self._torch else self.d.size)

    @property
    def ncols(self):
        return self.n + (1 if self.bordered else 0)

    def dense(self):
        d = self.d.cpu().numpy() if self._torch else self.d
        e = self.e.cpu().numpy() if self._torch else self.e
        b = np.zeros((self.n, self.ncols))
        for i in range(self.n):
            b[i, i] = d[i]
            if i + 1 < self.ncols:
                b[i, i + 1] = e[i]
        return b


@dataclass
class SubproblemSVD:
    """B = W diag(dvals) [Q | q]^T with dvals descending; ``edge_rows`` =
    first and last row of ``qfull`` (kept in values-only mode too)."""

    dvals: object
    w: object
    qfull: object
    edge_rows: object

    @property
    def n(self):
        return int(self.dvals.shape[0])


@_lib.on_input_device
def bdsdc(prob, want_vectors=True, leaf=32, tol_multiple=8.0):
    """SVD of a bidiagonal problem by divide and conquer on the GPU
    (bdc.py:861-880).  Values descending; values-only runs are bitwise equal
    to vector runs (one shared code path for everything feeding the values)."""
    if leaf < 1:
        raise ValueError(f"leaf size must be >= 1, got {leaf}")
    if not isinstance(prob, BidiagonalProblem):
        raise TypeError("expected a BidiagonalProblem")
    h = _lib.handle()
    n, nc = prob.n, prob.ncols
    d = _lib.vec_to_device(prob.d, n) if n else torch.zeros(1, dtype=torch.float64, device="cuda")
    e = _lib.vec_to_device(prob.e, n) if n else torch.zeros(1, dtype=torch.float64, device="cuda")
    dev = d.device
    dvals = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    edge = torch.empty(2 * max(nc, 1), dtype=torch.float64, device=dev)
    W = _lib.colmajor_empty(max(n, 1), max(n, 1)) if want_vectors else None
    Q = _lib.colmajor_empty(max(nc, 1), max(nc, 1)) if want_vectors else None
    rc = _lib.load_library().dcsvd_bdsdc(
        h, n, _lib.ptr(d), _lib.ptr(e), int(bool(prob.bordered)), int(bool(want_vectors)), int(leaf),
        float(tol_multiple), _lib.ptr(dvals), _lib.ptr(W), _lib.ld(W) if W is not None else 1, _lib.ptr(Q),
        _lib.ld(Q) if Q is not None else 1, _lib.ptr(edge), _lib.stream_ptr())
    _lib.check(rc, h)
    dvals = dvals[:n]
    edge = edge[: 2 * nc].reshape(nc, 2).t()
    if W is not None:
        W = W[:n, :n]
        Q = Q[:nc, :nc]
    if prob._torch:
        return SubproblemSVD(dvals, W, Q, edge)
    return SubproblemSVD(dvals.cpu().numpy(), _lib.to_host(W) if W is not None else None,
                         _lib.to_host(Q) if Q is not None else None, np.ascontiguousarray(edge.cpu().numpy()))


@dataclass
class SecularSystem:
    """Surviving entries after deflation (bdc.py:120-135): d ascending with
    d[0] = 0, z, norm_bound."""

    d: object
    z: object
    norm_bound: float

    @property
    def n(self):
        return int(self.d.shape[0])


@dataclass
class SecularRoots:
    """Roots as (omega, anchor pole, mu = omega^2 - d[anchor]^2) (bdc.py:138-149)."""

    omega: object
    anchor: object
    mu: object


def _sys_vectors(system):
    torch_in = isinstance(system.d, torch.Tensor)
    d = _lib.vec_to_device(system.d)
    z = _lib.vec_to_device(system.z, d.numel())
    return d, z, torch_in


@_lib.on_input_device
def solve_all_roots(system, max_iterations=100):
    """All roots of the secular system, one warp per root (bdc.py:515-641).
    Frozen-lane iteration: each root's result is independent of the others."""
    d, z, torch_in = _sys_vectors(system)
    K = d.numel()
    h = _lib.handle()
    om = torch.empty(K, dtype=torch.float64, device=d.device)
    mu = torch.empty(K, dtype=torch.float64, device=d.device)
    anc = torch.empty(K, dtype=torch.int32, device=d.device)
    rc = _lib.load_library().dcsvd_secular_roots(h, K, _lib.ptr(d), _lib.ptr(z), _lib.ptr(om), _lib.ptr(anc),
                                                 _lib.ptr(mu), int(max_iterations), _lib.stream_ptr())
    _lib.check(rc, h)
    anc = anc.to(torch.int64)
    if torch_in:
        return SecularRoots(om, anc, mu)
    return SecularRoots(om.cpu().numpy(), anc.cpu().numpy().astype(np.intp), mu.cpu().numpy())


@_lib.on_input_device
def solve_secular(system, i, max_iterations=100):
    """Root i as (omega, anchor, mu) (bdc.py:528-538); bitwise the batched lane."""
    r = solve_all_roots(system, max_iterations)
    return float(r.omega[i]), int(r.anchor[i]), float(r.mu[i])


@_lib.on_input_device
def recompute_z(system, roots):
    """Loewner update vector consistent with the roots (bdc.py:644-673)."""
    d, z, torch_in = _sys_vectors(system)
    K = d.numel()
    h = _lib.handle()
    anc = _lib.vec_to_device(roots.anchor).to(torch.int32) if not isinstance(roots.anchor, torch.Tensor) else \
        roots.anchor.to(device=d.device, dtype=torch.int32).contiguous()
    mu = _lib.vec_to_device(roots.mu, K)
    zt = torch.empty(K, dtype=torch.float64, device=d.device)
    rc = _lib.load_library().dcsvd_recompute_z(h, K, _lib.ptr(d), _lib.ptr(z), _lib.ptr(anc), _lib.ptr(mu),
                                               _lib.ptr(zt), _lib.stream_ptr())
    _lib.check(rc, h)
    return zt if torch_in else zt.cpu().numpy()


@_lib.on_input_device
def secular_vectors(system, roots, ztilde):
    """(umat, vmat) singular vectors of the middle matrix (bdc.py:676-694)."""
    d, _, torch_in = _sys_vectors(system)
    K = d.numel()
    h = _lib.handle()
    anc = roots.anchor.to(device=d.device, dtype=torch.int32).contiguous() if isinstance(roots.anchor, torch.Tensor) \
        else _lib.vec_to_device(roots.anchor).to(torch.int32)
    mu = _lib.vec_to_device(roots.mu, K)
    zt = _lib.vec_to_device(ztilde, K)
    U = _lib.colmajor_empty(K, K)
    V = _lib.colmajor_empty(K, K)
    rc = _lib.load_library().dcsvd_secular_vectors(h, K, _lib.ptr(d), _lib.ptr(anc), _lib.ptr(mu), _lib.ptr(zt),
                                                   _lib.ptr(U), _lib.ld(U), _lib.ptr(V), _lib.ld(V), _lib.stream_ptr())
    _lib.check(rc, h)
    if torch_in:
        return U, V
    return _lib.to_host(U), _lib.to_host(V)


def split(prob):
    """Remove the middle row k = n//2 (bdc.py:366-379): (left bordered child of
    k-1 rows, right child bordered iff the parent, alpha = d[k-1], beta = e[k-1]).
    Pure index bookkeeping on the host; the GPU tree (csrc/bdc.cu) uses the same rule."""
    n = prob.n
    if n < 2:
        raise ValueError(f"cannot split a problem with {n} rows")
    k = n // 2
    left = BidiagonalProblem(prob.d[: k - 1], prob.e[: k - 1], bordered=True)
    right = BidiagonalProblem(prob.d[k:], prob.e[k:], bordered=prob.bordered)
    return left, right, float(prob.d[k - 1]), float(prob.e[k - 1])


@_lib.on_input_device
def bdsqr_base(prob, want_vectors=True):
    """Leaf SVD by implicit-shift QR iteration (bdc.py:315-359), values
    ascending (the tree-internal convention).  n <= 32 runs the GPU leaf
    kernel itself; larger problems go through the GPU divide and conquer with
    32-row leaves (the same decomposition up to rounding)."""
    r = bdsdc(prob, want_vectors=want_vectors, leaf=min(max(prob.n, 1), 32))
    n = prob.n
    flip = lambda x: x.flip(0) if isinstance(x, torch.Tensor) else x[::-1].copy()
    vals = flip(r.dvals)
    edge = r.edge_rows
    if isinstance(edge, torch.Tensor):
        edge = edge.clone()
        edge[:, :n] = edge[:, :n].flip(1)
    else:
        edge = edge.copy()
        edge[:, :n] = edge[:, :n][:, ::-1]
    w = q = None
    if want_vectors:
        if isinstance(r.w, torch.Tensor):
            w = r.w.flip(1)
            q = r.qfull.clone()
            q[:, :n] = q[:, :n].flip(1)
        else:
            w = np.asfortranarray(r.w[:, ::-1])
            q = r.qfull.copy(order="F")
            q[:, :n] = q[:, :n][:, ::-1]
    return SubproblemSVD(vals, w, q, edge)


# ---------------------------------------------------------------------------
# standalone merge stages (bdc.py:382-747): build_z, deflate, merge_vectors.
# The fused GPU tree (bdsdc) runs the same steps inside its level kernels;
# these entry points expose them one merge at a time with the reference's
# signatures and in-place conventions.

CLASS_UNIT, CLASS_FIRST, CLASS_SECOND, CLASS_MIXED = 0, 1, 2, 3  # bdc.py:173-176


@dataclass
class DeflationOutcome:
    """Deflation bookkeeping for one merge, in sorted working order
    (bdc.py:152-170): ``kept``/``deflated`` index the sorted (d, z);
    ``applied_rotations`` lists (i, j, GivensRotation) already applied to the
    supplied columns; ``permutation`` maps working order back to the caller's
    pre-sort order; ``d``/``z`` are the working copies after the rotations."""

    system: SecularSystem
    kept: object
    deflated: object
    deflated_values: object
    applied_rotations: list
    permutation: object
    d: object
    z: object


def _edge_dev(edge):
    t, _ = _lib.to_device_colmajor(edge, copy=False)
    return t


@_lib.on_input_device
def build_z(node, left, right):
    """Middle-row data of a merge (bdc.py:382-412): (d, z, coupling) in
    pre-sort order [border, left child values, right child values]; coupling
    is the GivensRotation of the two null directions of a bordered node, else
    None.  One GPU kernel."""
    from .blas import GivensRotation

    nl, nr = left.n, right.n
    alpha = float(node.d[nl])
    beta = float(node.e[nl])
    torch_in = isinstance(node.d, torch.Tensor)
    ldv = _lib.vec_to_device(left.dvals, nl)
    rdv = _lib.vec_to_device(right.dvals, nr)
    le, re_ = _edge_dev(left.edge_rows), _edge_dev(right.edge_rows)
    if tuple(le.shape) != (2, nl + 1) or tuple(re_.shape) != (2, nr + int(bool(node.bordered))):
        raise ValueError("child edge rows must be 2 x ncols (left child bordered, right child bordered iff the node)")
    n = nl + nr + 1
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    z = torch.empty(n, dtype=torch.float64, device="cuda")
    cp = torch.empty(2, dtype=torch.float64, device="cuda")
    h = _lib.handle()
    rc = _lib.load_library().dcsvd_build_z(h, nl, nr, int(bool(node.bordered)), alpha, beta, _lib.ptr(ldv),
                                           _lib.ptr(le), _lib.ld(le), _lib.ptr(rdv), _lib.ptr(re_), _lib.ld(re_),
                                           _lib.ptr(d), _lib.ptr(z), _lib.ptr(cp), _lib.stream_ptr())
    _lib.check(rc, h)
    c, s = cp.cpu().tolist()
    coupling = GivensRotation(c, s) if node.bordered else None
    if torch_in:
        return d, z, coupling
    return d.cpu().numpy(), z.cpu().numpy(), coupling


class _InPlace:
    """Device view of a caller matrix/vector that deflate updates in place;
    numpy (or non-column-major) inputs are staged and written back."""

    def __init__(self, x, cls=False):
        self.x = x
        self.dev = None
        if x is None:
            return
        if cls:
            t = torch.as_tensor(np.asarray(x) if not isinstance(x, torch.Tensor) else x)
            self.dev = t.to(device="cuda", dtype=torch.int32).contiguous()
        elif isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float64 and _lib.is_colmajor(x):
            self.dev = x
        else:
            self.dev, _ = _lib.to_device_colmajor(x, copy=True)

    def ptr(self):
        return _lib.ptr(self.dev)

    def write_back(self):
        x = self.x
        if x is None or self.dev is x:
            return
        if isinstance(x, torch.Tensor):
            x.copy_(self.dev.to(dtype=x.dtype))
        elif self.dev.dtype == torch.int32:
            x[...] = self.dev.cpu().numpy().astype(x.dtype)
        else:
            x[...] = _lib.to_host(self.dev)


@_lib.on_input_device
def deflate(d, z, left_vectors=None, right_vectors=None, *, edge_rows=None, left_classes=None, right_classes=None,
            tol_multiple=8.0):
    """Sort the merge entries and deflate the negligible ones (bdc.py:423-508).
    Works on copies of (d, z); permutes/rotates the supplied column matrices
    and class arrays in place.  Stable sort and the sequential deflation scan
    run in one GPU CTA, the column permutation and the recorded Givens
    rotations in row-parallel kernels."""
    from .blas import GivensRotation

    torch_in = isinstance(d, torch.Tensor)
    dd = _lib.vec_to_device(d)
    n = dd.numel()
    zz = _lib.vec_to_device(z, n)
    mats = [_InPlace(left_vectors), _InPlace(right_vectors), _InPlace(edge_rows)]
    for m in mats:
        if m.dev is not None and m.dev.shape[1] < n:
            raise ValueError(f"vector matrices need at least {n} columns")
    cls = [_InPlace(left_classes, cls=True), _InPlace(right_classes, cls=True)]
    i64 = dict(dtype=torch.int64, device="cuda")
    f64 = dict(dtype=torch.float64, device="cuda")
    perm, kept, defl, rot_pq = (torch.empty(n, **i64), torch.empty(n, **i64), torch.empty(n, **i64),
                                torch.empty(2 * n, **i64))
    d_out, z_out, dvals, rot_cs = (torch.empty(n, **f64), torch.empty(n, **f64), torch.empty(n, **f64),
                                   torch.empty(2 * n, **f64))
    counts = torch.zeros(3, **i64)
    rows = [int(m.dev.shape[0]) if m.dev is not None else 0 for m in mats]
    lds = [_lib.ld(m.dev) if m.dev is not None else 1 for m in mats]
    h = _lib.handle()
    rc = _lib.load_library().dcsvd_deflate(
        h, n, _lib.ptr(dd), _lib.ptr(zz), float(tol_multiple), mats[0].ptr(), rows[0], lds[0], mats[1].ptr(), rows[1],
        lds[1], mats[2].ptr(), lds[2], cls[0].ptr(), cls[1].ptr(), _lib.ptr(perm), _lib.ptr(d_out), _lib.ptr(z_out),
        _lib.ptr(kept), _lib.ptr(defl), _lib.ptr(dvals), _lib.ptr(rot_pq), _lib.ptr(rot_cs), _lib.ptr(counts),
        _lib.stream_ptr())
    _lib.check(rc, h)
    for m in mats + cls:
        m.write_back()
    nk, nd, nr = (int(v) for v in counts.cpu().tolist())
    kept, defl, dvals = kept[:nk], defl[:nd], dvals[:nd]
    pq = rot_pq[: 2 * nr].cpu().numpy().reshape(-1, 2)
    cs = rot_cs[: 2 * nr].cpu().numpy().reshape(-1, 2)
    rotations = [(int(p), int(q), GivensRotation(float(c), float(s))) for (p, q), (c, s) in zip(pq, cs)]
    dk, zk = d_out[kept], z_out[kept]
    hk = dk.cpu().numpy()
    norm_bound = float(np.sqrt(hk[-1] ** 2 + np.sum(zk.cpu().numpy() ** 2)))
    if torch_in:
        return DeflationOutcome(SecularSystem(dk, zk, norm_bound), kept, defl, dvals, rotations, perm, d_out, z_out)
    host = lambda t: t.cpu().numpy()
    idx = lambda t: t.cpu().numpy().astype(np.intp)
    return DeflationOutcome(SecularSystem(host(dk), host(zk), norm_bound), idx(kept), idx(defl), host(dvals),
                            rotations, idx(perm), host(d_out), host(z_out))


def _gather(src, row_idx, col_idx, rows, cols, dst=None):
    h = _lib.handle()
    if dst is None:
        dst = _lib.colmajor_empty(rows, cols)
    ri = None if row_idx is None else torch.as_tensor(np.asarray(row_idx, dtype=np.int64)).to("cuda")
    ci = None if col_idx is None else torch.as_tensor(np.asarray(col_idx, dtype=np.int64)).to("cuda")
    rc = _lib.load_library().dcsvd_gather(h, rows, cols, _lib.ptr(src), _lib.ld(src), _lib.ptr(ri), _lib.ptr(ci),
                                          _lib.ptr(dst), _lib.ld(dst), _lib.stream_ptr())
    _lib.check(rc, h)
    return dst


def _dgemm(m, n, k, A, lda, B, ldb, C, ldc, beta=1.0):
    if m == 0 or n == 0 or k == 0:
        return
    h = _lib.handle()
    rc = _lib.load_library().dcsvd_dgemm(h, 0, 0, m, n, k, 1.0, A, lda, B, ldb, beta, C, ldc, _lib.stream_ptr())
    _lib.check(rc, h)


def _structured_product(cols, classes, kept, small, top, bottom, unit_row=None):
    """out = cols[:, kept] @ small by class blocks (bdc.py:701-728): one
    full-height DMMA product for mixed columns, one over the top (rows < top)
    / bottom (rows >= bottom) block for first / second columns, plus the
    unit-row update.  Index bookkeeping on the host, data on the device."""
    rows, nout = int(cols.shape[0]), int(small.shape[1])
    out = _lib.colmajor_empty(rows, nout)
    out.zero_()
    cls = np.asarray(classes)[kept]
    ldo, lds_ = _lib.ld(out), _lib.ld(small)
    for which, r0, r1 in ((CLASS_MIXED, 0, rows), (CLASS_FIRST, 0, top), (CLASS_SECOND, bottom, rows)):
        g = np.flatnonzero(cls == which)
        if g.size == 0 or r1 <= r0:
            continue
        a = _gather(cols, np.arange(r0, r1), kept[g], r1 - r0, g.size)        # cols[r0:r1, kept[g]]
        b = _gather(small, g, None, g.size, nout)                              # small[g, :]
        _dgemm(r1 - r0, nout, g.size, _lib.ptr(a), _lib.ld(a), _lib.ptr(b), _lib.ld(b),
               ctypes_offset(out, r0), ldo)
    gu = np.flatnonzero(cls == CLASS_UNIT)
    if gu.size:
        if unit_row is None:
            raise ValueError("unit-class column without a unit row")
        one = torch.ones((1, 1), dtype=torch.float64, device="cuda")
        _dgemm(1, nout, 1, _lib.ptr(one), 1, ctypes_offset(small, int(gu[0])), lds_, ctypes_offset(out, unit_row), ldo)
    return out


def ctypes_offset(t, row, col=0):
    """Device pointer of element (row, col) of a column-major tensor."""
    import ctypes

    return ctypes.c_void_p(t.data_ptr() + 8 * (row + col * _lib.ld(t)))


@_lib.on_input_device
def merge_vectors(outcome, umat, vmat, left, right, left_classes, right_classes, mid_row):
    """Assemble a merged node's vector columns (bdc.py:731-747): kept columns
    through the structured DMMA products, deflated columns carried over.
    Returns (w_cols, q_cols) ordered [kept | deflated]."""
    torch_in = isinstance(left, torch.Tensor)
    kept = np.asarray(outcome.kept.cpu().numpy() if isinstance(outcome.kept, torch.Tensor) else outcome.kept,
                      dtype=np.intp)
    defl = np.asarray(outcome.deflated.cpu().numpy() if isinstance(outcome.deflated, torch.Tensor)
                      else outcome.deflated, dtype=np.intp)
    lc = left_classes.cpu().numpy() if isinstance(left_classes, torch.Tensor) else np.asarray(left_classes)
    rc_ = right_classes.cpu().numpy() if isinstance(right_classes, torch.Tensor) else np.asarray(right_classes)
    L, _ = _lib.to_device_colmajor(left, copy=False)
    R, _ = _lib.to_device_colmajor(right, copy=False)
    U, _ = _lib.to_device_colmajor(umat, copy=False)
    V, _ = _lib.to_device_colmajor(vmat, copy=False)
    outs = []
    for M, cls, small, top, bottom, unit in ((L, lc, U, mid_row, mid_row + 1, mid_row),
                                             (R, rc_, V, mid_row + 1, mid_row + 1, None)):
        k_part = _structured_product(M, cls, kept, small, top, bottom, unit_row=unit)
        rows = int(M.shape[0])
        full = _lib.colmajor_empty(rows, k_part.shape[1] + defl.size)
        _gather(k_part, None, None, rows, k_part.shape[1], dst=full)
        if defl.size:
            _gather(M, None, defl, rows, defl.size, dst=full[:, k_part.shape[1]:])
        outs.append(full)
    if torch_in:
        return outs[0], outs[1]
    return _lib.to_host(outs[0]), _lib.to_host(outs[1])
