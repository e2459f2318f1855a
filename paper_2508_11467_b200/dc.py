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


def solve_all_roots(system, max_iterations=100):
    """All roots of the secular system, one warp per root (bdc.py:515-641).
    Frozen-lane iteration: each root's result is independent of the others."""
    if max_iterations != 100:
        raise ValueError("the GPU secular solver uses the reference's fixed 100-iteration budget")
    d, z, torch_in = _sys_vectors(system)
    K = d.numel()
    h = _lib.handle()
    om = torch.empty(K, dtype=torch.float64, device=d.device)
    mu = torch.empty(K, dtype=torch.float64, device=d.device)
    anc = torch.empty(K, dtype=torch.int32, device=d.device)
    rc = _lib.load_library().dcsvd_secular_roots(h, K, _lib.ptr(d), _lib.ptr(z), _lib.ptr(om), _lib.ptr(anc),
                                                 _lib.ptr(mu), _lib.stream_ptr())
    _lib.check(rc, h)
    anc = anc.to(torch.int64)
    if torch_in:
        return SecularRoots(om, anc, mu)
    return SecularRoots(om.cpu().numpy(), anc.cpu().numpy().astype(np.intp), mu.cpu().numpy())


def solve_secular(system, i, max_iterations=100):
    """Root i as (omega, anchor, mu) (bdc.py:528-538); bitwise the batched lane."""
    r = solve_all_roots(system, max_iterations)
    return float(r.omega[i]), int(r.anchor[i]), float(r.mu[i])


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


def bdsqr_base(prob, want_vectors=True):
    """Leaf SVD by implicit-shift QR iteration (bdc.py:315-359), values
    ascending (the tree-internal convention).  GPU leaf kernel: n <= 32."""
    if prob.n > 32:
        raise ValueError(f"GPU leaf solver handles n <= 32, got {prob.n}")
    r = bdsdc(prob, want_vectors=want_vectors, leaf=max(prob.n, 1))
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
