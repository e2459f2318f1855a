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
