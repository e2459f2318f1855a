"""GPU bidiagonalization with the reference API of
pkg/src/dcsvd/bidiag.py (``gebrd_blocked`` :168, ``labrd_panel`` :113,
``gebrd_unblocked`` :75, ``BidiagonalFactorization`` :29, ``PanelWorkspace``
:51).  In place on ``a`` like the reference: numpy inputs are written back,
column-major CUDA tensors are updated in device memory."""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


@dataclass
class BidiagonalFactorization:
    """Packed A = U1 B V1^T: column reflector essentials below the diagonal,
    row reflector essentials right of the superdiagonal; d/e the bidiagonal;
    tauq/taup the scalars (taup[-1] == 0)."""

    packed: object
    d: object
    e: object
    tauq: object
    taup: object

    @property
    def shape(self):
        return tuple(self.packed.shape)


@dataclass
class PanelWorkspace:
    """P (m x 2b) / Q (n x 2b) panel storage (bidiag.py:51-63)."""

    p: object
    q: object

    @classmethod
    def allocate(cls, m, n, block):
        return cls(p=np.zeros((m, 2 * block), order="F"), q=np.zeros((n, 2 * block), order="F"))


def _require_tall(shape):
    m, n = shape
    if n < 1:
        raise ValueError("matrix must have at least one column")
    if m < n:
        raise ValueError(f"bidiagonalization requires m >= n, got {m}x{n}")
    return m, n


def _writeback(orig, dev, was_np):
    if was_np:
        orig[...] = _lib.to_host(dev)
        return orig
    if isinstance(orig, torch.Tensor) and dev.data_ptr() != orig.data_ptr():
        orig.copy_(dev)
        return orig
    return dev


def _out_vec(t, like_np):
    return t.cpu().numpy() if like_np else t


@_lib.on_input_device
def gebrd_blocked(a, block=32):
    """Blocked one-stage bidiagonalization in place (bidiag.py:168-204):
    cooperative LABRD panel kernel + one DMMA trailing GEMM per panel."""
    m, n = _require_tall(tuple(a.shape))
    if block < 1:
        raise ValueError(f"block width must be >= 1, got {block}")
    h = _lib.handle()
    A, was_np = _lib.to_device_colmajor(a, copy=False)
    dev = A.device
    d = torch.empty(n, dtype=torch.float64, device=dev)
    e = torch.empty(max(n - 1, 1), dtype=torch.float64, device=dev)
    tq = torch.empty(n, dtype=torch.float64, device=dev)
    tp = torch.empty(n, dtype=torch.float64, device=dev)
    rc = _lib.load_library().dcsvd_gebrd(h, m, n, _lib.ptr(A), _lib.ld(A), _lib.ptr(d), _lib.ptr(e), _lib.ptr(tq),
                                         _lib.ptr(tp), int(block), _lib.stream_ptr())
    _lib.check(rc, h)
    packed = _writeback(a, A, was_np)
    e = e[: n - 1]
    return BidiagonalFactorization(packed, _out_vec(d, was_np), _out_vec(e, was_np), _out_vec(tq, was_np),
                                   _out_vec(tp, was_np))


@_lib.on_input_device
def gebrd_unblocked(a):
    """Unblocked (GEBD2) reduction in place (bidiag.py:75-110)."""
    m, n = _require_tall(tuple(a.shape))
    return gebrd_blocked(a, block=max(n, 1))


@_lib.on_input_device
def labrd_panel(a, block, work, d, e, tauq, taup):
    """One merged rank-(2 block) panel of the view ``a`` (bidiag.py:113-165).
    Writes the panel rows/columns of ``a`` and the d/e/tauq/taup segments;
    returns the (P, Q) panel matrices (views into ``work``)."""
    m, n = tuple(a.shape)
    if not 1 <= block < n <= m:
        raise ValueError(f"panel width {block} needs block < ncols <= nrows, view is {m}x{n}")
    h = _lib.handle()
    A, was_np = _lib.to_device_colmajor(a, copy=False)
    P = _lib.colmajor_empty(m, 2 * block)
    Q = _lib.colmajor_empty(n, 2 * block)
    dev = A.device
    dd = torch.empty(block, dtype=torch.float64, device=dev)
    ee = torch.empty(block, dtype=torch.float64, device=dev)
    tq = torch.empty(block, dtype=torch.float64, device=dev)
    tp = torch.empty(block, dtype=torch.float64, device=dev)
    rc = _lib.load_library().dcsvd_labrd(h, m, n, _lib.ptr(A), _lib.ld(A), _lib.ptr(dd), _lib.ptr(ee),
                                         _lib.ptr(tq), _lib.ptr(tp), int(block), _lib.ptr(P), _lib.ld(P),
                                         _lib.ptr(Q), _lib.ld(Q), _lib.stream_ptr())
    _lib.check(rc, h)
    _writeback(a, A, was_np)
    for dst, src in ((d, dd), (e, ee), (tauq, tq), (taup, tp)):
        if isinstance(dst, torch.Tensor):
            dst[:block].copy_(src)
        else:
            dst[:block] = src.cpu().numpy()
    p = work.p[:m, : 2 * block]
    q = work.q[:n, : 2 * block]
    if isinstance(p, torch.Tensor):
        p.copy_(P)
        q.copy_(Q)
    else:
        p[...] = _lib.to_host(P)
        q[...] = _lib.to_host(Q)
    return p, q
