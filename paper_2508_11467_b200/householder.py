"""GPU Householder QR and back-transformations with the reference API of
pkg/src/dcsvd/qrblock.py (``geqrf_blocked`` :122, ``orgqr`` :147,
``QRFactorization`` :30) and pkg/src/dcsvd/backtransform.py
(``ReflectorSequence`` :30, ``column_reflectors`` :47, ``row_reflectors``
:54, ``ormqr_like`` :90, ``ormlq_like`` :112).  Inverse-T compact-WY blocks
applied as DMMA GEMMs (csrc/qr.cu)."""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


@dataclass
class QRFactorization:
    """Packed blocked QR: R in the upper triangle, essentials below, tau."""

    packed: object
    tau: object

    @property
    def shape(self):
        return tuple(self.packed.shape)


@dataclass
class ReflectorSequence:
    """Packed Householder product and its geometry (backtransform.py:30-44)."""

    packed: object
    tau: object
    side: str
    offset: int
    count: int


def column_reflectors(fact):
    """U1 = H_1...H_n of a bidiagonalization (backtransform.py:47-51)."""
    return ReflectorSequence(fact.packed, fact.tauq, "left", 0, fact.packed.shape[1])


def row_reflectors(fact):
    """V1 = G_1...G_{n-1} of a bidiagonalization (backtransform.py:54-57)."""
    n = fact.packed.shape[1]
    return ReflectorSequence(fact.packed, fact.taup, "right", 1, max(n - 1, 0))


def _writeback(orig, dev, was_np):
    if was_np:
        orig[...] = _lib.to_host(dev)
        return orig
    if isinstance(orig, torch.Tensor) and dev.data_ptr() != orig.data_ptr():
        orig.copy_(dev)
        return orig
    return dev


@_lib.on_input_device
def geqrf_blocked(a, block=32):
    """Blocked Householder QR in place (qrblock.py:122-144): cooperative
    shared-memory panel kernel + CWY trailing update."""
    m, n = tuple(a.shape)
    if n < 1:
        raise ValueError("matrix must have at least one column")
    if m < n:
        raise ValueError(f"QR factorization requires m >= n, got {m}x{n}")
    if block < 1:
        raise ValueError(f"block width must be >= 1, got {block}")
    h = _lib.handle()
    A, was_np = _lib.to_device_colmajor(a, copy=False)
    tau = torch.empty(n, dtype=torch.float64, device=A.device)
    rc = _lib.load_library().dcsvd_geqrf(h, m, n, _lib.ptr(A), _lib.ld(A), _lib.ptr(tau), int(block),
                                         _lib.stream_ptr())
    _lib.check(rc, h)
    packed = _writeback(a, A, was_np)
    return QRFactorization(packed, tau.cpu().numpy() if was_np else tau)


@_lib.on_input_device
def orgqr(fact, k, block=64):
    """First k columns of Q = H_1...H_n (qrblock.py:147-164)."""
    m, n = fact.shape
    if not 1 <= k <= m:
        raise ValueError(f"need 1 <= k <= {m} columns of Q, got {k}")
    h = _lib.handle()
    A, was_np = _lib.to_device_colmajor(fact.packed, copy=False)
    tau = _lib.vec_to_device(fact.tau, n)
    Q = _lib.colmajor_empty(m, k)
    rc = _lib.load_library().dcsvd_orgqr(h, m, n, k, _lib.ptr(A), _lib.ld(A), _lib.ptr(tau), _lib.ptr(Q),
                                         _lib.ld(Q), int(block), _lib.stream_ptr())
    _lib.check(rc, h)
    return _lib.to_host(Q) if was_np else Q


def _apply(seq, c, vect, transpose, block):
    m, n = seq.packed.shape
    if vect == "Q":
        n = int(seq.count)  # the first `count` column reflectors (columns beyond are not read)
    h = _lib.handle()
    A, _ = _lib.to_device_colmajor(seq.packed, copy=False)
    tau = _lib.vec_to_device(seq.tau)[:n].contiguous()
    C, c_np = _lib.to_device_colmajor(c, copy=False)
    rc = _lib.load_library().dcsvd_ormbr(h, vect.encode(), int(bool(transpose)), m, n, _lib.ptr(A), _lib.ld(A),
                                         _lib.ptr(tau), _lib.ptr(C), C.shape[0], C.shape[1], _lib.ld(C),
                                         int(block), _lib.stream_ptr())
    _lib.check(rc, h)
    return _writeback(c, C, c_np)


@_lib.on_input_device
def ormqr_like(seq, c, transpose=False, block=64):
    """C <- U1 C (or U1^T C) with the left (column) reflectors
    (backtransform.py:90-109)."""
    if seq.side != "left":
        raise ValueError(f"expected a left-side sequence, got {seq.side!r}")
    if c.shape[0] != seq.packed.shape[0]:
        raise ValueError(f"C has {c.shape[0]} rows, sequence acts on {seq.packed.shape[0]}")
    if seq.offset != 0 or not 0 <= seq.count <= min(seq.packed.shape):
        raise ValueError("column reflectors need offset 0 and 0 <= count <= min(packed.shape)")
    if seq.count == 0:
        return c
    return _apply(seq, c, "Q", transpose, block)


@_lib.on_input_device
def ormlq_like(seq, c, transpose=False, block=64):
    """C <- C V1 (or C V1^T) with the right (row) reflectors
    (backtransform.py:112-131)."""
    if seq.side != "right":
        raise ValueError(f"expected a right-side sequence, got {seq.side!r}")
    if c.shape[1] != seq.packed.shape[1]:
        raise ValueError(f"C has {c.shape[1]} columns, sequence acts on {seq.packed.shape[1]}")
    if seq.count != max(seq.packed.shape[1] - 1, 0) or seq.offset != 1:
        raise ValueError("GPU ormlq_like supports the full row-reflector sequence of a bidiagonalization")
    return _apply(seq, c, "P", transpose, block)


@dataclass
class CompactWYBlock:
    """One reflector block (Y, Tinv), H_1...H_b = I - Y Tinv^-1 Y^T (qrblock.py:43-48)."""

    y: object
    tinv: object


@_lib.on_input_device
def build_tinv(y, tau):
    """Tinv = strict-upper(Y^T Y) + diag(1/tau) (1 for tau == 0)
    (qrblock.py:90-100): one DMMA GEMM + one kernel."""
    rows, b = tuple(y.shape)
    h = _lib.handle()
    Y, was_np = _lib.to_device_colmajor(y, copy=False)
    t = _lib.vec_to_device(tau, b)
    out = _lib.colmajor_empty(b, b)
    rc = _lib.load_library().dcsvd_build_tinv(h, rows, b, _lib.ptr(Y), _lib.ld(Y), _lib.ptr(t), _lib.ptr(out),
                                              _lib.ld(out), _lib.stream_ptr())
    _lib.check(rc, h)
    return _lib.to_host(out) if was_np else out


def _apply_block(block, c, transpose, side):
    rows_y, b = tuple(block.y.shape)
    h = _lib.handle()
    Y, _ = _lib.to_device_colmajor(block.y, copy=False)
    T, _ = _lib.to_device_colmajor(block.tinv, copy=False)
    C, c_np = _lib.to_device_colmajor(c, copy=False)
    other = C.shape[1] if side == "L" else C.shape[0]
    rc = _lib.load_library().dcsvd_block_reflector(h, side.encode(), int(bool(transpose)), rows_y, b, _lib.ptr(Y),
                                                   _lib.ld(Y), _lib.ptr(T), _lib.ld(T), _lib.ptr(C), _lib.ld(C), other,
                                                   _lib.stream_ptr())
    _lib.check(rc, h)
    return _writeback(c, C, c_np)


@_lib.on_input_device
def apply_block_reflector_left(block, c, transpose=False):
    """C <- (I - Y T Y^T) C, or the transposed block (qrblock.py:103-111)."""
    if c.shape[0] != block.y.shape[0]:
        raise ValueError(f"C has {c.shape[0]} rows, block acts on {block.y.shape[0]}")
    return _apply_block(block, c, transpose, "L")


@_lib.on_input_device
def apply_block_reflector_right(block, c, transpose=False):
    """C <- C (I - Y T Y^T), or the transposed block (qrblock.py:114-119)."""
    if c.shape[1] != block.y.shape[0]:
        raise ValueError(f"C has {c.shape[1]} columns, block acts on {block.y.shape[0]}")
    return _apply_block(block, c, transpose, "R")


@_lib.on_input_device
def geqrf_panel(a, tau):
    """Unblocked Householder QR of a tall panel in place (qrblock.py:51-71);
    cooperative kernel with the panel's row slabs in shared memory."""
    m, n = tuple(a.shape)
    if m < n:
        raise ValueError(f"panel must be tall, got {m}x{n}")
    h = _lib.handle()
    A, was_np = _lib.to_device_colmajor(a, copy=False)
    t = torch.empty(max(n, 1), dtype=torch.float64, device=A.device)
    rc = _lib.load_library().dcsvd_geqrf_panel(h, m, n, _lib.ptr(A), _lib.ld(A), _lib.ptr(t), _lib.stream_ptr())
    _lib.check(rc, h)
    _writeback(a, A, was_np)
    if isinstance(tau, torch.Tensor):
        tau[:n].copy_(t[:n])
    else:
        tau[:n] = t[:n].cpu().numpy()
    return a
