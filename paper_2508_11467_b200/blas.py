"""Dense-kernel entry points on the GPU: GEMM / GEMV with the reference
semantics of pkg/src/dcsvd/densecore.py:73-111 (``matmul_accumulate``,
``matvec_accumulate``), plus the shared array plumbing used by the other
modules.  Arrays may be numpy (copied to the device and back, written in
place like the reference) or CUDA torch tensors (computed in place)."""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


@dataclass
class HouseholderReflector:
    """H = I - tau y y^T, y = (1, essential) (densecore.py:33-43)."""

    tau: float
    essential: object
    pivot_value: float


@dataclass
class GivensRotation:
    """[[c, s], [-s, c]] (densecore.py:46-51)."""

    c: float
    s: float


@_lib.on_input_device
def householder_generate(alpha, x):
    """Reflector mapping (alpha, x) onto (pivot, 0...), no safmin rescaling
    (densecore.py:114-128); one GPU kernel (norm, scalars, essential)."""
    torch_in = isinstance(x, torch.Tensor)
    xv = _lib.vec_to_device(x).reshape(-1)
    h = _lib.handle()
    al = torch.tensor([float(alpha)], dtype=torch.float64, device=xv.device)
    out = torch.empty(2, dtype=torch.float64, device=xv.device)
    ess = torch.empty(max(xv.numel(), 1), dtype=torch.float64, device=xv.device)
    rc = _lib.load_library().dcsvd_larfg(h, xv.numel(), _lib.ptr(al), _lib.ptr(xv), 1, _lib.ptr(out), _lib.ptr(ess),
                                         _lib.stream_ptr())
    _lib.check(rc, h)
    tau, beta = (float(v) for v in out.cpu())
    ess = ess[: xv.numel()]
    return HouseholderReflector(tau, ess if torch_in else ess.cpu().numpy(), beta)


@_lib.on_input_device
def givens_generate(a, b):
    """(GivensRotation, r) with c a + s b = r >= 0 (densecore.py:131-140)."""
    h = _lib.handle()
    ab = torch.tensor([float(a), float(b)], dtype=torch.float64, device="cuda")
    out = torch.empty(3, dtype=torch.float64, device="cuda")
    rc = _lib.load_library().dcsvd_lartg(h, 1, _lib.ptr(ab), ctypes_offset(ab, 1), _lib.ptr(out), _lib.stream_ptr())
    _lib.check(rc, h)
    c, s, r = (float(v) for v in out.cpu())
    return GivensRotation(c, s), r


def ctypes_offset(t, elems):
    import ctypes

    return ctypes.c_void_p(t.data_ptr() + 8 * elems)


@_lib.on_input_device
def triangular_solve(t, b, side="left", trans=False):
    """Solve against an upper-triangular T in place on ``b``
    (densecore.py:143-171): left B <- T^-1 B (T^-T B), right B <- B T^-1 (B T^-T).
    Raises LinAlgError on a zero diagonal."""
    if t.shape[0] != t.shape[1]:
        raise ValueError(f"triangular factor must be square, got {tuple(t.shape)}")
    n = t.shape[0]
    if side == "left":
        if b.shape[0] != n:
            raise ValueError(f"shape mismatch: T is {tuple(t.shape)}, B has {b.shape[0]} rows")
        other = b.shape[1]
    elif side == "right":
        if b.shape[1] != n:
            raise ValueError(f"shape mismatch: T is {tuple(t.shape)}, B has {b.shape[1]} columns")
        other = b.shape[0]
    else:
        raise ValueError(f"side must be 'left' or 'right', got {side!r}")
    h = _lib.handle()
    T, _ = _lib.to_device_colmajor(t, copy=False)
    B, b_np = _lib.to_device_colmajor(b, copy=False)
    rc = _lib.load_library().dcsvd_trsm(h, b"L" if side == "left" else b"R", int(bool(trans)), n, _lib.ptr(T), _lib.ld(T),
                                        _lib.ptr(B), _lib.ld(B), other, _lib.stream_ptr())
    _lib.check(rc, h)
    if b_np:
        b[...] = _lib.to_host(B)
    elif B.data_ptr() != b.data_ptr():
        b.copy_(B)
    return b


def _op_shape(shape, trans):
    return (shape[1], shape[0]) if trans else tuple(shape)


@_lib.on_input_device
def matmul_accumulate(alpha, a, trans_a, b, trans_b, beta, c):
    """C <- beta*C + alpha*op(A) op(B), in place into ``c`` (densecore.py:73-93);
    beta == 0 overwrites C without reading it.  DMMA kernel."""
    ma, ka = _op_shape(a.shape, trans_a)
    kb, nb = _op_shape(b.shape, trans_b)
    if ka != kb or tuple(c.shape) != (ma, nb):
        raise ValueError(
            f"matmul_accumulate shape mismatch: op(A)={ma}x{ka}, op(B)={kb}x{nb}, C={c.shape[0]}x{c.shape[1]}"
        )
    h = _lib.handle()
    A, _ = _lib.to_device_colmajor(a, copy=False)
    B, _ = _lib.to_device_colmajor(b, copy=False)
    C, c_np = _lib.to_device_colmajor(c, copy=False)
    inplace_torch = isinstance(c, torch.Tensor) and C.data_ptr() == c.data_ptr()
    rc = _lib.load_library().dcsvd_dgemm(
        h, int(bool(trans_a)), int(bool(trans_b)), ma, nb, ka, float(alpha), _lib.ptr(A), _lib.ld(A),
        _lib.ptr(B), _lib.ld(B), float(beta), _lib.ptr(C), _lib.ld(C), _lib.stream_ptr())
    _lib.check(rc, h)
    if c_np:
        c[...] = _lib.to_host(C)
    elif not inplace_torch:
        c.copy_(C)
    return c


@_lib.on_input_device
def matvec_accumulate(alpha, a, trans_a, x, beta, y):
    """y <- beta*y + alpha*op(A) x, in place (densecore.py:96-111)."""
    ma, ka = _op_shape(a.shape, trans_a)
    if tuple(x.shape) != (ka,) or tuple(y.shape) != (ma,):
        raise ValueError(f"matvec_accumulate shape mismatch: op(A)={ma}x{ka}, x={tuple(x.shape)}, y={tuple(y.shape)}")
    h = _lib.handle()
    A, _ = _lib.to_device_colmajor(a, copy=False)
    X = _lib.vec_to_device(x)
    Y = _lib.vec_to_device(y)
    rc = _lib.load_library().dcsvd_dgemv(h, int(bool(trans_a)), A.shape[0], A.shape[1], float(alpha), _lib.ptr(A),
                                         _lib.ld(A), _lib.ptr(X), float(beta), _lib.ptr(Y), _lib.stream_ptr())
    _lib.check(rc, h)
    if isinstance(y, torch.Tensor):
        if Y.data_ptr() != y.data_ptr():
            y.copy_(Y)
    else:
        y[...] = Y.cpu().numpy()
    return y


def dense_matrix(m, n):
    """Zero m x n column-major float64 matrix (densecore.py:54-58)."""
    if m < 0 or n < 0:
        raise ValueError(f"matrix dimensions must be nonnegative, got {m}x{n}")
    return np.zeros((m, n), dtype=np.float64, order="F")


def as_dense(a):
    """Column-major float64 copy (densecore.py:61-66)."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError(f"expected a 2-d array, got ndim={a.ndim}")
    return np.asfortranarray(a).copy(order="F")
