"""Dense-kernel entry points on the GPU: GEMM / GEMV with the reference
semantics of pkg/src/dcsvd/densecore.py:73-111 (``matmul_accumulate``,
``matvec_accumulate``), plus the shared array plumbing used by the other
modules.  Arrays may be numpy (copied to the device and back, written in
place like the reference) or CUDA torch tensors (computed in place)."""

import numpy as np
import torch

from . import _lib


def _op_shape(shape, trans):
    return (shape[1], shape[0]) if trans else tuple(shape)


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
