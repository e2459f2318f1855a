"""End-to-end GPU SVD with the reference driver API
(pkg/src/dcsvd/driver.py: ``PHASE_NAMES`` :31, ``SVDOptions`` :34-63,
``SVDResult`` :66-73, ``PhaseProfile`` :76-82, ``gesdd`` :147-157,
``phase_profile`` :160-170).

The dispatch (wide -> transpose, tall-skinny -> QR first, else square core)
runs inside the native driver (csrc/api.cu); this module only moves arrays
and maps options/status codes.  numpy in -> numpy out (the reference
contract); CUDA torch tensor in -> CUDA torch tensors out (device-resident
use, no host copies)."""

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

PHASE_NAMES = ("geqrf", "orgqr", "gebrd", "bdcdc", "ormqr+ormlq", "gemm")


@dataclass
class SVDOptions:
    """Tuning knobs (driver.py:34-63), validated like the reference.  Values
    above the GPU kernels' widths (bidiag 32, QR panel 64, CWY 128, leaf 32)
    run at those widths: the same factorization up to rounding."""

    want_vectors: bool = True
    bidiag_block: int = 32
    qr_block: int = 32
    orgqr_block: int = 64
    apply_block: int = 64
    leaf_size: int = 32
    ts_crossover: float = 5.0 / 3.0
    deflation_multiple: float = 8.0

    def __post_init__(self):
        for name in ("bidiag_block", "qr_block", "orgqr_block", "apply_block", "leaf_size"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be >= 1, got {getattr(self, name)}")
        if not self.ts_crossover >= 1.0:
            raise ValueError(f"ts_crossover must be >= 1, got {self.ts_crossover}")
        if not self.deflation_multiple > 0.0:
            raise ValueError(f"deflation_multiple must be > 0, got {self.deflation_multiple}")

    def _native(self):
        return _lib.DcsvdOpts(int(bool(self.want_vectors)), int(self.bidiag_block), int(self.qr_block),
                              int(self.orgqr_block), int(self.apply_block), int(self.leaf_size),
                              float(self.ts_crossover), float(self.deflation_multiple))


@dataclass
class SVDResult:
    """sigma descending; economy U (m x k), Vt (k x n), or None (values only)."""

    sigma: object
    u: object
    vt: object


@dataclass
class PhaseProfile:
    """Per-phase DEVICE seconds (CUDA events on the call's stream), one entry
    per PHASE_NAMES name, plus the device total."""

    phases: list
    total: float


def _run(a, options, prof):
    opts = options if options is not None else SVDOptions()
    if isinstance(a, torch.Tensor):
        if a.dim() != 2:
            raise ValueError(f"expected a 2-d array, got ndim={a.dim()}")
    else:
        a = np.asarray(a, dtype=np.float64)
        if a.ndim != 2:
            raise ValueError(f"expected a 2-d array, got ndim={a.ndim}")
    m, n = int(a.shape[0]), int(a.shape[1])
    if m < 1 or n < 1:
        raise ValueError(f"matrix must be nonempty, got {m}x{n}")
    h = _lib.handle()
    A, was_np = _lib.to_device_colmajor(a, copy=True)  # input never modified (driver.py:154)
    k = min(m, n)
    dev = A.device
    S = torch.empty(k, dtype=torch.float64, device=dev)
    U = VT = None
    if opts.want_vectors:
        U = _lib.colmajor_empty(m, k, dev.index)
        VT = _lib.colmajor_empty(k, n, dev.index)
    no = opts._native()
    pt = _lib.DcsvdPhaseTimes() if prof else None
    rc = _lib.load_library().dcsvd_gesdd(
        h, m, n, _lib.ptr(A), _lib.ld(A), _lib.ptr(S), _lib.ptr(U), _lib.ld(U) if U is not None else 1,
        _lib.ptr(VT), _lib.ld(VT) if VT is not None else 1, ctypes.byref(no),
        ctypes.byref(pt) if pt is not None else None, _lib.stream_ptr())
    _lib.check(rc, h)
    if was_np:
        res = SVDResult(S.cpu().numpy(), _lib.to_host(U), _lib.to_host(VT))
    else:
        res = SVDResult(S, U, VT)
    return res, pt


@_lib.on_input_device
def gesdd(a, options=None):
    """Economy SVD A = U diag(sigma) Vt on the GPU (driver.py:147-157).
    The input is not modified."""
    return _run(a, options, False)[0]


svd = gesdd


@_lib.on_input_device
def phase_profile(a, options=None):
    """gesdd with per-phase device time attribution (driver.py:160-170)."""
    _, pt = _run(a, options, True)
    phases = [("geqrf", pt.geqrf), ("orgqr", pt.orgqr), ("gebrd", pt.gebrd), ("bdcdc", pt.bdcdc),
              ("ormqr+ormlq", pt.ormbr), ("gemm", pt.gemm)]
    return PhaseProfile(phases, pt.total)


@_lib.on_input_device
def gesdd_batched(mats, options=None, concurrency=0):
    """Independent SVDs of a list of equally shaped matrices (BASELINE
    config 5).  Device tensors in -> device tensors out; numpy -> numpy."""
    if len(mats) == 0:
        return []
    opts = options if options is not None else SVDOptions()
    m, n = int(mats[0].shape[0]), int(mats[0].shape[1])
    for x in mats:
        if tuple(x.shape) != (m, n):
            raise ValueError("all matrices in a batch must share one shape")
    h = _lib.handle()
    k = min(m, n)
    devs, nps = [], []
    for x in mats:
        t, was_np = _lib.to_device_colmajor(x, copy=True)
        devs.append(t)
        nps.append(was_np)
    dev = devs[0].device
    Ss = [torch.empty(k, dtype=torch.float64, device=dev) for _ in mats]
    Us = [_lib.colmajor_empty(m, k, dev.index) for _ in mats] if opts.want_vectors else None
    VTs = [_lib.colmajor_empty(k, n, dev.index) for _ in mats] if opts.want_vectors else None
    P = ctypes.c_void_p * len(mats)
    a_p = P(*[t.data_ptr() for t in devs])
    s_p = P(*[t.data_ptr() for t in Ss])
    u_p = P(*[t.data_ptr() for t in Us]) if Us else None
    v_p = P(*[t.data_ptr() for t in VTs]) if VTs else None
    no = opts._native()
    rc = _lib.load_library().dcsvd_gesdd_batched(
        h, len(mats), m, n, a_p, m, s_p, u_p, m, v_p, k, ctypes.byref(no), int(concurrency), _lib.stream_ptr())
    _lib.check(rc, h)
    out = []
    for i, was_np in enumerate(nps):
        u = Us[i] if Us else None
        vt = VTs[i] if VTs else None
        if was_np:
            out.append(SVDResult(Ss[i].cpu().numpy(), _lib.to_host(u), _lib.to_host(vt)))
        else:
            out.append(SVDResult(Ss[i], u, vt))
    return out
