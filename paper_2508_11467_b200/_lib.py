"""ctypes binding of libdcsvd_b200.so (C ABI in include/dcsvd_b200.h).

This is the only place Python touches the native library.  There is no
fallback: if the shared library or a CUDA device is missing, every entry
point raises.  PyTorch provides device memory and the current stream.
"""

import ctypes
import functools
import os
import threading

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdcsvd_b200.so")

# status codes (include/dcsvd_b200.h)
OK, EINVAL, ENOCONV, EARITH, ESINGULAR, ECUDA = range(6)

EXPORTED = (
    "dcsvd_create", "dcsvd_destroy", "dcsvd_last_error", "dcsvd_version", "dcsvd_launch_count",
    "dcsvd_dgemm", "dcsvd_dgemv", "dcsvd_gebrd", "dcsvd_labrd", "dcsvd_bdsdc", "dcsvd_geqrf",
    "dcsvd_orgqr", "dcsvd_ormbr", "dcsvd_gesdd", "dcsvd_gesdd_batched", "dcsvd_set_stats", "dcsvd_get_stats",
    "dcsvd_larfg", "dcsvd_lartg", "dcsvd_trsm", "dcsvd_build_tinv", "dcsvd_block_reflector", "dcsvd_geqrf_panel",
    "dcsvd_secular_roots", "dcsvd_recompute_z", "dcsvd_secular_vectors",
    "dcsvd_build_z", "dcsvd_deflate", "dcsvd_gather",
    "dcsvd_philox", "dcsvd_prescribed_singular_values", "dcsvd_generate_matrix", "dcsvd_accuracy",
)


class ConvergenceError(RuntimeError):
    """An iterative kernel exceeded its iteration budget
    (pkg/src/dcsvd/densecore.py:29-30)."""


class DcsvdOpts(ctypes.Structure):
    _fields_ = [
        ("want_vectors", ctypes.c_int),
        ("bidiag_block", ctypes.c_int),
        ("qr_block", ctypes.c_int),
        ("orgqr_block", ctypes.c_int),
        ("apply_block", ctypes.c_int),
        ("leaf_size", ctypes.c_int),
        ("ts_crossover", ctypes.c_double),
        ("deflation_multiple", ctypes.c_double),
    ]


class DcsvdPhaseTimes(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("geqrf", "orgqr", "gebrd", "bdcdc", "ormbr", "gemm", "total")]


_lib = None
_lib_lock = threading.Lock()


def load_library(path=None):
    """Load (once) and prototype the native library.  Raises if absent."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise RuntimeError(
                f"libdcsvd_b200.so not found at {p}; build it with "
                "`python -m paper_2508_11467_b200.build` (no CPU fallback exists)"
            )
        lib = ctypes.CDLL(p)
        V, I, I64, D, C = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_char
        U64 = ctypes.c_uint64
        proto = {
            "dcsvd_create": (I, [ctypes.POINTER(V), I]),
            "dcsvd_destroy": (I, [V]),
            "dcsvd_last_error": (ctypes.c_char_p, [V]),
            "dcsvd_version": (I, []),
            "dcsvd_launch_count": (ctypes.c_longlong, [V]),
            "dcsvd_set_stats": (I, [V, I]),
            "dcsvd_get_stats": (I, [V, I, ctypes.POINTER(D), ctypes.POINTER(D), ctypes.POINTER(ctypes.c_longlong)]),
            "dcsvd_dgemm": (I, [V, I, I, I64, I64, I64, D, V, I64, V, I64, D, V, I64, V]),
            "dcsvd_dgemv": (I, [V, I, I64, I64, D, V, I64, V, D, V, V]),
            "dcsvd_gebrd": (I, [V, I64, I64, V, I64, V, V, V, V, I, V]),
            "dcsvd_labrd": (I, [V, I64, I64, V, I64, V, V, V, V, I, V, I64, V, I64, V]),
            "dcsvd_bdsdc": (I, [V, I64, V, V, I, I, I, D, V, V, I64, V, I64, V, V]),
            "dcsvd_geqrf": (I, [V, I64, I64, V, I64, V, I, V]),
            "dcsvd_orgqr": (I, [V, I64, I64, I64, V, I64, V, V, I64, I, V]),
            "dcsvd_ormbr": (I, [V, C, I, I64, I64, V, I64, V, V, I64, I64, I64, I, V]),
            "dcsvd_gesdd": (I, [V, I64, I64, V, I64, V, V, I64, V, I64, ctypes.POINTER(DcsvdOpts),
                                ctypes.POINTER(DcsvdPhaseTimes), V]),
            "dcsvd_larfg": (I, [V, I64, V, V, I64, V, V, V]),
            "dcsvd_lartg": (I, [V, I64, V, V, V, V]),
            "dcsvd_trsm": (I, [V, C, I, I64, V, I64, V, I64, I64, V]),
            "dcsvd_build_tinv": (I, [V, I64, I, V, I64, V, V, I64, V]),
            "dcsvd_block_reflector": (I, [V, C, I, I64, I, V, I64, V, I64, V, I64, I64, V]),
            "dcsvd_geqrf_panel": (I, [V, I64, I, V, I64, V, V]),
            "dcsvd_secular_roots": (I, [V, I, V, V, V, V, V, I, V]),
            "dcsvd_recompute_z": (I, [V, I, V, V, V, V, V, V]),
            "dcsvd_secular_vectors": (I, [V, I, V, V, V, V, V, I64, V, I64, V]),
            "dcsvd_build_z": (I, [V, I, I, I, D, D, V, V, I64, V, V, I64, V, V, V, V]),
            "dcsvd_deflate": (I, [V, I, V, V, D, V, I64, I64, V, I64, I64, V, I64, V, V, V, V, V, V, V, V, V, V,
                                  V, V]),
            "dcsvd_gather": (I, [V, I64, I64, V, I64, V, V, V, I64, V]),
            "dcsvd_philox": (I, [V, U64, U64, U64, I64, I, V, I64, I64, V]),
            "dcsvd_prescribed_singular_values": (I, [V, I, I64, D, U64, U64, V, V]),
            "dcsvd_generate_matrix": (I, [V, I, I64, I64, D, U64, U64, V, I64, V]),
            "dcsvd_accuracy": (I, [V, I64, I64, V, I64, V, V, I64, V, I64, V, ctypes.POINTER(D), V]),
            "dcsvd_gesdd_batched": (I, [V, I, I64, I64, ctypes.POINTER(V), I64, ctypes.POINTER(V),
                                        ctypes.POINTER(V), I64, ctypes.POINTER(V), I64,
                                        ctypes.POINTER(DcsvdOpts), I, V]),
        }
        for name, (res, args) in proto.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
        return lib


_handles = {}
_handles_lock = threading.Lock()


def handle(device=None):
    """Per-(thread, device) library handle."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2508_11467_b200 requires a CUDA device (B200); no CPU fallback exists")
    lib = load_library()
    dev = torch.cuda.current_device() if device is None else int(device)
    key = (threading.get_ident(), dev)
    with _handles_lock:
        h = _handles.get(key)
        if h is None:
            hv = ctypes.c_void_p()
            rc = lib.dcsvd_create(ctypes.byref(hv), dev)
            if rc != 0:
                raise RuntimeError(f"dcsvd_create failed on device {dev} (status {rc})")
            h = hv
            _handles[key] = h
    return h


def check(rc, h):
    if rc == OK:
        return
    msg = load_library().dcsvd_last_error(h).decode(errors="replace")
    if rc == EINVAL:
        raise ValueError(msg)
    if rc == ENOCONV:
        raise ConvergenceError(msg)
    if rc == EARITH:
        raise ArithmeticError(msg)
    if rc == ESINGULAR:
        raise np.linalg.LinAlgError(msg)
    raise RuntimeError(msg)


def _cuda_devices(obj, out, depth=0):
    if isinstance(obj, torch.Tensor):
        if obj.is_cuda:
            out.add(obj.device.index)
    elif depth < 2 and isinstance(obj, (list, tuple)):
        for x in obj:
            _cuda_devices(x, out, depth + 1)
    elif depth < 2 and isinstance(obj, dict):
        for x in obj.values():
            _cuda_devices(x, out, depth + 1)
    elif depth < 1 and hasattr(obj, "__dict__") and not isinstance(obj, type):
        for x in vars(obj).values():  # dataclass containers (problems, reflector sequences, results)
            _cuda_devices(x, out, depth + 1)


def on_input_device(fn):
    """Run a public entry point on the device its CUDA tensor arguments live
    on (handle, stream and outputs all follow ``torch.cuda.current_device``);
    numpy-only calls use the current device.  Mixed devices are rejected."""

    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        devs = set()
        for x in list(args) + list(kwargs.values()):
            _cuda_devices(x, devs)
        if len(devs) > 1:
            raise ValueError(f"arguments live on different CUDA devices {sorted(devs)}")
        if not devs or not torch.cuda.is_available():
            return fn(*args, **kwargs)
        with torch.cuda.device(devs.pop()):
            return fn(*args, **kwargs)

    return wrapper


def stream_ptr():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def launch_count():
    return int(load_library().dcsvd_launch_count(None))


# ---------------------------------------------------------------------------
# array plumbing: column-major fp64 device tensors


def colmajor_empty(m, n, device=None):
    """m x n float64 CUDA tensor with column-major strides (1, m)."""
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    return torch.empty((n, m), dtype=torch.float64, device=dev).t()


def is_colmajor(t):
    return t.dim() == 2 and t.stride(0) == 1 and (t.shape[1] <= 1 or t.stride(1) >= max(t.shape[0], 1))


def to_device_colmajor(x, copy=True):
    """Return (tensor, was_numpy).  numpy input is copied to the current CUDA
    device; torch input keeps its memory unless it must be re-laid-out (or
    ``copy``)."""
    if isinstance(x, torch.Tensor):
        if x.dim() != 2:
            raise ValueError(f"expected a 2-d array, got ndim={x.dim()}")
        t = x
        if not t.is_cuda:
            t = t.to("cuda")
        if t.dtype != torch.float64:
            t = t.to(torch.float64)
        if copy or not is_colmajor(t):
            c = colmajor_empty(t.shape[0], t.shape[1], t.device.index)
            c.copy_(t)
            t = c
        return t, False
    a = np.asarray(x, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError(f"expected a 2-d array, got ndim={a.ndim}")
    m, n = a.shape
    t = colmajor_empty(m, n)
    # a.T as C-contiguous == a in Fortran order; copy through a pinned staging tensor
    arr = np.ascontiguousarray(a.T)
    if not arr.flags.writeable:  # e.g. read_matrix's frombuffer views
        arr = arr.copy()
    host = torch.from_numpy(arr)
    t.t().copy_(host, non_blocking=False)
    return t, True


def vec_to_device(v, n=None):
    if isinstance(v, torch.Tensor):
        t = v.to(device="cuda", dtype=torch.float64).contiguous()
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(v, dtype=np.float64))).to("cuda")
    if n is not None and t.numel() != n:
        raise ValueError(f"expected {n} entries, got {t.numel()}")
    return t


def to_host(t):
    """Device tensor -> numpy (Fortran order for matrices)."""
    if t is None:
        return None
    if t.dim() == 2:
        return np.asfortranarray(t.t().contiguous().cpu().numpy().T)
    return t.cpu().numpy()


def ptr(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def ld(t):
    """Leading dimension of a column-major 2-d tensor."""
    return max(int(t.stride(1)), max(int(t.shape[0]), 1)) if t.shape[1] > 1 else max(int(t.shape[0]), 1)


def set_stats(enable, device=None):
    h = handle(device)
    check(load_library().dcsvd_set_stats(h, int(bool(enable))), h)


def get_stats(kind, device=None):
    """(milliseconds, work, launches) accumulated for a kernel family."""
    h = handle(device)
    ms, work, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_longlong()
    check(load_library().dcsvd_get_stats(h, int(kind), ctypes.byref(ms), ctypes.byref(work), ctypes.byref(n)), h)
    return ms.value, work.value, n.value
