"""Probe the TMA gather GEMM (gemm_launch_device_stack) on single host-built
descriptors over a 6-buffer ld x ld stack: which (row, col, k) combinations
work; compares with torch."""
import sys, os, ctypes, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2508_11467_b200 import _lib
lib = _lib.load_library(); h = _lib.handle(); st = _lib.stream_ptr(); lib.dcsvd_debug_ws_flags(8)
class GD(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int), ("n", ctypes.c_int), ("k", ctypes.c_int), ("A", ctypes.c_void_p), ("lda", ctypes.c_longlong),
                ("acol", ctypes.c_void_p), ("B", ctypes.c_void_p), ("ldb", ctypes.c_longlong), ("C", ctypes.c_void_p),
                ("ldc", ctypes.c_longlong), ("ccol", ctypes.c_void_p), ("alpha", ctypes.c_double), ("beta", ctypes.c_double)]
ld = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
V = ctypes.c_void_p
lib.dcsvd_debug_gemm_stack.argtypes = [V, V, ctypes.c_int, ctypes.c_int, ctypes.c_int, V, ctypes.c_int64, ctypes.c_int, V]
stack = torch.randn(6 * ld, ld, dtype=torch.float64, device="cuda")  # row-major (6ld, ld) = col-major ld x 6ld
base = stack.data_ptr()
def col(c): return base + 8 * ld * c
acol = torch.randperm(ld, device="cuda", dtype=torch.int64).to(torch.int32)
ccol = torch.arange(ld, device="cuda", dtype=torch.int32)
S = stack.t()  # ld x 6ld column-major view
cases = [(0, 0, 2000, 29, 59, 28), (61, 1000, 3061, 31, 62, 31), (92, 1000, 3061, 32, 62, 32), (186, 1000, 3186, 31, 62, 31),
         (61, 0, 2061, 31, 62, 31), (0, 0, 2000, 128, 64, 32), (0, 1000, 3000, 128, 64, 32), (1, 0, 2000, 128, 64, 33)]
for (row, cA, cB, m, n, k) in cases:
    for rb in (row, 0):
        g = GD(m, n, k, base + 8 * (row + ld * cA), ld, acol.data_ptr(), base + 8 * (rb + ld * cB), ld,
               col(4 * ld) + 8 * row, ld, ccol.data_ptr(), 1.0, 0.0)
        S[:, 4 * ld:5 * ld] = 0
        rc = lib.dcsvd_debug_gemm_stack(h, ctypes.byref(g), 1, m, n, ctypes.c_void_p(base), ld, 6, st)
        msg = lib.dcsvd_last_error(h).decode() if rc else ""
        ok = None
        if rc == 0:
            Ag = S[row:row + m, cA + acol[:k].long()]
            Bb = S[rb:rb + k, cB:cB + n]
            ref = Ag @ Bb
            ok = float((S[row:row + m, 4 * ld:4 * ld + n] - ref).abs().max())
        print(json.dumps(dict(row=row, rb=rb, cA=cA, cB=cB, m=m, n=n, k=k, rc=rc, err=ok, msg=msg[:60])), flush=True)
        if rc:
            sys.exit(0)
