"""Runs the ORMBR-shaped GEMMs once each (for ncu captures; dev tool).
  rank-128 update  C(8192x8192) -= Y(8192x128) X(128x8192)
  split-K          Z(128x8192)   = Y^T(128x8192) C(8192x8192)
  trailing rank-64 C(8160x8160) -= P(8160x64) Q(8160x64)^T"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2508_11467_b200 import _lib
lib = _lib.load_library(); h = _lib.handle(); st = _lib.stream_ptr()
def col(r, c):
    return torch.randn(c, r, dtype=torch.float64, device="cuda").t()
n = 8192
C = col(n, n); Y = col(n, 128); X = col(128, n); Z = col(128, n)
P = col(8160, 64); Q = col(8160, 64); C2 = col(8160, 8160)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
if len(sys.argv) > 2:
    lib.dcsvd_debug_gemm_route(int(sys.argv[2]))
    print('route', sys.argv[2])
for _ in range(reps):
    lib.dcsvd_dgemm(h, 0, 0, n, n, 128, -1.0, _lib.ptr(Y), n, _lib.ptr(X), 128, 1.0, _lib.ptr(C), n, st)
    lib.dcsvd_dgemm(h, 1, 0, 128, n, n, 1.0, _lib.ptr(Y), n, _lib.ptr(C), n, 0.0, _lib.ptr(Z), 128, st)
    lib.dcsvd_dgemm(h, 0, 1, 8160, 8160, 64, -1.0, _lib.ptr(P), 8160, _lib.ptr(Q), 8160, 1.0, _lib.ptr(C2), 8160, st)
torch.cuda.synchronize()
if reps > 1:
    import time
    for name, f, fl in [("rank128", lambda: lib.dcsvd_dgemm(h, 0, 0, n, n, 128, -1.0, _lib.ptr(Y), n, _lib.ptr(X), 128, 1.0, _lib.ptr(C), n, st), 2*n*n*128),
                        ("splitk", lambda: lib.dcsvd_dgemm(h, 1, 0, 128, n, n, 1.0, _lib.ptr(Y), n, _lib.ptr(C), n, 0.0, _lib.ptr(Z), 128, st), 2*n*n*128),
                        ("rank64", lambda: lib.dcsvd_dgemm(h, 0, 1, 8160, 8160, 64, -1.0, _lib.ptr(P), 8160, _lib.ptr(Q), 8160, 1.0, _lib.ptr(C2), 8160, st), 2*8160*8160*64)]:
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f(); torch.cuda.synchronize(); s.record()
        for _ in range(10): f()
        e.record(); torch.cuda.synchronize()
        t = s.elapsed_time(e) / 10 * 1e-3
        print(f"{name}: {t*1e3:.3f} ms  {fl/t/1e12:.1f} TF/s")
