"""DMMA GEMM microbenchmark vs cuBLAS (measuring stick only)."""
import sys, os, json, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2508_11467_b200 import _lib
lib = _lib.load_library(); h = _lib.handle(); st = _lib.stream_ptr()
def t(fn, it=5):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / it * 1e-3
res = []
for (m, n, k, ta, tb) in [(4096, 8192, 128, 0, 0), (128, 8192, 4096, 1, 0), (128, 8192, 128, 0, 0), (8192, 8192, 8192, 0, 0), (8160, 8160, 64, 0, 1), (64, 8192, 8192, 1, 0), (8192, 8192, 64, 0, 0), (4096, 6900, 3450, 0, 0), (65536, 1024, 1024, 0, 0), (8192, 64, 8192, 0, 0)]:
    A = torch.randn(k if ta else m, m if ta else k, dtype=torch.float64, device="cuda").t().contiguous().t()
    B = torch.randn(n if tb else k, k if tb else n, dtype=torch.float64, device="cuda").t().contiguous().t()
    C = torch.randn(m, n, dtype=torch.float64, device="cuda").t().contiguous().t()
    f = lambda: lib.dcsvd_dgemm(h, ta, tb, m, n, k, 1.0, _lib.ptr(A), A.stride(1), _lib.ptr(B), B.stride(1), 1.0, _lib.ptr(C), C.stride(1), st)
    tt = t(f)
    Aop = A.t() if ta else A; Bop = B.t() if tb else B
    tc = t(lambda: torch.addmm(C, Aop, Bop, out=C))
    r = dict(m=m, n=n, k=k, ta=ta, tb=tb, ours_tflops=2*m*n*k/tt/1e12, cublas_tflops=2*m*n*k/tc/1e12)
    print(json.dumps(r), flush=True); res.append(r)
