"""One rank-64 streaming update at 8160^2 (the first GEBRD trailing update of C2), for ncu."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2508_11467_b200 import _lib
lib = _lib.load_library(); h = _lib.handle(); st = _lib.stream_ptr()
m = n = int(sys.argv[1]) if len(sys.argv) > 1 else 8160
k = 64
A = torch.randn(k, m, dtype=torch.float64, device="cuda").t()
B = torch.randn(k, n, dtype=torch.float64, device="cuda").t()
C = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
for _ in range(3):
    lib.dcsvd_dgemm(h, 0, 1, m, n, k, -1.0, _lib.ptr(A), A.stride(1), _lib.ptr(B), B.stride(1), 1.0, _lib.ptr(C), C.stride(1), st)
torch.cuda.synchronize()
