"""One DMMA GEMM call (for ncu): python tools/gemm_one.py m n k ta tb [reps]."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2508_11467_b200 import _lib
lib = _lib.load_library(); h = _lib.handle(); st = _lib.stream_ptr()
m, n, k, ta, tb = (int(x) for x in sys.argv[1:6])
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 3
lib.dcsvd_debug_ws_flags(int(os.environ.get('WS_FLAGS', '0')))
lib.dcsvd_debug_dgemm_ws(int(os.environ.get('DGEMM_WS', '1')))
A = torch.randn(m if ta else k, k if ta else m, dtype=torch.float64, device="cuda").t()
B = torch.randn(k if tb else n, n if tb else k, dtype=torch.float64, device="cuda").t()
C = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
for _ in range(reps):
    lib.dcsvd_dgemm(h, ta, tb, m, n, k, -1.0, _lib.ptr(A), A.stride(1), _lib.ptr(B), B.stride(1), 1.0, _lib.ptr(C), C.stride(1), st)
torch.cuda.synchronize()
