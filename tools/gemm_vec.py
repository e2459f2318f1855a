"""16-byte vs 8-byte cp.async staging in the DMMA GEMM (debug route 5; dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2508_11467_b200 import _lib
lib = _lib.load_library(); h = _lib.handle(); st = _lib.stream_ptr()
def col(r, c):
    return torch.randn(c, r, dtype=torch.float64, device="cuda").t()
for (m, n, k) in [(8192, 8192, 8192), (8192, 6000, 6000), (4096, 4096, 2048)]:
    A, B, C = col(m, k), col(k, n), col(m, n)
    for route in [int(x) for x in (sys.argv[1:] or ['0', '5'])]:
        lib.dcsvd_debug_gemm_route(route)
        f = lambda: lib.dcsvd_dgemm(h, 0, 0, m, n, k, 1.0, _lib.ptr(A), m, _lib.ptr(B), k, 0.0, _lib.ptr(C), m, st)
        f(); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(3): f()
        e.record(); torch.cuda.synchronize()
        t = s.elapsed_time(e) / 3e3
        print(f"{m}x{n}x{k} route {route}: {2*m*n*k/t/1e12:.1f} TF/s")
lib.dcsvd_debug_gemm_route(0)
