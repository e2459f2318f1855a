"""General DMMA GEMM: warp-specialized TMA kernel (dgemm_ws_kernel, 1) vs the
cp.async dgemm_kernel (0) on pipeline shapes (CWY inner products, TS
recombination, big square), incl. split-K through block_reflector; max error
vs torch fp64 and TFLOP/s."""
import sys, os, json
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
torch.manual_seed(0)
for (m, n, k, ta, tb, beta) in [(128, 8192, 8192, 1, 0, 0.0), (8192, 128, 8192, 0, 1, 0.0), (65536, 1024, 1024, 0, 0, 0.0),
                                (8192, 8192, 8192, 0, 0, 1.0), (4096, 6900, 3450, 0, 0, 0.0), (1000, 777, 333, 1, 1, 0.5),
                                (2000, 3000, 130, 0, 1, 1.0), (128, 1024, 65536, 1, 0, 0.0)]:
    A = torch.randn(k if ta else m, m if ta else k, dtype=torch.float64, device="cuda").t().contiguous().t()
    B = torch.randn(n if tb else k, k if tb else n, dtype=torch.float64, device="cuda").t().contiguous().t()
    C0 = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
    ref = beta * C0 + 0.75 * ((A.t() if ta else A) @ (B.t() if tb else B))
    out = dict(m=m, n=n, k=k, ta=ta, tb=tb)
    for w in (1, 0):
        lib.dcsvd_debug_dgemm_ws(w)
        C = C0.clone()
        f = lambda: lib.dcsvd_dgemm(h, ta, tb, m, n, k, 0.75, _lib.ptr(A), A.stride(1), _lib.ptr(B), B.stride(1), beta, _lib.ptr(C), C.stride(1), st)
        f(); torch.cuda.synchronize()
        out[f"err{w}"] = float((C - ref).abs().max() / ref.abs().max())
        if beta == 0.0:
            out[f"tf{w}"] = round(2 * m * n * k / t(f) / 1e12, 2)
    lib.dcsvd_debug_dgemm_ws(1)
    print(json.dumps(out), flush=True)
