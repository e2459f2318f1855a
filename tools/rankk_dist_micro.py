"""Rank-k streaming kernel alone: TFLOP/s vs C prefetch distance (tiles ahead; 0 = off)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2508_11467_b200 import _lib
lib = _lib.load_library(); h = _lib.handle(); st = _lib.stream_ptr()
def t(fn, it=10):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / it * 1e-3
for (m, n, k, tb) in [(8160, 8160, 64, 1), (8192, 8192, 128, 0), (4064, 4064, 64, 1), (2016, 2016, 64, 1)]:
    A = torch.randn(k, m, dtype=torch.float64, device="cuda").t()
    B = (torch.randn(k, n, dtype=torch.float64, device="cuda") if tb else torch.randn(n, k, dtype=torch.float64, device="cuda").t())
    B = B.t() if tb else B  # tb: B stored n x k (ld = n)
    B = torch.randn(k, n, dtype=torch.float64, device="cuda").t() if tb else torch.randn(n, k, dtype=torch.float64, device="cuda").t()
    C = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
    out = dict(m=m, n=n, k=k, tb=tb)
    for d in (1, 2, 3, 0):
        lib.dcsvd_debug_rankk_prefetch(d)
        f = lambda: lib.dcsvd_dgemm(h, 0, tb, m, n, k, -1.0, _lib.ptr(A), A.stride(1), _lib.ptr(B), B.stride(1), 1.0, _lib.ptr(C), C.stride(1), st)
        out[f"d{d}"] = round(2 * m * n * k / t(f) / 1e12, 2)
    lib.dcsvd_debug_rankk_prefetch(1)
    print(json.dumps(out), flush=True)
