"""rankk_ws_kernel knob sweep: work-unit chunk (row tiles per B strip) and
the C L2 prefetch, on the GEBRD (K=64) and ORMBR (K=128) shapes."""
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
for (m, n, k, tb) in [(8160, 8160, 64, 1), (8192, 8192, 128, 0), (65536, 1024, 128, 0)]:
    A = torch.randn(k, m, dtype=torch.float64, device="cuda").t()
    B = torch.randn(k, n, dtype=torch.float64, device="cuda").t() if tb else torch.randn(n, k, dtype=torch.float64, device="cuda").t()
    C = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
    f = lambda: lib.dcsvd_dgemm(h, 0, tb, m, n, k, -1.0, _lib.ptr(A), A.stride(1), _lib.ptr(B), B.stride(1), 1.0, _lib.ptr(C), C.stride(1), st)
    out = dict(m=m, n=n, k=k)
    for fl in (0, 2, 6):
        lib.dcsvd_debug_ws_flags(fl)
        for c in (0,):
            lib.dcsvd_debug_rankk_chunk(c)
            out[f"f{fl}c{c}"] = round(2 * m * n * k / t(f) / 1e12, 2)
    lib.dcsvd_debug_ws_flags(0); lib.dcsvd_debug_rankk_chunk(0)
    print(json.dumps(out), flush=True)
