"""Rank-k update: warp-specialized TMA kernel (rankk_ws_kernel, 1) vs
rankk_stream_kernel (0).  Micro TFLOP/s + max error vs torch on pipeline
shapes, then full-SVD phase times.

Usage: python tools/rankk_ws_ab.py [svd n, 0 = skip]
"""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
lib = _lib.load_library(); h = _lib.handle(); st = _lib.stream_ptr()
def t(fn, it=10):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / it * 1e-3
for (m, n, k, tb) in [(8160, 8160, 64, 1), (4064, 4064, 64, 1), (2016, 2016, 64, 1), (8192, 8192, 128, 0),
                      (8192, 4096, 128, 0), (2048, 2048, 128, 0), (65536, 1024, 128, 0), (8192, 8192, 40, 1),
                      (3000, 2999, 37, 1), (2050, 1500, 99, 0), (1024, 1024, 64, 1)]:
    A = torch.randn(k, m, dtype=torch.float64, device="cuda").t()
    B = torch.randn(k, n, dtype=torch.float64, device="cuda").t() if tb else torch.randn(n, k, dtype=torch.float64, device="cuda").t()
    C0 = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
    out = dict(m=m, n=n, k=k, tb=tb)
    ref = C0 - A @ (B.t() if tb else B)
    for r in (1, 0):
        lib.dcsvd_debug_rankk_ws(r)
        C = C0.clone()
        f = lambda: lib.dcsvd_dgemm(h, 0, tb, m, n, k, -1.0, _lib.ptr(A), A.stride(1), _lib.ptr(B), B.stride(1), 1.0, _lib.ptr(C), C.stride(1), st)
        f(); torch.cuda.synchronize()
        out[f"err{r}"] = float((C - ref).abs().max())
        out[f"tf{r}"] = round(2 * m * n * k / t(f) / 1e12, 2)
    lib.dcsvd_debug_rankk_ws(1)
    print(json.dumps(out), flush=True)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
if N:
    a = torch.rand(N, N, dtype=torch.float64, device="cuda").t()
    g.gesdd(a)
    for rep in range(2):
        for r in (1, 0):
            lib.dcsvd_debug_rankk_ws(r)
            p = g.phase_profile(a)
            print(json.dumps(dict(ws=r, total=round(p.total * 1e3, 2), **{k: round(v * 1e3, 2) for k, v in p.phases})), flush=True)
    lib.dcsvd_debug_rankk_ws(1)
