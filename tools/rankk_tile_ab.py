"""Rank-k TMA tile kernels: register-prefetched C (dgemm_ws 1 / 3 = any K) vs
C staged in shared memory by the producer (4 = K > 64, 5 = any K), against
the streaming kernel (0); correctness vs torch and TFLOP/s, then C2 phases."""
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
for (m, n, k, tb) in [(8160, 8160, 64, 1), (4064, 4064, 64, 1), (2016, 2016, 64, 1), (992, 992, 64, 1), (8192, 8192, 128, 0), (65536, 1024, 128, 0), (2048, 2048, 128, 0), (1024, 1024, 128, 0), (2000, 3000, 100, 1), (65536, 896, 128, 0)]:
    A = torch.randn(k, m, dtype=torch.float64, device="cuda").t()
    B = torch.randn(k, n, dtype=torch.float64, device="cuda").t() if tb else torch.randn(n, k, dtype=torch.float64, device="cuda").t()
    C0 = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
    ref = C0 - A @ (B.t() if tb else B)
    out = dict(m=m, n=n, k=k)
    for w in (0, 3, 5):
        lib.dcsvd_debug_dgemm_ws(w)
        C = C0.clone()
        f = lambda: lib.dcsvd_dgemm(h, 0, tb, m, n, k, -1.0, _lib.ptr(A), A.stride(1), _lib.ptr(B), B.stride(1), 1.0, _lib.ptr(C), C.stride(1), st)
        f(); torch.cuda.synchronize()
        out[f"err{w}"] = float((C - ref).abs().max())
        out[f"tf{w}"] = round(2 * m * n * k / t(f) / 1e12, 2)
    lib.dcsvd_debug_dgemm_ws(1)
    print(json.dumps(out), flush=True)
for (mm, nn, sd) in [(8192, 8192, 2), (65536, 1024, 3), (1024, 1024, 1), (2048, 2048, 1000)]:
  a = g.generate_matrix(g.MatrixSpec("random", mm, nn, seed=sd), device=True)
  for w in (1, 5, 1, 5):
    lib.dcsvd_debug_dgemm_ws(w); g.gesdd(a); p = g.phase_profile(a)
    print(json.dumps(dict(n=mm, w=w, total=round(p.total * 1e3, 2), **{k: round(v * 1e3, 2) for k, v in p.phases})), flush=True)
lib.dcsvd_debug_dgemm_ws(1)
