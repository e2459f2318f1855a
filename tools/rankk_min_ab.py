"""Smallest C routed to the streaming rank-k kernel: full SVD / GEBRD phase times per threshold."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
lib = _lib.load_library()
lib.dcsvd_debug_rankk_min.argtypes = [ctypes.c_longlong]
for (m, n) in [(1024, 1024), (2048, 2048), (65536, 1024)]:
    a = torch.rand(n, m, dtype=torch.float64, device="cuda").t()
    g.gesdd(a)
    for rep in range(3):
        for mn in (1024 * 1024, 512 * 512, 256 * 256):
            lib.dcsvd_debug_rankk_min(mn)
            p = g.phase_profile(a)
            print(f"{m}x{n} min={mn}: total {p.total*1e3:8.3f} ms  " + "  ".join(f"{k} {v*1e3:.3f}" for k, v in p.phases if v), flush=True)
    lib.dcsvd_debug_rankk_min(0)
