"""A/B of evict_last / evict_first L2 hints on the large-panel LABRD GEMV passes
(dcsvd_debug_labrd_l2keep): GEBRD phase time of full SVDs per kept-bytes setting.

Usage: python tools/labrd_l2keep_ab.py [n] [MB ...]
"""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
lib = _lib.load_library()
lib.dcsvd_debug_labrd_l2keep.argtypes = [ctypes.c_double]
lib.dcsvd_debug_labrd_l2keep_min.argtypes = [ctypes.c_double]
if os.environ.get("L2KEEP_MIN_MB"):
    lib.dcsvd_debug_labrd_l2keep_min(float(os.environ["L2KEEP_MIN_MB"]) * 2**20)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
mbs = [float(x) for x in sys.argv[2:]] or [0, 48, 64, 80, 96]
a = torch.rand(n, n, dtype=torch.float64, device="cuda").t()
g.gesdd(a)
for rep in range(2):
    for mb in mbs:
        lib.dcsvd_debug_labrd_l2keep(mb * 2**20)
        p = g.phase_profile(a)
        print(f"n {n} l2keep {mb:5.0f} MB: total {p.total*1e3:8.2f} ms  gebrd {dict(p.phases)['gebrd']*1e3:8.2f} ms", flush=True)
lib.dcsvd_debug_labrd_l2keep(0.0)
