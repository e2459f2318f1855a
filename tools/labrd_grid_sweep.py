"""GEBRD time vs the LABRD grid cap (dcsvd_debug_labrd_gmax) on small squares.

Usage: python tools/labrd_grid_sweep.py [n ...]
"""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
lib = _lib.load_library()
sizes = [int(x) for x in sys.argv[1:]] or [512, 1024, 2048]
for n in sizes:
    a = torch.rand(n, n, dtype=torch.float64, device="cuda").t()
    row = []
    for gmax in (16, 32, 48, 64, 96, 128, 0):
        lib.dcsvd_debug_labrd_gmax(gmax)
        g.gebrd_blocked(a.clone().t().contiguous().t())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        bufs = [a.clone().t().contiguous().t() for _ in range(3)]
        e0.record()
        for b in bufs:
            g.gebrd_blocked(b)
        e1.record()
        torch.cuda.synchronize()
        row.append((gmax or 148, e0.elapsed_time(e1) / 3))
    lib.dcsvd_debug_labrd_gmax(0)
    print(f"n {n}: " + "  ".join(f"G<={gm}: {t:.2f} ms" for gm, t in row), flush=True)
