"""GEBRD (and C2 gesdd) time with half-width panels in the middle range
(dcsvd_debug_labrd_halfwidth): 0 = always 32-wide, 1 = 16-wide where that lets
the two-phase LABRD kernel run, 2 = also 8-wide."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
lib = _lib.load_library()


def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


sizes = [int(x) for x in sys.argv[1:]] or [2048, 3072, 4096, 6144, 8192]
for n in sizes:
    a = g.generate_matrix(g.MatrixSpec("random", n, n, seed=2), device=True)
    row, ds = [], {}
    for mode in (0, 1, 2):
        lib.dcsvd_debug_labrd_halfwidth(mode, 0)
        t = timed(lambda: g.gebrd_blocked(a.clone()))
        f = g.gebrd_blocked(a.clone()); torch.cuda.synchronize()
        ds[mode] = f.d.abs()
        row.append(f"mode {mode}: {t:8.2f} ms")
    dev = max(float((ds[mm] - ds[0]).abs().max() / ds[0].abs().max()) for mm in (1, 2))
    print(f"gebrd {n}: " + "  ".join(row) + f"  |d| rel dev {dev:.1e}", flush=True)
n = 8192
a = g.generate_matrix(g.MatrixSpec("random", n, n, seed=2), device=True)
for mode in (0, 1, 2):
    lib.dcsvd_debug_labrd_halfwidth(mode, 0)
    t = timed(lambda: g.gesdd(a), reps=2)
    r = g.gesdd(a)
    print(f"gesdd {n} mode {mode}: {t:8.2f} ms  sigma[0] {float(r.sigma[0]):.15e}", flush=True)
lib.dcsvd_debug_labrd_halfwidth(1, 0)
