"""GEBRD 8192^2 time vs the large-panel GEMV L2 eviction-hint window
(dcsvd_debug_labrd_l2keep bytes kept evict_last per pass, dcsvd_debug_labrd_l2keep_min
smallest panel matrix that uses the hints)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
lib = _lib.load_library()
lib.dcsvd_debug_labrd_l2keep.argtypes = [ctypes.c_double]
lib.dcsvd_debug_labrd_l2keep_min.argtypes = [ctypes.c_double]
a = g.generate_matrix(g.MatrixSpec("random", 8192, 8192, seed=2), device=True)
def timed(reps=2):
    g.gebrd_blocked(a.clone()); torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        b = a.clone()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.gebrd_blocked(b); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return min(ts)
MB = float(1 << 20)
for keep, kmin in ((20, 160), (0, 160), (12, 160), (28, 160), (36, 160), (20, 120), (20, 240), (28, 240), (20, 160)):
    lib.dcsvd_debug_labrd_l2keep(keep * MB); lib.dcsvd_debug_labrd_l2keep_min(kmin * MB)
    print(f"keep {keep} MB, min {kmin} MB: gebrd {timed():.2f} ms", flush=True)
lib.dcsvd_debug_labrd_l2keep(20 * MB); lib.dcsvd_debug_labrd_l2keep_min(160 * MB)
