"""C2 gesdd / GEBRD with 8-wide panels allowed only for views up to a size bound
(dcsvd_debug_labrd_halfwidth(2, max_elems)) vs the default rule."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
lib = _lib.load_library()
n = 8192
a = g.generate_matrix(g.MatrixSpec("random", n, n, seed=2), device=True)
def timed(fn, reps=3):
    fn(); torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return min(ts)
for mode, mx in ((1, 0), (2, 4352 * 4352), (2, 4608 * 4608), (2, 5120 * 5120), (1, 0)):
    lib.dcsvd_debug_labrd_halfwidth(mode, mx)
    print(f"mode {mode} max {mx}: gebrd {timed(lambda: g.gebrd_blocked(a.clone())):.2f} ms  gesdd {timed(lambda: g.gesdd(a)):.2f} ms", flush=True)
lib.dcsvd_debug_labrd_halfwidth(1, 0)
