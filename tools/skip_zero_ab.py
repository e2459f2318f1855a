"""GEBRD panels without the P / Q zero fill (dcsvd_debug_labrd_skip_zero 1) vs with (0):
gesdd / GEBRD time and bitwise equality of the factorization and the SVD."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
lib = _lib.load_library()
def timed(fn, reps=3):
    fn(); torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return min(ts)
for n in [int(x) for x in sys.argv[1:]] or [1024, 3072, 8192]:
    a = g.generate_matrix(g.MatrixSpec("random", n, n, seed=2), device=True)
    out = {}
    for on in (0, 1, 0, 1):
        lib.dcsvd_debug_labrd_skip_zero(on)
        tg = timed(lambda: g.gebrd_blocked(a.clone()))
        ts = timed(lambda: g.gesdd(a), reps=2)
        b = a.clone(); f = g.gebrd_blocked(b); r = g.gesdd(a)
        out[on] = (b, f.d, f.e, r.sigma, r.u, r.vt)
        print(f"n {n} skip {on}: gebrd {tg:.2f} ms gesdd {ts:.2f} ms", flush=True)
    same = all(torch.equal(x, y) for x, y in zip(out[0], out[1]))
    print(f"n {n}: bitwise identical: {same}", flush=True)
lib.dcsvd_debug_labrd_skip_zero(1)
