"""Time GEBRD and gesdd with a given build of the library (A/B across builds).
Usage: python tools/lib_ab.py LIBPATH n [n ...]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2508_11467_b200 import _lib
_lib.load_library(sys.argv[1])
import paper_2508_11467_b200 as g


def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


for n in [int(x) for x in sys.argv[2:]]:
    a = g.generate_matrix(g.MatrixSpec("random", n, n, seed=2), device=True)
    tg = timed(lambda: g.gebrd_blocked(a.clone()))
    ts = timed(lambda: g.gesdd(a))
    s = g.gesdd(a).sigma
    print(f"{os.path.basename(sys.argv[1])} n {n}: gebrd {tg:8.2f} ms  gesdd {ts:8.2f} ms  sigma0 {float(s[0]):.15e}", flush=True)
