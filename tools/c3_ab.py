"""C3 gesdd (65536 x 1024) time and phases with a given library build.
Usage: python tools/c3_ab.py LIBPATH"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2508_11467_b200 import _lib
_lib.load_library(sys.argv[1])
import paper_2508_11467_b200 as g
a = g.generate_matrix(g.MatrixSpec("random", 65536, 1024, seed=3), device=True)
g.gesdd(a); torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); r = g.gesdd(a); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ph = g.phase_profile(a)
print(f"{os.path.basename(sys.argv[1])}: C3 {min(ts):.2f} ms  phases " +
      " ".join(f"{k} {v * 1e3:.2f}" for k, v in ph.phases) + f"  sigma0 {float(r.sigma[0]):.15e}", flush=True)
