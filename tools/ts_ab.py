"""TS recombination A/B: literal ORGQR + GEMM (1, driver.py:141-142) vs the
fused reflector apply to [U0; 0] (0).  C3 shape; phase times + accuracy."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
lib = _lib.load_library()
m, n = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (65536, 1024)
a = g.generate_matrix(g.MatrixSpec("random", m, n, seed=3), device=True)
for rep in range(2):
    for lit in (1, 0):
        lib.dcsvd_debug_ts_literal(lit)
        g.gesdd(a)
        torch.cuda.synchronize()
        p = g.phase_profile(a)
        r = g.gesdd(a)
        acc = g.accuracy(a, r)
        print(json.dumps(dict(literal=lit, total=round(p.total * 1e3, 3), **{k: round(v * 1e3, 3) for k, v in p.phases},
                              resid=acc.e_svd / m, orth_u=acc.orth_u / n)), flush=True)
lib.dcsvd_debug_ts_literal(1)
