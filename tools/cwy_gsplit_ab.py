"""G = Y^T Y with its own split-K on the TMA GEMM (1) vs sharing the Z split (0): C2 / C3 / C1 phases."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
lib = _lib.load_library()
for (m, n, seed) in [(8192, 8192, 2), (65536, 1024, 3), (1024, 1024, 1)]:
    a = g.generate_matrix(g.MatrixSpec("random", m, n, seed=seed), device=True)
    for rep in range(2):
        for mode in (1, 0):
            lib.dcsvd_debug_cwy_gsplit(mode)
            g.gesdd(a)
            p = g.phase_profile(a)
            r = g.gesdd(a)
            acc = g.accuracy(a, r)
            print(json.dumps(dict(m=m, mode=mode, total=round(p.total * 1e3, 2), resid=acc.e_svd / max(m, n), orth=acc.orth_u / n,
                                  **{k: round(v * 1e3, 2) for k, v in p.phases})), flush=True)
lib.dcsvd_debug_cwy_gsplit(1)
