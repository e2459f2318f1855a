"""CWY split-K rule A/B: wave-quantised rule for the TMA GEMM (1) vs the
round-1 rule (0); C2-size ORMBR and C3 phases."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
lib = _lib.load_library()
for (m, n, seed) in [(8192, 8192, 2), (65536, 1024, 3)]:
    a = g.generate_matrix(g.MatrixSpec("random", m, n, seed=seed), device=True)
    for rep in range(2):
        for mode in (1, 0):
            lib.dcsvd_debug_cwy_split(mode)
            g.gesdd(a)
            p = g.phase_profile(a)
            print(json.dumps(dict(m=m, mode=mode, total=round(p.total * 1e3, 2), **{k: round(v * 1e3, 2) for k, v in p.phases})), flush=True)
lib.dcsvd_debug_cwy_split(1)
