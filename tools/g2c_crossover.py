"""GEBRD time vs the two-phase-LABRD / cluster-GEBD2 crossover (dcsvd_debug_gebd2_max_cols)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
lib = _lib.load_library()
for n in [int(x) for x in sys.argv[1:]] or [512, 1024, 2048]:
    a = g.generate_matrix(g.MatrixSpec("random", n, n, seed=2), device=True)
    row = []
    for mc in [int(x) for x in os.environ.get("MCS", "128 192 256 320 384 448 512").split()]:
        lib.dcsvd_debug_gebd2_max_cols(mc)
        g.gebrd_blocked(a.clone()); torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            b = a.clone()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); g.gebrd_blocked(b); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        row.append(f"{mc}: {min(ts):6.2f}")
    lib.dcsvd_debug_gebd2_max_cols(512)
    print(f"gebrd {n}: " + "  ".join(row), flush=True)
