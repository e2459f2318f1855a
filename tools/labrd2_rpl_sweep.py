"""GEBRD time per forced two-phase LABRD geometry (rows per lane) on squares
whose panels all run the two-phase kernel (dcsvd_debug_labrd2_rpl)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
lib = _lib.load_library()
for n in [int(x) for x in sys.argv[1:]] or [768, 1024, 1536, 2048]:
    a = g.generate_matrix(g.MatrixSpec("random", n, n, seed=2), device=True)
    row = []
    for rpl in (0, 2, 4, 8, 16):
        lib.dcsvd_debug_labrd2_rpl(rpl)
        try:
            g.gebrd_blocked(a.clone()); torch.cuda.synchronize()
            ts = []
            for _ in range(3):
                b = a.clone()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); g.gebrd_blocked(b); e1.record(); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            row.append(f"rpl {rpl or 'auto'}: {min(ts):7.2f}")
        except Exception as ex:
            row.append(f"rpl {rpl}: n/a")
    lib.dcsvd_debug_labrd2_rpl(0)
    print(f"gebrd {n}: " + "  ".join(row), flush=True)
