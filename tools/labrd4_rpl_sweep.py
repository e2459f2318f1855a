"""GEBRD 8192^2 / 6144^2 time per forced four-phase LABRD geometry (dcsvd_debug_labrd4_rpl)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
lib = _lib.load_library()
for n in [int(x) for x in sys.argv[1:]] or [8192, 6144]:
    a = g.generate_matrix(g.MatrixSpec("random", n, n, seed=2), device=True)
    row = []
    for rpl in (0, 4, 8, 16):
        lib.dcsvd_debug_labrd4_rpl(rpl)
        try:
            g.gebrd_blocked(a.clone()); torch.cuda.synchronize()
            ts = []
            for _ in range(2):
                b = a.clone()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); g.gebrd_blocked(b); e1.record(); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            row.append(f"rpl {rpl or 'auto'}: {min(ts):7.2f}")
        except Exception as ex:
            row.append(f"rpl {rpl}: n/a ({str(ex)[:40]})")
    lib.dcsvd_debug_labrd4_rpl(0)
    print(f"gebrd {n}: " + "  ".join(row), flush=True)
