"""ORMBR preparation (Y of every CWY block, batched op(T)) on the side stream during BDC
(dcsvd_debug_ormbr_overlap 1) vs after it (0): gesdd time, phases, U/Vt agreement."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
lib = _lib.load_library()
for n in [int(x) for x in sys.argv[1:]] or [1024, 2048, 8192]:
    a = g.generate_matrix(g.MatrixSpec("random", n, n, seed=2), device=True)
    res = {}
    for on in (0, 1, 0, 1):
        lib.dcsvd_debug_ormbr_overlap(on)
        r = g.gesdd(a); torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); g.gesdd(a); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        ph = [round(t * 1e3, 2) for _, t in g.phase_profile(a).phases][2:5]
        res[on] = r
        print(f"n {n} overlap {on}: gesdd {min(ts):.2f} ms phases gebrd/bdc/ormbr {ph}", flush=True)
    r0, r1 = res[0], res[1]
    print(f"n {n}: dsigma {float((r0.sigma - r1.sigma).abs().max()):.1e} dU {float((r0.u - r1.u).abs().max()):.1e} "
          f"dVt {float((r0.vt - r1.vt).abs().max()):.1e}", flush=True)
lib.dcsvd_debug_ormbr_overlap(1)
