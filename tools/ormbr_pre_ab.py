"""ORMBR with op(T) of all CWY blocks precomputed in batched launches
(dcsvd_debug_ormbr_pre 1) vs per block (0): gesdd time, ORMBR phase time,
sigma / U / Vt agreement."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
lib = _lib.load_library()
for n in [int(x) for x in sys.argv[1:]] or [1024, 2048, 8192]:
    a = g.generate_matrix(g.MatrixSpec("random", n, n, seed=2), device=True)
    res = {}
    for pre in (0, 1):
        lib.dcsvd_debug_ormbr_pre(pre)
        r = g.gesdd(a); torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); g.gesdd(a); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        prof = [round(t * 1e3, 2) for _, t in g.phase_profile(a).phases][2:5]
        res[pre] = (r, min(ts), prof)
    r0, r1 = res[0][0], res[1][0]
    du = float((r0.u - r1.u).abs().max()); dv = float((r0.vt - r1.vt).abs().max())
    ds = float((r0.sigma - r1.sigma).abs().max() / r0.sigma[0])
    print(f"n {n}: gesdd per-block T {res[0][1]:.2f} ms, batched T {res[1][1]:.2f} ms | phases {res[0][2]} -> {res[1][2]} | "
          f"dsigma {ds:.1e} dU {du:.1e} dVt {dv:.1e}", flush=True)
lib.dcsvd_debug_ormbr_pre(1)
