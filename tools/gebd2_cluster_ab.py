"""A/B of the cluster GEBD2 tail (dcsvd_debug_gebd2_cluster) on GEBRD and full SVDs,
with the bidiagonal of both paths compared.

Usage: python tools/gebd2_cluster_ab.py [n ...]
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
lib = _lib.load_library()
sizes = [int(x) for x in sys.argv[1:]] or [256, 512, 1024, 2048]


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for n in sizes:
    a = torch.rand(n, n, dtype=torch.float64, device="cuda").t()
    out = {}
    for on in (0, 1):
        lib.dcsvd_debug_gebd2_cluster(on)
        b = a.clone().t().contiguous().t()
        f = g.gebrd_blocked(b)
        dd = np.asarray(f.d.cpu() if isinstance(f.d, torch.Tensor) else f.d)
        ee = np.asarray(f.e.cpu() if isinstance(f.e, torch.Tensor) else f.e)
        t_gebrd = timed(lambda: g.gebrd_blocked(a.clone().t().contiguous().t()))
        t_svd = timed(lambda: g.gesdd(a), reps=2)
        out[on] = (dd, ee, t_gebrd, t_svd)
    lib.dcsvd_debug_gebd2_cluster(1)
    dd0, ee0 = out[0][0], out[0][1]
    dd1, ee1 = out[1][0], out[1][1]
    scale = max(np.max(np.abs(dd0)), 1.0)
    print(f"n {n}: gebrd {out[0][2]:.2f} -> {out[1][2]:.2f} ms, gesdd {out[0][3]:.2f} -> {out[1][3]:.2f} ms; "
          f"max |d| diff {np.max(np.abs(np.abs(dd1) - np.abs(dd0))) / scale:.1e}, |e| diff "
          f"{np.max(np.abs(np.abs(ee1) - np.abs(ee0))) / scale:.1e}", flush=True)
