"""A/B of the rank-k kernel's next-tile L2 prefetch on full SVDs (phase times).

Usage: python tools/rankk_prefetch_ab.py [m] [n] [reps]
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
lib = _lib.load_library()
m = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
n = int(sys.argv[2]) if len(sys.argv) > 2 else m
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
a = torch.rand(n, m, dtype=torch.float64, device="cuda").t()
g.gesdd(a)
res = {0: [], 1: []}
for r in range(reps):
    for on in (1, 0):
        lib.dcsvd_debug_rankk_prefetch(on)
        p = g.phase_profile(a)
        res[on].append(p)
lib.dcsvd_debug_rankk_prefetch(1)
for on in (1, 0):
    ps = res[on]
    names = [k for k, _ in ps[0].phases]
    avg = {k: sum(dict(p.phases)[k] for p in ps) / len(ps) for k in names}
    tot = sum(p.total for p in ps) / len(ps)
    print(f"{m}x{n} prefetch={on}: total {tot*1e3:8.2f} ms  " + "  ".join(f"{k} {v*1e3:.2f}" for k, v in avg.items()), flush=True)
