"""A/B of the rank-k kernel's C prefetch distance (tiles ahead; 0 = off) on full SVDs.

Usage: python tools/rankk_dist_ab.py [m] [n] [reps] [dists, comma-separated]
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
dists = [int(x) for x in (sys.argv[4] if len(sys.argv) > 4 else "1,2,3,0").split(",")]
a = torch.rand(n, m, dtype=torch.float64, device="cuda").t()
g.gesdd(a)
res = {d: [] for d in dists}
for r in range(reps):
    for d in dists:
        lib.dcsvd_debug_rankk_prefetch(d)
        res[d].append(g.phase_profile(a))
lib.dcsvd_debug_rankk_prefetch(1)
for d in dists:
    ps = res[d]
    names = [k for k, _ in ps[0].phases]
    avg = {k: sum(dict(p.phases)[k] for p in ps) / len(ps) for k in names}
    tot = sum(p.total for p in ps) / len(ps)
    print(f"{m}x{n} dist={d}: total {tot*1e3:8.2f} ms  " + "  ".join(f"{k} {v*1e3:.2f}" for k, v in avg.items()), flush=True)
