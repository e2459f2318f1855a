"""Per-CTA phase timestamps of one GEQR2 panel launch (columns 5 and 6).

Marks per column: 0 = iteration start (after the grid barrier), 1 = partials
and pivot row reduced, 2 = reflector applied, 3 = next column's partials
stored.  Usage: python tools/geqr2_tlog.py [m] [w]
"""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
lib = _lib.load_library()
m = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
w = int(sys.argv[2]) if len(sys.argv) > 2 else 32
a = torch.rand(w, m, dtype=torch.float64, device="cuda").t()
tau = torch.zeros(w, dtype=torch.float64, device="cuda")
g.geqrf_panel(a.clone().t().contiguous().t(), tau)  # warm
buf = torch.zeros(24 * 256, dtype=torch.int64, device="cuda")
lib.dcsvd_debug_labrd_tlog(ctypes.c_void_p(buf.data_ptr()))
g.geqrf_panel(a.clone().t().contiguous().t(), tau)
torch.cuda.synchronize()
lib.dcsvd_debug_labrd_tlog(ctypes.c_void_p(0))
tc = buf.cpu().numpy().astype(np.float64).reshape(24, 256)
t = tc[:8]
ck = tc[8:16]
sub = tc[16:24]
G = int((t[0] > 0).sum())
t = t[:, :G]
ck = ck[:, :G]
sub = sub[:, :G]
t0 = t[0].min()
print(f"m {m} w {w} CTAs {G}; times in us relative to the earliest column-5 start")
for k in range(8):
    r = (t[k] - t0) / 1e3
    print(f"  col {5 + k // 4} mark {k % 4}: min {r.min():7.2f}  median {np.median(r):7.2f}  max {r.max():7.2f}")
print("per-CTA phase durations (median / max over CTAs), column 5:")
for k, nm in enumerate(["reduce", "apply", "partials"]):
    d = (t[k + 1] - t[k]) / 1e3
    print(f"  {nm:9s} {np.median(d):6.2f} {d.max():6.2f}")
d = (t[4] - t[3]) / 1e3
print(f"  barrier   {np.median(d):6.2f} {d.max():6.2f}  (last arrival -> first release: {(t[4].min() - t[3].max()) / 1e3:.2f})")
d = (ck[4] - ck[0]) / ((t[4] - t[0]) / 1e3)
print(f"SM clock over column 5 (clock64 / globaltimer): median {np.median(d):.0f} MHz")
for k, nm in enumerate(["reduce", "apply", "partials", "barrier"]):
    print(f"  {nm:9s} {np.median(ck[k + 1] - ck[k]):8.0f} cycles (median CTA)")
if False:  # sub-marks: removed with the register variant

    print("column-5 sub-marks (reg kernel; cycles from mark 1, median CTA):")
    for k, nm in enumerate(["tau + sh_tw", "sync", "update", "butterfly", "sync", "sum + store"]):
        print(f"  {nm:12s} {np.median(sub[k] - ck[1]):8.0f}")
