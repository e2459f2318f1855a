"""Per-phase cycles of the cluster GEBD2 kernel (CTA 0, column 5).

Usage: python tools/gebd2c_tlog.py [n]
"""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
lib = _lib.load_library()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
a = torch.rand(n, n, dtype=torch.float64, device="cuda").t()
g.gebrd_blocked(a.clone().t().contiguous().t(), 32)
buf = torch.zeros(16, dtype=torch.int64, device="cuda")
lib.dcsvd_debug_labrd_tlog(ctypes.c_void_p(buf.data_ptr()))
g.gebrd_blocked(a.clone().t().contiguous().t(), 32)
torch.cuda.synchronize()
lib.dcsvd_debug_labrd_tlog(ctypes.c_void_p(0))
t = buf.cpu().numpy().astype(np.float64)
names = ["norm partial", "sync1", "larfg+scale", "w partial", "sync2", "w reduce", "sync3", "gather+update",
         "row refl", "sync4", "u, x, update"]
print(f"n {n}: column 5, CTA 0, cycles per phase (total {t[11] - t[0]:.0f})")
for i, nm in enumerate(names):
    print(f"  {nm:14s} {t[i + 1] - t[i]:8.0f}")
