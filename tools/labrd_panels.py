"""Per-panel LABRD time and effective bandwidth over one GEBRD (dev tool)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a = torch.rand(n, n, dtype=torch.float64, device="cuda").t()
g.gebrd_blocked(a.clone().t().contiguous().t())
_lib.set_stats(True)
g.gebrd_blocked(a.clone().t().contiguous().t())
lib = _lib.load_library(); h = _lib.handle()
cap = 4096
ms = np.zeros(cap); wk = np.zeros(cap)
c = lib.dcsvd_debug_stat_records(h, 0, ms.ctypes.data_as(ctypes.c_void_p), wk.ctypes.data_as(ctypes.c_void_p), cap)
ms, wk = ms[:c], wk[:c]
print(f"panels {c}, total labrd {ms.sum():.1f} ms, bytes {wk.sum()/1e9:.1f} GB, eff {wk.sum()/ms.sum()/1e6:.0f} GB/s")
for lo in range(0, c, max(1, c // 16)):
    sl = slice(lo, min(c, lo + max(1, c // 16)))
    nv = n - 32 * lo
    print(f"  n'~{nv:5d}: {ms[sl].sum():7.2f} ms  {wk[sl].sum()/ms[sl].sum()/1e6:7.0f} GB/s  per-col {ms[sl].sum()*1e3/(32*len(ms[sl])):6.1f} us")
