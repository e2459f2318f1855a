"""Per-phase timeline of one LABRD panel launch (CTA 0 view)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
lib = _lib.load_library()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a = torch.rand(n, n, dtype=torch.float64, device="cuda").t()
g.gebrd_blocked(a.clone().t().contiguous().t())  # warm
buf = torch.zeros(1 + 10 * 32, dtype=torch.int64, device="cuda")
lib.dcsvd_debug_labrd_tlog(ctypes.c_void_p(buf.data_ptr()))
g.gebrd_blocked(a.clone().t().contiguous().t())
t = buf.cpu().numpy().astype(np.float64)
lib.dcsvd_debug_labrd_variant.restype = ctypes.c_int
two = lib.dcsvd_debug_labrd_variant() == 2  # variant of the LAST panel; the logged one is the first
two = two and n <= 2048
W = 8 if two else 10
tt = t[1:1 + W * 32].reshape(32, W)
nxt = np.append(tt[1:, 0], tt[-1, -1])
deltas = np.diff(np.concatenate([tt, nxt[:, None]], axis=1), axis=1)
names = (["A_crit", "A_pre", "A_gemv", "bar", "B_crit", "B_pre", "B_gemv", "bar"] if two else
         ["p2_larfg", "p2_gemv", "bar", "p3", "bar", "p4_larfg", "p4_gemv", "bar", "p5", "bar"])
print("n", n, "two-phase" if two else "four-phase", "per-column us (mean over cols 0..30):")
for i, nm in enumerate(names):
    print(f"  {nm:10s} {deltas[:31, i].mean()/1e3:8.2f}")
print("  total/col  ", deltas[:31].sum(axis=1).mean() / 1e3)
