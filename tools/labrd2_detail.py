"""Fine timeline of the two-phase LABRD critical parts (debug marks 600+; dev tool)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2508_11467_b200 as g
lib = g._lib.load_library()
n = int(sys.argv[1])
a = torch.rand(n, n, dtype=torch.float64, device="cuda").t()
g.gebrd_blocked(a.clone().t().contiguous().t())
buf = torch.zeros(1024, dtype=torch.int64, device="cuda")
lib.dcsvd_debug_labrd_tlog(ctypes.c_void_p(buf.data_ptr()))
g.gebrd_blocked(a.clone().t().contiguous().t())
t = buf.cpu().numpy().astype(np.float64)
main = t[1:1 + 8 * 32].reshape(32, 8)
det = t[600:600 + 8 * 32].reshape(32, 8)
ks = range(2, 30)
def m(x): return np.mean(x) / 1e3
print("A: start->loads+pxs", m([det[k,0]-main[k,0] for k in ks]), " larfg+u", m([det[k,1]-det[k,0] for k in ks]),
      " x/c", m([det[k,2]-det[k,1] for k in ks]), " block_sum", m([main[k,1]-det[k,2] for k in ks]))
print("B: start->loads", m([det[k,4]-main[k,4] for k in ks]), " larfg", m([det[k,5]-det[k,4] for k in ks]),
      " v,y,r", m([det[k,6]-det[k,5] for k in ks]), " block_sum", m([main[k,5]-det[k,6] for k in ks]))
