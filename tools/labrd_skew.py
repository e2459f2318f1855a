"""Per-CTA GEMV completion skew in one column step of the first LABRD panel
(four-phase kernel; dev tool).  Slots: 400 GEMV1 done, 600 after barrier,
800 GEMV2 done, 1000 after barrier."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2508_11467_b200 as g
lib = g._lib.load_library()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a = torch.rand(n, n, dtype=torch.float64, device="cuda").t()
g.gebrd_blocked(a.clone().t().contiguous().t())
buf = torch.zeros(1200, dtype=torch.int64, device="cuda")
lib.dcsvd_debug_labrd_tlog(ctypes.c_void_p(buf.data_ptr()))
g.gebrd_blocked(a.clone().t().contiguous().t())
t = buf.cpu().numpy().astype(np.float64)
for name, s0, s1 in (("GEMV1 (A^T v)", 400, 600), ("GEMV2 (A u)", 800, 1000)):
    done = t[s0:s0 + 148]; rel = t[s1:s1 + 148]
    G = int(np.count_nonzero(done))
    done, rel = done[:G], rel[:G]
    start = rel.min()
    w = rel.max() - done
    print(f"{name}: CTAs {G}; finish spread {(done.max()-done.min())/1e3:.2f} us; mean wait at barrier {w.mean()/1e3:.2f} us; "
          f"max wait {w.max()/1e3:.2f} us; release spread {(rel.max()-rel.min())/1e3:.2f} us")
    order = np.argsort(done)
    print("   slowest CTAs:", order[-6:], "fastest:", order[:6])
