"""Run bdsdc on the bidiagonal of an n x n random matrix or the C4 fixture (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np, time
import paper_2508_11467_b200 as g
which = sys.argv[1] if len(sys.argv) > 1 else "c4"
if which == "c4":
    z = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests/golden/c4_n16384.npz"))
    d, e = torch.from_numpy(z["d"]).cuda(), torch.from_numpy(z["e"]).cuda()
else:
    n = int(which)
    a = torch.rand(n, n, dtype=torch.float64, device="cuda").t()
    f = g.gebrd_blocked(a.clone().t().contiguous().t())
    d, e = f.d, f.e
prob = g.BidiagonalProblem(d, e)
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = g.bdsdc(prob); torch.cuda.synchronize()
    print(which, "bdsdc", (time.perf_counter() - t0) * 1e3, "ms", flush=True)
