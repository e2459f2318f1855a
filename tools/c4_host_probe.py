"""C4 (bdsdc n=16384 fixture): device time per call (events) vs host wall per call,
and the launches per call, to see whether the calls are host-bound."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
z = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "c4_n16384.npz"))
d = torch.from_numpy(z["d"]).cuda(); e = torch.from_numpy(z["e"]).cuda()
prob = g.BidiagonalProblem(d, e)
for _ in range(3): g.bdsdc(prob)
torch.cuda.synchronize()
l0 = _lib.launch_count()
t0 = time.perf_counter()
ev = []
for _ in range(10):
    s, f = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); g.bdsdc(prob); f.record(); ev.append((s, f))
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / 10 * 1e3
dev = [s.elapsed_time(f) for s, f in ev]
print(f"wall/call {wall:.2f} ms, device/call min {min(dev):.2f} median {sorted(dev)[5]:.2f} ms, "
      f"launches/call {(_lib.launch_count() - l0) / 10:.0f}", flush=True)
