"""C4 host gap: per-call wall time vs GPU span of bdsdc on the n = 16384 fixture,
and the same with a CUDA-event-only view of each call's first and last kernel."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_11467_b200 as g
z = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "c4_n16384.npz"))
d = torch.from_numpy(z["d"]).cuda(); e = torch.from_numpy(z["e"]).cuda()
prob = g.BidiagonalProblem(d, e)
for _ in range(3): r = g.bdsdc(prob)
torch.cuda.synchronize()
walls = []
for _ in range(10):
    t0 = time.perf_counter(); r = g.bdsdc(prob); walls.append((time.perf_counter() - t0) * 1e3)
print("wall per call ms:", [round(w, 2) for w in walls])
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(5): r = g.bdsdc(prob)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(8)
