"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_11467_b200 as g
rng = np.random.default_rng(0)
for (m, n) in [(97, 97), (150, 61), (61, 150), (400, 100)]:
    a = rng.standard_normal((m, n)); r = g.gesdd(a)
    print(m, n, float(np.abs(np.sort(r.sigma)[::-1] - np.linalg.svd(a, compute_uv=False)).max()), flush=True)
for n, leaf, bord in [(77, 8, True), (130, 32, False), (40, 1, False)]:
    d = rng.standard_normal(n); e = rng.standard_normal(n if bord else n - 1)
    g.bdsdc(g.BidiagonalProblem(d, e, bord), leaf=leaf)
g.gesdd_batched([rng.standard_normal((90, 90)) for _ in range(3)], concurrency=3)
a = rng.standard_normal((300, 260)); g.matmul_accumulate(1.0, a, False, a, True, 0.0, np.zeros((300, 300)))
print("done")
