"""Small runs for compute-sanitizer racecheck (the full sanitize_small.py exceeds
the racecheck time budget with its 1500^2 SVD): cluster GEBD2 tail, two-phase
LABRD, the TMA rank-k / GEMM kernels on their smallest routed shapes, BDC."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_11467_b200 as g
a = g.generate_matrix(g.MatrixSpec("random", 300, 300, seed=2), device=True)
r = g.gesdd(a)                                                     # cluster GEBD2 + two-phase LABRD
t = torch.randn(512, 512, dtype=torch.float64, device="cuda").t()
p_ = torch.randn(64, 512, dtype=torch.float64, device="cuda").t()
g.matmul_accumulate(-1.0, p_, False, p_, True, 1.0, t)             # rankk_tilec_kernel (K = 64)
big = torch.randn(9600, 300, dtype=torch.float64, device="cuda").t()
ya = torch.randn(128, 300, dtype=torch.float64, device="cuda").t()
w_ = torch.zeros(9600, 128, dtype=torch.float64, device="cuda").t()
g.matmul_accumulate(1.0, ya, True, big, False, 0.0, w_)            # dgemm_ws_kernel
d = np.random.default_rng(0).standard_normal(200); e = np.random.default_rng(1).standard_normal(199)
g.bdsdc(g.BidiagonalProblem(d, e))
torch.cuda.synchronize()
print("race_small done", float(r.sigma[0]))
