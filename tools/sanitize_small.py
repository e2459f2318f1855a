"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_11467_b200 as g
import oracle  # inputs only (test infrastructure)
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

# round-1 additions: two-phase LABRD panels, one-barrier GEQRF panel, side-stream
# back-transform, standalone merge stages, GPU harness
a = oracle.make_matrix("random", 300, 300, seed=2)
r = g.gesdd(a)                                    # two-phase LABRD + concurrent U / V^T back-transforms
a = oracle.make_matrix("random", 900, 90, seed=3)
r = g.gesdd(a)                                    # TS path: one-barrier GEQRF panel
d, z = np.array([0.0, 3.0, 1.0, 1.0, 2.0]), np.array([1.0, 0.5, 0.6, 0.8, 1e-20])
L = np.asfortranarray(np.random.default_rng(0).standard_normal((5, 5)))
R = np.asfortranarray(np.random.default_rng(1).standard_normal((6, 5)))
out = g.deflate(d, z, L, R, left_classes=np.array([0, 1, 1, 2, 2]), right_classes=np.array([3, 1, 1, 2, 2]))
prob = g.BidiagonalProblem(np.linspace(1, 2, 9), np.full(9, 0.3), True)
lp, rp, _, _ = g.split(prob)
dz = g.build_z(prob, g.bdsqr_base(lp), g.bdsqr_base(rp))
x = g.generate_matrix(g.MatrixSpec("logrand", 40, 30, 1e6, seed=1))
rep = g.accuracy(x, g.gesdd(x), reference_sigma=g.prescribed_singular_values("logrand", 30, 1e6, seed=1))
torch.cuda.synchronize()
print("sanitize_small round-1 additions ok", rep)

# round-2 additions: the TMA kernels (rank-k tile kernel with smem C, warp-specialized
# long-K GEMM with split-K, BDC gather4 merge products over the workspace stack)
t = torch.randn(1024, 1024, dtype=torch.float64, device="cuda").t()            # 1024^2 C
p_ = torch.randn(64, 1024, dtype=torch.float64, device="cuda").t()
q_ = torch.randn(64, 1024, dtype=torch.float64, device="cuda").t()
g.matmul_accumulate(-1.0, p_, False, q_, True, 1.0, t)                           # rankk_tilec_kernel, K = 64
y_ = torch.randn(128, 1024, dtype=torch.float64, device="cuda").t()
x_ = torch.randn(1024, 128, dtype=torch.float64, device="cuda").t()
g.matmul_accumulate(-1.0, y_, False, x_, False, 1.0, t)                          # rankk_tilec_kernel, K = 128
big = torch.randn(9600, 300, dtype=torch.float64, device="cuda").t()            # 300 x 9600
ya = torch.randn(128, 300, dtype=torch.float64, device="cuda").t()              # 300 x 128
w_ = torch.zeros(9600, 128, dtype=torch.float64, device="cuda").t()             # 128 x 9600
g.matmul_accumulate(1.0, ya, True, big, False, 0.0, w_)                         # dgemm_ws_kernel (TA), 150 tiles
a = g.generate_matrix(g.MatrixSpec("random", 1500, 1500, seed=5), device=True)
r = g.gesdd(a)                                    # ORMBR CWY split-K products (dgemm_ws), BDC gather4
print("round-2 done", float(r.sigma[0]))
