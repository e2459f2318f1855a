"""One GEBRD (gebrd_blocked, nb = 32) of MatrixSpec('random', n, n, seed=2) on the GPU (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_11467_b200 as g
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a = g.generate_matrix(g.MatrixSpec("random", n, n, seed=2), device=True)
g.gebrd_blocked(a)
torch.cuda.synchronize()
