"""One GEBRD of an n x n uniform matrix, then ONE bdsdc with vectors of its
bidiagonal (for ncu launch lists / captures of the BDC merge GEMMs)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_11467_b200 as g
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a = g.generate_matrix(g.MatrixSpec("random", n, n, seed=2), device=True)
f = g.gebrd_blocked(a)
torch.cuda.synchronize()
r = g.bdsdc(g.BidiagonalProblem(f.d, f.e))
torch.cuda.synchronize()
