"""One C3 gesdd (65536 x 1024 MatrixSpec('random', seed=3)) after a warm-up, for launch lists."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_11467_b200 as g
a = g.generate_matrix(g.MatrixSpec("random", 65536, 1024, seed=3), device=True)
g.gesdd(a)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
g.gesdd(a)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
