"""C5-shaped batch (2048^2, 8 sub-contexts) throughput with a given library build.
Usage: python tools/c5_lib_ab.py LIBPATH [batch]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2508_11467_b200 import _lib
_lib.load_library(sys.argv[1])
import paper_2508_11467_b200 as g
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 64
mats = [g.generate_matrix(g.MatrixSpec("random", 2048, 2048, seed=1000 + i), device=True) for i in range(batch)]
g.gesdd_batched(mats); torch.cuda.synchronize()
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.gesdd_batched(mats); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print(f"{os.path.basename(sys.argv[1])}: {min(ts) / batch:.2f} ms/SVD ({batch * 1e3 / min(ts):.1f} SVD/s)", flush=True)
