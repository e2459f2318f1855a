"""BDC merge-GEMM flops / time and column-move bytes at n = 8192 (stats kinds 2/3; dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
n = 8192
a = torch.rand(n, n, dtype=torch.float64, device="cuda").t()
f = g.gebrd_blocked(a.clone().t().contiguous().t())
prob = g.BidiagonalProblem(f.d, f.e)
g.bdsdc(prob); torch.cuda.synchronize()
_lib.set_stats(True)
r = g.bdsdc(prob); torch.cuda.synchronize()
ms, fl, nl = _lib.get_stats(2)
mv_ms, mv_b, _ = _lib.get_stats(3)
_lib.set_stats(False)
print(f"BDC merge GEMMs: {fl/1e12:.3f} TFLOP in {ms:.2f} ms -> {fl/ms/1e9:.1f} TF/s, {nl} launches; moves {mv_b/1e9:.2f} GB in {mv_ms:.2f} ms")
