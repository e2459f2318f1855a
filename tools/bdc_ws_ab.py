"""BDC merge products on the TMA GEMM (1) vs dgemm_kernel with gather (0):
bdsdc of the bidiagonal of an n x n uniform matrix; time, sigma/vector
agreement between the two paths, orthogonality of W."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
lib = _lib.load_library()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a = g.generate_matrix(g.MatrixSpec("random", n, n, seed=2), device=True)
f = g.gebrd_blocked(a)
prob = g.BidiagonalProblem(f.d, f.e)
res = {}
for w in (1, 0, 1):
    lib.dcsvd_debug_dgemm_ws(w)
    g.bdsdc(prob); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); r = g.bdsdc(prob); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    res[w] = r
    eye = torch.eye(n, dtype=torch.float64, device="cuda")
    orth = float(torch.linalg.matrix_norm(r.w.t() @ r.w - eye)) / n
    print(json.dumps(dict(ws=w, ms=round(min(ts), 3), orth_w=orth)), flush=True)
lib.dcsvd_debug_dgemm_ws(1)
print(json.dumps(dict(dvals_equal=bool(torch.equal(res[0].dvals, res[1].dvals)),
                      w_maxdiff=float((res[0].w - res[1].w).abs().max()), q_maxdiff=float((res[0].qfull - res[1].qfull).abs().max()))))
