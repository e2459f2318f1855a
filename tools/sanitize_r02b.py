"""compute-sanitizer cases for the kernels changed in the last round-2 session:
two-phase LABRD reduce-scatters (labrd2 at 300^2 / 700^2), 16-wide panels
(gebrd 2400^2), batched ORMBR op(T) precompute (gesdd 700^2: 5 full CWY blocks
per side)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_11467_b200 as g
big = len(sys.argv) > 1 and sys.argv[1] == "big"
for n in (300, 700):
    a = g.generate_matrix(g.MatrixSpec("random", n, n, seed=2), device=True)
    r = g.gesdd(a)
    s = torch.linalg.svdvals(a)
    print(n, float((r.sigma - s).abs().max() / s[0]), flush=True)
if big:
    a = g.generate_matrix(g.MatrixSpec("random", 2400, 2400, seed=2), device=True)
    f = g.gebrd_blocked(a.clone())
    print("gebrd 2400 ok", float(f.d.abs().max()), flush=True)
print("done")
