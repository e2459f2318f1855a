"""GPU GEBRD vs the CPU oracle on a few shapes: max deviations (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2508_11467_b200 as g
import oracle

rng = np.random.default_rng(0)
shapes = [(70, 70, 32), (90, 50, 8), (300, 300, 32), (129, 100, 16), (40, 40, 64), (512, 512, 32),
          (1000, 600, 32), (600, 600, 32), (2048, 300, 32)]
for (m, n, nb) in shapes:
    a = rng.standard_normal((m, n))
    a1 = np.asfortranarray(a.copy()); a2 = np.asfortranarray(a.copy())
    f = g.gebrd_blocked(a1, nb)
    d, e, tq, tp = oracle.gebrd(a2, nb)
    print(f"gebrd {m}x{n} nb={nb}: d {np.max(np.abs(f.d - d)):.2e} e {np.max(np.abs(f.e - e)):.2e} "
          f"tauq {np.max(np.abs(f.tauq - tq)):.2e} taup {np.max(np.abs(f.taup - tp)):.2e} "
          f"packed {np.max(np.abs(a1 - a2)):.2e}", flush=True)
