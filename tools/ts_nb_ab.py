"""TS pre-step QR panel width A/B (dcsvd_debug_ts_qr_nb: 32 = options.qr_block, 64)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
lib = _lib.load_library()
a = g.generate_matrix(g.MatrixSpec("random", 65536, 1024, seed=3), device=True)
ref = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests/golden/c3_sigma.npz"))["sigma"]
for rep in range(2):
    for nb in (0, 64):
        lib.dcsvd_debug_ts_qr_nb(nb)
        g.gesdd(a)
        p = g.phase_profile(a)
        r = g.gesdd(a)
        err = float(np.max(np.abs(r.sigma.cpu().numpy() - ref)) / ref[0])
        print(json.dumps(dict(nb=nb, total=round(p.total * 1e3, 2), sig=err, **{k: round(v * 1e3, 2) for k, v in p.phases})), flush=True)
lib.dcsvd_debug_ts_qr_nb(0)
