"""Per-segment timeline of the two-phase LABRD kernel (CTA 0's %globaltimer
marks, mean over the columns of the first panel; dev tool).
usage: python tools/labrd2_timeline.py n [n ...]"""
import sys, os, ctypes, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2508_11467_b200 as g
lib = g._lib.load_library()
for n in [int(x) for x in sys.argv[1:]]:
    a = torch.rand(n, n, dtype=torch.float64, device="cuda").t()
    g.gebrd_blocked(a.clone().t().contiguous().t())
    buf = torch.zeros(1024, dtype=torch.int64, device="cuda")
    lib.dcsvd_debug_labrd_tlog(ctypes.c_void_p(buf.data_ptr()))
    g.gebrd_blocked(a.clone().t().contiguous().t())
    lib.dcsvd_debug_labrd_variant.restype = ctypes.c_int
    t = buf.cpu().numpy().astype(np.float64)
    main = t[1:1 + 8 * 33].reshape(33, 8)
    det = t[600:600 + 8 * 33].reshape(33, 8)
    ks = list(range(2, 30))
    def m(f): return round(float(np.mean([f(k) for k in ks])) / 1e3, 3)
    seg = {
        "A_loads": m(lambda k: det[k, 0] - main[k, 0]), "A_larfg_u": m(lambda k: det[k, 1] - det[k, 0]),
        "A_x_c": m(lambda k: det[k, 2] - det[k, 1]), "A_blocksum": m(lambda k: main[k, 1] - det[k, 2]),
        "A_corr": m(lambda k: main[k, 2] - main[k, 1]), "A_gemv": m(lambda k: main[k, 3] - main[k, 2]),
        "A_barrier": m(lambda k: main[k, 4] - main[k, 3]),
        "B_loads": m(lambda k: det[k, 4] - main[k, 4]), "B_larfg": m(lambda k: det[k, 5] - det[k, 4]),
        "B_vyr": m(lambda k: det[k, 6] - det[k, 5]), "B_blocksum": m(lambda k: main[k, 5] - det[k, 6]),
        "B_corr": m(lambda k: main[k, 6] - main[k, 5]), "B_gemv": m(lambda k: main[k, 7] - main[k, 6]),
        "B_barrier": m(lambda k: main[k + 1, 0] - main[k, 7]),
        "column": m(lambda k: main[k + 1, 0] - main[k, 0]),
    }
    print(json.dumps({"n": n, "variant": lib.dcsvd_debug_labrd_variant(), "us": seg}), flush=True)
