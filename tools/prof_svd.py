"""Phase profile of the GPU SVD at a given size (dev tool)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_11467_b200 as g
m = int(sys.argv[1]); n = int(sys.argv[2]) if len(sys.argv) > 2 else m
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
a = torch.rand(n, m, dtype=torch.float64, device="cuda").t()
for r in range(reps):
    p = g.phase_profile(a)
    print(json.dumps({"m": m, "n": n, "total_s": p.total, **{k: round(v, 5) for k, v in p.phases}}), flush=True)
