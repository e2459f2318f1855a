"""Run GPU GEBRD once at n (default 8192) for profiling."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2508_11467_b200 as g
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a = torch.rand(n, n, dtype=torch.float64, device="cuda").t()
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    b = a.clone().t().contiguous().t()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); f = g.gebrd_blocked(b); e.record(); torch.cuda.synchronize()
    print("gebrd", n, s.elapsed_time(e), "ms", flush=True)
