"""Batched 2048^2 SVD throughput vs concurrency (dev tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_11467_b200 as g
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
B = int(sys.argv[2]) if len(sys.argv) > 2 else 32
mats = [torch.rand(n, n, dtype=torch.float64, device="cuda").t() for _ in range(B)]
for conc in (1, 2, 4, 6, 8, 12):
    g.gesdd_batched(mats[:conc * 2], concurrency=conc)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    g.gesdd_batched(mats, concurrency=conc)
    torch.cuda.synchronize(); t = time.perf_counter() - t0
    print(f"n={n} B={B} conc={conc}: {t*1e3/B:.2f} ms/SVD, {B/t:.1f} SVD/s", flush=True)
