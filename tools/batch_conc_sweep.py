"""C5-shaped batch throughput vs the number of concurrent sub-contexts.

Usage: python tools/batch_conc_sweep.py [n] [batch]
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_11467_b200 as g
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 16
mats = [torch.rand(n, n, dtype=torch.float64, device="cuda").t() for _ in range(batch)]
for conc in [int(x) for x in os.environ.get("CONCS", "2 4 6 8 12 16").split()]:
    g.gesdd_batched(mats, concurrency=conc)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(2):
        g.gesdd_batched(mats, concurrency=conc)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 2
    print(f"n {n} batch {batch} conc {conc:2d}: {ms:8.2f} ms/step  {ms / batch:6.2f} ms/SVD", flush=True)
