"""C5-shaped batch (2048^2) throughput vs the GEBRD panel-width rule
(dcsvd_debug_labrd_halfwidth 0/1/2) and the concurrency.

Usage: python tools/c5_halfwidth_ab.py [n] [batch]
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_11467_b200 as g
from paper_2508_11467_b200 import _lib
lib = _lib.load_library()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 32
mats = [torch.rand(n, n, dtype=torch.float64, device="cuda").t() for _ in range(batch)]
for conc in (6, 8, 12):
    for mode in (0, 1, 2):
        lib.dcsvd_debug_labrd_halfwidth(mode, 0)
        g.gesdd_batched(mats, concurrency=conc)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(2):
            g.gesdd_batched(mats, concurrency=conc)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 2
        print(f"n {n} batch {batch} conc {conc:2d} halfwidth {mode}: {ms / batch:6.2f} ms/SVD", flush=True)
lib.dcsvd_debug_labrd_halfwidth(1, 0)
