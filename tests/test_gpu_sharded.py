"""Config C5 sharding on the GPU: two ranks run
``batch.batched_svd_sharded`` on their contiguous slices of a batch of
MatrixSpec('random', 2048, 2048, seed=1000+i) inputs, gather sigma with
``batch.gather_sigma``, and rank 0 checks every item against the REAL
reference's sigma on the same bytes (tests/golden/c5_sigma.npz) within the
north-star 1e-12 n.  Both ranks share cuda:0 over a gloo group (NCCL refuses
two ranks on one device); on an 8-GPU box bench.py uses NCCL, one rank per GPU."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, total, q):
    import torch
    import torch.distributed as dist

    import paper_2508_11467_b200 as g
    from paper_2508_11467_b200.batch import batched_svd_sharded, gather_sigma

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=ws)

    def make(i):
        return g.generate_matrix(g.MatrixSpec("random", 2048, 2048, seed=1000 + i), device=True)

    res, _ = batched_svd_sharded(make, total)
    local = torch.stack([r.sigma for r in res])
    # residual / orthogonality of this rank's first item on the device
    rep = g.accuracy(make(dist.get_rank() * (total // ws)), res[0])
    full = gather_sigma(local, total)
    q.put((rank, full.cpu().numpy(), rep.e_svd / 2048, rep.orth_u / 2048, rep.orth_v / 2048))
    dist.barrier()
    dist.destroy_process_group()


def test_c5_sharded_two_ranks(cuda):
    p = os.path.join(GOLDEN, "c5_sigma.npz")
    if not os.path.exists(p):
        pytest.skip("c5_sigma.npz not generated")
    ref = np.load(p)["sigma"]
    total, ws = 10, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, total, q)) for r in range(ws)]
    for pr in procs:
        pr.start()
    got = sorted([q.get(timeout=600) for _ in range(ws)], key=lambda x: x[0])
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    for rank, full, resid, ou, ov in got:
        assert full.shape == (total, 2048)
        err = np.max(np.abs(full - ref[:total]) / ref[:total, :1])
        assert err <= 1e-12 * 2048, (rank, err)
        assert resid <= 1e-14 and ou <= 1e-14 and ov <= 1e-14
    assert np.array_equal(got[0][1], got[1][1])
