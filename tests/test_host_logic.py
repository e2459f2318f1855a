"""CPU-only tests of the host layer: library loading/exports, option
validation, containers, and the multi-process batch sharding (gloo)."""

import ctypes
import os
import re
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    text = open(os.path.join(ROOT, "include", "dcsvd_b200.h")).read()
    return sorted(set(re.findall(r"\b(dcsvd_[a-z_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2508_11467_b200 import _lib
    from paper_2508_11467_b200.build import build

    build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = _header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTED)
    assert lib.dcsvd_version() == 100


def test_no_cpu_fallback_without_gpu():
    import paper_2508_11467_b200 as g

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(RuntimeError, match="CUDA"):
        g.gesdd(np.eye(3))


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2508_11467_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            src = open(os.path.join(pkg, f)).read()
            assert "import oracle" not in src and "from oracle" not in src, f


def test_svd_options_validation():
    from paper_2508_11467_b200 import SVDOptions

    SVDOptions()
    for kw in ({"bidiag_block": 0}, {"leaf_size": 0}, {"ts_crossover": 0.5}, {"deflation_multiple": 0.0}):
        with pytest.raises(ValueError):
            SVDOptions(**kw)
    o = SVDOptions(want_vectors=False)._native()
    assert o.want_vectors == 0 and o.bidiag_block == 32 and o.leaf_size == 32


def test_bidiagonal_problem_container():
    from paper_2508_11467_b200 import BidiagonalProblem

    p = BidiagonalProblem([1.0, 2.0], [3.0])
    assert p.e.size == 2 and p.e[1] == 0.0 and p.ncols == 2
    p = BidiagonalProblem([1.0, 2.0], [3.0, 4.0], bordered=True)
    assert p.ncols == 3
    np.testing.assert_array_equal(p.dense(), [[1.0, 3.0, 0.0], [0.0, 2.0, 4.0]])
    with pytest.raises(ValueError):
        BidiagonalProblem([1.0, 2.0, 3.0], [1.0])


def test_shard_range_partitions():
    from paper_2508_11467_b200.batch import shard_range

    for total in (0, 1, 7, 512):
        for ws in (1, 2, 4, 8):
            got = [shard_range(total, ws, r) for r in range(ws)]
            assert got[0][0] == 0 and got[-1][1] == total
            for (a, b), (c, d) in zip(got, got[1:]):
                assert b == c
            sizes = [b - a for a, b in got]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, ws, port, q):
    import torch.distributed as dist

    from paper_2508_11467_b200.batch import gather_to_owner, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    lo, hi = shard_range(10, ws, rank)
    # stand-in results: (sigma, U, Vt) tensors tagged with the global index
    local = [(torch.full((3,), float(i)), torch.eye(3) * i, torch.eye(3)) for i in range(lo, hi)]
    full = gather_to_owner(local, dst=0)
    if rank == 0:
        q.put([float(item[0][0]) for item in full])
    dist.barrier()
    dist.destroy_process_group()


def test_batch_gather_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    order = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert order == [float(i) for i in range(10)]


def _gloo_sigma_worker(rank, ws, port, q):
    import torch.distributed as dist

    from paper_2508_11467_b200.batch import gather_sigma, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    total, k = 11, 4
    lo, hi = shard_range(total, ws, rank)
    local = torch.stack([torch.arange(k, dtype=torch.float64) + 10.0 * i for i in range(lo, hi)])
    full = gather_sigma(local, total)
    q.put((rank, full.numpy().tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("ws", [2, 3])
def test_gather_sigma_gloo(ws):
    """batch.gather_sigma (the C5 sigma gather) at world size 2 and 3 with
    uneven shards: every rank gets the rows in global batch order."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_sigma_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(ws)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = [[10.0 * i + j for j in range(4)] for i in range(11)]
    for _, rows in got:
        assert rows == want


def test_bench_spawns_ranks_for_gpus_flag(monkeypatch):
    """`bench.py --gpus N` outside torchrun re-launches itself under
    torch.distributed.run with N ranks on 127.0.0.1 (bench.maybe_spawn)."""
    import sys

    sys.path.insert(0, ROOT)
    import bench

    calls = []
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--workload", "c5"])
    args = type("A", (), {"gpus": 4})()
    assert bench.maybe_spawn(args) == 0
    cmd = calls[0]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1" and cmd[-2:] == ["--workload", "c5"]
    monkeypatch.setenv("WORLD_SIZE", "4")
    assert bench.maybe_spawn(args) is None


# the `dcsvd` shim: reference module layout -> this package
REFERENCE_ALL = (  # pkg/src/dcsvd/__init__.py:87-129
    "AccuracyReport BidiagonalFactorization BidiagonalProblem CompactWYBlock ConvergenceError DeflationOutcome "
    "GivensRotation HouseholderReflector MatrixSpec PhaseProfile QRFactorization ReflectorSequence SVDOptions "
    "SVDResult SecularRoots SecularSystem SubproblemSVD accuracy apply_block_reflector_left "
    "apply_block_reflector_right as_dense bdsdc bdsqr_base build_tinv build_z cli_main column_reflectors deflate "
    "dense_matrix gebrd_blocked gebrd_unblocked generate_matrix geqrf_blocked geqrf_panel gesdd givens_generate "
    "householder_generate labrd_panel matmul_accumulate matvec_accumulate merge_vectors orgqr ormlq_like ormqr_like "
    "phase_profile prescribed_singular_values read_matrix recompute_z row_reflectors secular_vectors "
    "solve_all_roots solve_secular split triangular_solve write_matrix").split()


def test_dcsvd_shim_layout():
    import importlib
    import os
    import sys

    shim = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "shim")
    sys.path.insert(0, shim)
    try:
        d = importlib.import_module("dcsvd")
        for name in REFERENCE_ALL:
            assert hasattr(d, name), name
        for mod, names in (("driver", "gesdd phase_profile SVDOptions SVDResult PhaseProfile PHASE_NAMES"),
                           ("bdc", "bdsdc deflate build_z merge_vectors split bdsqr_base"),
                           ("bidiag", "gebrd_blocked labrd_panel gebrd_unblocked"),
                           ("qrblock", "geqrf_blocked orgqr build_tinv"),
                           ("backtransform", "ormqr_like ormlq_like column_reflectors row_reflectors"),
                           ("densecore", "matmul_accumulate householder_generate ConvergenceError"),
                           ("harness", "MatrixSpec generate_matrix accuracy read_matrix write_matrix cli_main")):
            m = importlib.import_module("dcsvd." + mod)
            for name in names.split():
                assert hasattr(m, name), (mod, name)
        import paper_2508_11467_b200 as g
        assert d.gesdd is g.gesdd and d.bdc.deflate is g.deflate
    finally:
        sys.path.remove(shim)
        for k in [k for k in sys.modules if k == "dcsvd" or k.startswith("dcsvd.")]:
            del sys.modules[k]
