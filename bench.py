"""Benchmark: fp64 SVD (U, Sigma, V) on B200 -- BASELINE.json metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c1|c3|c4|c5]
                    [--impl ours|reference]

One step = one full economy SVD with vectors of the workload's input (C2:
the 8192 x 8192 uniform(0,1) matrix of MatrixSpec("random", 8192, 8192,
seed=2)).  `value` = GFLOP/s on the 28/3 n^3 convention with
the input resident in HBM (512 MiB > L2, so no flush is needed); `e2e` = the
same through the public API from pinned host memory with the results copied
back.  Multi-GPU (torchrun): the single SVD does not shard, so
each rank runs a replica ("scaling": "weak"; value = total flops / max time).
`--impl reference` times the CPU oracle port (oracle/, the reference
algorithm restated in numpy, bitwise-equal to the reference on the golden
vectors) on a bounded sample of the workload on this host.
"""

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def flops_square(n):
    return 28.0 / 3.0 * n ** 3


def flops_ts(m, n):
    return 6.0 * m * n * n + 8.0 * n ** 3


WORKLOADS = {
    # name: (m, n, seed, description)
    "c1": (1024, 1024, 1, "C1 random 1024x1024 fp64 full SVD with U,S,V"),
    "c2": (8192, 8192, 2, "C2 square 8192x8192 fp64 full SVD with U,S,V (headline)"),
    "c3": (65536, 1024, 3, "C3 tall-skinny 65536x1024 fp64 SVD (GEQRF pre-step + GEBRD + BDC)"),
    "c5": (2048, 2048, 1000, "C5 batch of independent 2048x2048 fp64 SVDs"),
    "c4": (16384, 16384, 4, "C4 bidiagonal BDC only, n=16384, clustered singular values (heavy deflation), with vectors"),
}


def workload_flops(m, n):
    k, M = min(m, n), max(m, n)
    if M >= 5.0 / 3.0 * k and M > k:
        return flops_ts(M, k)
    return flops_square(k)


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
            return self
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.1)

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=1.0)

    def summary(self):
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh), "measured"
    return {"hbm_gbs": 6650.0}, "fallback"


def load_ncu_traffic():
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(p):
        try:
            with open(p) as fh:
                return json.load(fh)
        except Exception:
            return None
    return None


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def ref_kind():
    """"reference" when the unmodified reference package is installed in
    baseline/_ref (pip --target), else the oracle
    port ("port")."""
    return "reference" if os.path.isfile(os.path.join(REF_DIR, "dcsvd", "driver.py")) else "port"


def cpu_sample(n, threads, seed=1, m=None, values_only=False):
    """Time one CPU SVD (the real reference's `dcsvd.gesdd` from baseline/_ref
    when installed, else the oracle port) of MatrixSpec('random', m, n, seed)
    in a subprocess with `threads` BLAS threads; returns seconds."""
    m = n if m is None else m
    if ref_kind() == "reference":
        code = (
            "import sys,time; sys.path.insert(0, %r); import dcsvd;"
            "a=dcsvd.generate_matrix(dcsvd.MatrixSpec('random',%d,%d,seed=%d)); t=time.perf_counter();"
            "dcsvd.gesdd(a, dcsvd.SVDOptions(want_vectors=%r)); print(time.perf_counter()-t)"
            % (REF_DIR, m, n, seed, not values_only)
        )
    else:
        code = (
            "import sys,time,numpy as np; sys.path.insert(0, %r); import oracle;"
            "a=oracle.make_matrix('random',%d,%d,seed=%d); t=time.perf_counter(); oracle.svd(a);"
            "print(time.perf_counter()-t)" % (ROOT, m, n, seed)
        )
    env = dict(os.environ)
    for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        env[k] = str(threads)
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=3600)
    if out.returncode != 0:
        raise RuntimeError(out.stderr)
    return float(out.stdout.strip().splitlines()[-1])


def cpu_parallel(n, procs, seed0):
    """`procs` concurrent single-thread CPU SVDs of n x n (seeds seed0..):
    the SURVEY 8(d) C5 plan (one BLAS thread per process, one process per
    core).  Returns the wall seconds of the slowest."""
    import concurrent.futures as cf
    with cf.ThreadPoolExecutor(max_workers=procs) as ex:
        ts = list(ex.map(lambda i: cpu_sample(n, 1, seed=seed0 + i), range(procs)))
    return max(ts)


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def free_port():
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return port


def maybe_spawn(args):
    """`python bench.py --gpus N` (N > 1) outside torchrun: re-launch this
    script under torch.distributed.run with N ranks (one process per GPU,
    rendezvous on 127.0.0.1) and return its exit code."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    print("[bench] spawning %d ranks: %s" % (args.gpus, " ".join(cmd)), file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def init_dist(torch, dist, ws, rank, local):
    """One process per GPU; NCCL process group when ws > 1 (logged).  More
    ranks than GPUs (a world-size-2 check on a 1-GPU box) share GPUs
    round-robin over a gloo group: NCCL refuses two ranks on one device."""
    ndev = torch.cuda.device_count()
    dev = local % max(ndev, 1)
    torch.cuda.set_device(dev)
    if ws > 1:
        if ws <= ndev:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
            nccl = ".".join(map(str, torch.cuda.nccl.version()))
            print(f"[bench] rank {rank}/{ws}: NCCL {nccl} process group initialised on cuda:{dev}",
                  file=sys.stderr, flush=True)
        else:
            dist.init_process_group("gloo")
            print(f"[bench] rank {rank}/{ws}: {ws} ranks > {ndev} GPU(s): gloo process group, ranks share "
                  f"cuda:{dev}", file=sys.stderr, flush=True)
    return dev


def max_over_ranks(torch, dist, ws, local, v):
    if ws <= 1:
        return v
    on_gpu = dist.get_backend() == "nccl"
    t = torch.tensor([v], dtype=torch.float64, device=f"cuda:{local}" if on_gpu else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def load_sigma_fixture(tag):
    """Reference sigma on the same Philox input bytes (tests/golden/make_large_sigma.py)."""
    p = os.path.join(ROOT, "tests", "golden", f"{tag}_sigma.npz")
    if not os.path.exists(p):
        return None
    return np.load(p)


def sigma_rel(sig, ref):
    """max_i |sigma_i - sigma_i^ref| / sigma_max (north-star check, tolerance 1e-12 n)."""
    sig = np.asarray(sig, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(sig - ref)) / ref[0])


def run_reference(args):
    """--impl reference: the reference's own CPU implementation (the unmodified
    `dcsvd` package in baseline/_ref when installed, else the oracle port) on
    this host's cores, on a bounded sample of the workload per step."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    m, n, seed, desc = WORKLOADS[args.workload]
    cores = host_cores()
    kind = ref_kind()
    who = "reference dcsvd 0.1.0 (baseline/_ref)" if kind == "reference" else "oracle port (numpy restatement)"
    steps = max(args.steps, 1)
    if args.workload == "c5":
        # full-size C5 items, one single-thread process per core
        procs = max(1, min(cores, 64))
        for _ in range(args.warmup):
            cpu_sample(128, 1)
        times = [cpu_parallel(n, procs, 1000 + 1000 * s_) for s_ in range(steps)]
        t = float(np.mean(times))
        svd_s = procs / t
        val, unit = svd_s, "SVD/s"
        metric = "batched fp64 SVD (U,S,V) throughput, 2048x2048 items"
        sample = (f"{who}: {procs} concurrent processes x 1 BLAS thread, one full 2048^2 SVD each per step "
                  f"(seeds 1000+i); 512 items extrapolate to {512 / svd_s:.0f} s")
        cfg = {"workload": desc, "m": m, "n": n, "items_per_step": procs}
        ms = t * 1e3
        hib = True
    elif args.workload == "c4":
        # BDC only on the C4 fixture (n = 16384) takes ~57 s with vectors: time
        # the reference bdsdc on a leading n_s slice of the same bidiagonal
        n_s = 4096
        fx = os.path.join(ROOT, "tests", "golden", "c4_n16384.npz")
        if kind == "reference":
            code = ("import sys,time,numpy as np; sys.path.insert(0,%r); import dcsvd;"
                    "z=np.load(%r); p=dcsvd.BidiagonalProblem(z['d'][:%d].copy(), z['e'][:%d].copy());"
                    "t=time.perf_counter(); dcsvd.bdsdc(p); print(time.perf_counter()-t)"
                    % (REF_DIR, fx, n_s, n_s - 1))
        else:
            code = ("import sys,time,numpy as np; sys.path.insert(0,%r); import oracle;"
                    "z=np.load(%r); p=oracle.Bidiag(z['d'][:%d].copy(), z['e'][:%d].copy());"
                    "t=time.perf_counter(); oracle.bdc(p); print(time.perf_counter()-t)"
                    % (ROOT, fx, n_s, n_s - 1))
        env = dict(os.environ, OPENBLAS_NUM_THREADS=str(cores), PYTHONDONTWRITEBYTECODE="1")
        times = []
        for i in range(args.warmup + steps):
            out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=3600)
            if out.returncode != 0:
                raise RuntimeError(out.stderr)
            if i >= args.warmup:
                times.append(float(out.stdout.strip().splitlines()[-1]))
        t = float(np.mean(times))
        val, unit, ms, hib = t, "s", t * 1e3, False
        metric = "BDC stage time (bdsdc with vectors), seconds"
        sample = (f"{who} bdsdc with vectors on the leading {n_s} x {n_s} block of the C4 fixture bidiagonal, "
                  f"{cores} BLAS threads; the full n=16384 fixture takes 57.2 s with vectors (BASELINE.md)")
        cfg = {"workload": desc, "n": n, "sample_n": n_s}
    else:
        # bounded sample with the workload's shape: square n_s (C1/C2) or a
        # 64:1 tall-skinny m_s x n_s (C3) sized so K + W steps take minutes
        if args.workload == "c3":
            n_s, m_s = 256, 256 * 64
        else:
            n_s = int(min(n, 2048 * (150.0 / (21.0 * steps)) ** (1.0 / 3.0)) // 128 * 128)
            n_s = max(n_s, 256)
            m_s = n_s
        for _ in range(args.warmup):
            cpu_sample(256, cores)
        times = [cpu_sample(n_s, cores, m=m_s) for _ in range(steps)]
        t = float(np.mean(times))
        val, unit, ms, hib = workload_flops(m_s, n_s) / t / 1e9, "GFLOP/s", t * 1e3, True
        metric = "fp64 SVD (U,S,V) GFLOP/s (28/3 n^3 convention)"
        sample = (f"{who}, {cores} BLAS threads, full SVD of MatrixSpec('random',{m_s},{n_s}) per step; "
                  "the full C2 took 563.4 s on a B200 box's 16 host cores (profiles/ref_fullsize_r02.md)")
        cfg = {"workload": desc, "m": m, "n": n, "sample_m": m_s, "sample_n": n_s}
    line = {
        "impl": "reference", "metric": metric, "value": val,
        "unit": unit, "n_gpus": ws, "steps": steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": hib, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfg,
        "cpu_baseline": {"value": val, "unit": unit, "cores": cores if args.workload != "c5" else cfg["items_per_step"],
                         "kind": kind, "sample": sample},
        "e2e": {"value": val, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_c4(args, dcs, _lib, torch, dist, ws, rank, local):
    """BDC-only workload on the committed C4 fixture (tests/golden/c4_n16384.npz)."""
    z = np.load(os.path.join(ROOT, "tests", "golden", "c4_n16384.npz"))
    n = z["d"].size
    d = torch.from_numpy(z["d"]).to(f"cuda:{local}")
    e = torch.from_numpy(z["e"]).to(f"cuda:{local}")
    prob = dcs.BidiagonalProblem(d, e)
    F = 8.0 / 3.0 * n ** 3
    for _ in range(args.warmup):
        dcs.bdsdc(prob)
    torch.cuda.synchronize()
    s, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = _lib.launch_count()
    with ClockSampler(local) as clk:  # timed pass: no per-kernel instrumentation
        s.record()
        for _ in range(args.steps):
            r = dcs.bdsdc(prob)
        e1.record()
        torch.cuda.synchronize()
    t_ms = s.elapsed_time(e1) / args.steps
    l1 = _lib.launch_count()
    _lib.set_stats(True)  # separate instrumented pass for the per-family times
    for _ in range(args.steps):
        r = dcs.bdsdc(prob)
    torch.cuda.synchronize()
    g_ms, g_flops, g_n = _lib.get_stats(2)
    mv_ms, mv_bytes, mv_n = _lib.get_stats(3)
    _lib.set_stats(False)
    peaks, _ = load_peaks()
    dmma_peak = 148 * 128 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12
    g_ach = g_flops / (g_ms * 1e-3) / 1e12 if g_ms > 0 else None
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    mv_ach = mv_bytes / (mv_ms * 1e-3) / 1e9 if mv_ms > 0 else None
    roof_gemm = {
        "kernel": "dgemm_kernel, grouped BDC merge products (gathered columns, device descriptors)",
        "bound": "tensor", "achieved": g_ach, "peak": dmma_peak, "unit": "TFLOP/s",
        "frac": (g_ach / dmma_peak) if g_ach else None,
        "peak_source": "FP64 DMMA peak 148 SMs x 128 flop/clk at sm_max_mhz (MEASURED_PEAKS.json)",
        "traffic": None,
        "algorithmic_flops_per_step": g_flops / max(args.steps, 1),
        "launches_per_step": g_n / max(args.steps, 1),
        "share_of_step": (g_ms / args.steps) / t_ms if t_ms > 0 else None,
        "note": "instrumented pass of the same K steps after the timed pass; flops = sum 2 m n k of the structured merge products, counted on the device from the "
                "post-deflation sizes; heavy deflation leaves them small",
    }
    roof_moves = {
        "kernel": "bdc_defl_copy_kernel + bdc_copyback_kernel (deflated W/Q columns into place, node blocks back)",
        "bound": "hbm", "achieved": mv_ach, "peak": hbm, "unit": "GB/s",
        "frac": (mv_ach / hbm) if mv_ach else None,
        "peak_source": "MEASURED_PEAKS.json hbm_gbs",
        "traffic": None,
        "algorithmic_bytes_per_step": mv_bytes / max(args.steps, 1),
        "launches_per_step": mv_n / max(args.steps, 1),
        "share_of_step": (mv_ms / args.steps) / t_ms if t_ms > 0 else None,
        "note": "instrumented pass of the same K steps after the timed pass; bytes = 16 x rows x columns moved (read + write; deflated-column counts from the device); the "
                "sequential deflation scan (bdc_prep_kernel, latency-bound) is the other large share",
    }
    roof_c4 = (roof_moves, roof_gemm) if mv_ms >= g_ms else (roof_gemm, roof_moves)
    vals = r.dvals.cpu().numpy()
    w = r.w
    gram = _lib.colmajor_empty(n, n)
    gram.copy_(torch.eye(n, dtype=torch.float64, device=w.device))
    dcs.matmul_accumulate(1.0, w, True, w, False, -1.0, gram)  # W^T W - I with the DMMA GEMM
    orth_w = float(gram.norm().item()) / n
    # --- e2e: host d/e (pinned) -> bdsdc through the public API -> dvals, W, Q back to pinned host
    hd = torch.from_numpy(z["d"]).pin_memory()
    he = torch.from_numpy(z["e"]).pin_memory()
    out_d = torch.empty(n, dtype=torch.float64).pin_memory()
    out_w = torch.empty(r.w.numel(), dtype=torch.float64).pin_memory()
    out_q = torch.empty(r.qfull.numel(), dtype=torch.float64).pin_memory()
    h2d = (hd.numel() + he.numel()) * 8
    d2h = (out_d.numel() + out_w.numel() + out_q.numel()) * 8

    def e2e_step():
        pr = dcs.BidiagonalProblem(hd.to(f"cuda:{local}", non_blocking=True),
                                   he.to(f"cuda:{local}", non_blocking=True))
        rr = dcs.bdsdc(pr)
        out_d.copy_(rr.dvals, non_blocking=True)
        out_w.copy_(rr.w.t().reshape(-1), non_blocking=True)
        out_q.copy_(rr.qfull.t().reshape(-1), non_blocking=True)

    e2e_step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.record()
    for _ in range(args.e2e_steps):
        e2e_step()
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = max(s.elapsed_time(e1), (time.perf_counter() - t0) * 1e3) / args.e2e_steps
    t0 = time.perf_counter()
    rv = dcs.bdsdc(prob, want_vectors=False)
    torch.cuda.synchronize()
    t_vo = time.perf_counter() - t0
    line = {
        "metric": "BDC stage time (bdsdc with vectors), seconds", "value": t_ms * 1e-3,
        "unit": "s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms,
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "executed_merge_gemm_flops": g_flops / max(args.steps, 1),
        "note": "heavy deflation: the nominal 8/3 n^3 = %.3g flop is not executed; the merge GEMMs run the "
                "executed_merge_gemm_flops count" % F,
        "data": "C4 fixture tests/golden/c4_n16384.npz (LAPACK dgebrd of U diag(sigma) V^T, 8 clusters)",
        "config": {"workload": WORKLOADS["c4"][3], "n": n},
        "accuracy": {"max_abs_sigma_vs_reference": float(np.max(np.abs(vals - z["sigma_ref"]))),
                     "max_abs_sigma_vs_prescribed": float(np.max(np.abs(vals - z["sigma_prescribed"]))),
                     "orth_w_scaled": orth_w,
                     "values_only_bitwise_equal": bool(np.array_equal(rv.dvals.cpu().numpy(), vals))},
        "values_only_seconds": t_vo,
        "gpu_launches": int((l1 - l0) // max(args.steps, 1)),
        "roofline": roof_c4[0],
        "roofline_secondary": roof_c4[1],
        "clocks": clk.summary(),
        "e2e": {"value": e2e_ms * 1e-3, "unit": "s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms},
        "reference_full_size": {"seconds_with_vectors": 57.2, "seconds_values_only": float(z["ref_seconds_values_only"]),
                                "where": "build container, 7 BLAS threads (BASELINE.md §2; fixture creation)"},
    }
    if not args.no_cpu_baseline and ws == 1:
        n_s, cores = 4096, host_cores()
        kind = ref_kind()
        fx = os.path.join(ROOT, "tests", "golden", "c4_n16384.npz")
        if kind == "reference":
            code = ("import sys,time,numpy as np; sys.path.insert(0,%r); import dcsvd;"
                    "z=np.load(%r); p=dcsvd.BidiagonalProblem(z['d'][:%d].copy(), z['e'][:%d].copy());"
                    "t=time.perf_counter(); dcsvd.bdsdc(p); print(time.perf_counter()-t)" % (REF_DIR, fx, n_s, n_s - 1))
        else:
            code = ("import sys,time,numpy as np; sys.path.insert(0,%r); import oracle;"
                    "z=np.load(%r); p=oracle.Bidiag(z['d'][:%d].copy(), z['e'][:%d].copy());"
                    "t=time.perf_counter(); oracle.bdc(p); print(time.perf_counter()-t)" % (ROOT, fx, n_s, n_s - 1))
        env = dict(os.environ, OPENBLAS_NUM_THREADS=str(cores), PYTHONDONTWRITEBYTECODE="1")
        out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=1800)
        if out.returncode == 0:
            t_cpu = float(out.stdout.strip().splitlines()[-1])
            line["cpu_baseline"] = {"value": t_cpu, "unit": "s", "cores": cores, "kind": kind,
                                    "sample": f"bdsdc with vectors on the leading {n_s}x{n_s} block of the C4 "
                                              f"fixture bidiagonal ({kind}), {cores} BLAS threads; the full "
                                              "n=16384 fixture: 57.2 s with vectors (reference_full_size)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--batch", type=int, default=16, help="C5: matrices per GPU per step")
    ap.add_argument("--c5-total", type=int, default=512, help="C5: matrices in the whole job (sharded over ranks)")
    args = ap.parse_args()
    rc = maybe_spawn(args)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    local = init_dist(torch, dist, ws, rank, local)
    import paper_2508_11467_b200 as dcs
    from paper_2508_11467_b200 import _lib

    m, n, seed, desc = WORKLOADS[args.workload]
    if args.workload == "c4":
        return run_c4(args, dcs, _lib, torch, dist, ws, rank, local)
    k = min(m, n)
    c5 = args.workload == "c5"
    if c5:
        # BASELINE config 5: c5_total independent SVDs, contiguous shards per
        # rank (batch.shard_range), no data-path collective
        from paper_2508_11467_b200.batch import gather_sigma, shard_range
        lo, hi = shard_range(args.c5_total, ws, rank)
        seeds = [seed + i for i in range(lo, hi)]
    else:
        lo, hi, seeds = 0, 1, [seed]  # single SVD: every rank runs a replica
    batch = len(seeds)
    # inputs: MatrixSpec('random', m, n, seed) bytes from the GPU Philox
    # (bit-identical to harness._Stream), mirrored once into pinned host
    # memory for the end-to-end pass
    dev_inputs, host = [], []
    for s_ in seeds:
        a = dcs.generate_matrix(dcs.MatrixSpec("random", m, n, seed=s_), device=True)
        dev_inputs.append(a)
        h = torch.empty((n, m), dtype=torch.float64).pin_memory()  # (n, m) row-major == A col-major
        h.copy_(a.t())
        host.append(h)
    F = workload_flops(m, n) * batch

    def step():
        if not c5:
            return dcs.gesdd(dev_inputs[0])
        return dcs.gesdd_batched(dev_inputs)

    stream = torch.cuda.current_stream()

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    # timed pass: no per-kernel instrumentation inside it
    l0 = _lib.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        barrier()
    launches = (_lib.launch_count() - l0) // max(args.steps, 1)
    t_ms = ev0.elapsed_time(ev1) / args.steps
    # separate instrumented pass (same K steps) for the per-family kernel times:
    # CUDA events around each launch on its own stream (dcsvd_set_stats)
    _lib.set_stats(True)
    for _ in range(args.steps):
        step()
    barrier()
    lab_ms, lab_bytes, lab_n = _lib.get_stats(0)
    gem_ms, gem_flops, gem_n = _lib.get_stats(1)
    bdc_ms, bdc_flops, bdc_n = _lib.get_stats(2)  # BDC merge GEMMs (device-counted flops)
    gem_ms, gem_flops, gem_n = gem_ms + bdc_ms, gem_flops + bdc_flops, gem_n + bdc_n
    lib = _lib.load_library()
    lib.dcsvd_debug_batch_streams.restype = ctypes.c_int
    streams = max(1, lib.dcsvd_debug_batch_streams(_lib.handle()))
    _lib.set_stats(False)
    t_ms = max_over_ranks(torch, dist, ws, local, t_ms)
    value = F * ws / (t_ms * 1e-3) / 1e9

    # --- e2e through the public numpy-free API with pinned host buffers
    out_s = torch.empty(k, dtype=torch.float64).pin_memory()
    out_u = torch.empty((k, m), dtype=torch.float64).pin_memory()
    out_vt = torch.empty((n, k), dtype=torch.float64).pin_memory()
    h2d = d2h = 0

    def e2e_step():
        nonlocal h2d, d2h
        h2d = d2h = 0
        devs = []
        for hb in host:
            devs.append(hb.to(f"cuda:{local}", non_blocking=True).t())
            h2d += hb.numel() * 8
        rs = dcs.gesdd_batched(devs) if c5 else [dcs.gesdd(devs[0])]
        for r in rs:
            out_s.copy_(r.sigma, non_blocking=True)
            out_u.copy_(r.u.t(), non_blocking=True)
            out_vt.copy_(r.vt.t(), non_blocking=True)
            d2h += (out_s.numel() + out_u.numel() + out_vt.numel()) * 8

    e2e_step()
    barrier()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.e2e_steps):
        e2e_step()
    e1.record(stream)
    barrier()
    e2e_ms = max(e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3) / args.e2e_steps
    e2e_ms = max_over_ranks(torch, dist, ws, local, e2e_ms)
    e2e_value = F * ws / (e2e_ms * 1e-3) / 1e9

    # --- accuracy of the last device result on this rank (north-star checks),
    # products and norms on the GPU through the library (harness.accuracy)
    r = dcs.gesdd(dev_inputs[0])
    rep = dcs.accuracy(dev_inputs[0], r)
    resid = rep.e_svd / max(m, n)
    orth_u = rep.orth_u / k
    orth_v = rep.orth_v / k
    fx = load_sigma_fixture(args.workload)
    sig_items = 1
    if c5:
        # sigma of the whole sharded batch gathered to every rank (NCCL
        # all-gather, off the timed path), compared with the reference on the
        # fixture's seeds
        rs = dcs.gesdd_batched(dev_inputs, dcs.SVDOptions(want_vectors=False))
        full = gather_sigma(torch.stack([x.sigma for x in rs]), args.c5_total).cpu().numpy()
        del rs
        sig_rel, sig_items = None, 0
        if fx is not None:
            cnt = min(len(fx["sigma"]), args.c5_total)
            sig_rel = max(sigma_rel(full[i], fx["sigma"][i]) for i in range(cnt))
            sig_items = cnt
    else:
        sig_rel = sigma_rel(r.sigma.cpu().numpy(), fx["sigma"]) if fx is not None else None
    prof = dcs.phase_profile(dev_inputs[0])

    if rank != 0:
        if ws > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0
    peaks, peak_kind = load_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    achieved = (lab_bytes / (lab_ms * 1e-3) / 1e9) if lab_ms > 0 else None
    ncu = load_ncu_traffic() or {}
    note_streams = (f"; batched: {streams} concurrent streams" if streams > 1 else "") + \
        "; family time = wall-clock union of its launch intervals across streams"
    roof_lab = {
        "kernel": "labrd4_kernel + labrd2_kernel (GEBRD panels: 2 GEMVs per column over the trailing matrix)",
        "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
        "frac": (achieved / hbm) if achieved else None,
        "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
        "traffic": ncu.get("labrd_dram_bytes_per_step") if args.workload == "c2" else None,
        "traffic_note": ("DRAM bytes per step = sum of dram__bytes_read + dram__bytes_write over all 300 LABRD/GEBD2 "
                         "launches of one 8192^2 GEBRD (ncu --cache-control none, profiles/labrd_dram_r02.csv, "
                         "profiles/ncu_r02_labrd_dram.md): 65 % of the algorithmic bytes -- the snake order and L2 "
                         "hints serve the rest from L2") if args.workload == "c2" else "C2 capture only",
        "algorithmic_bytes_per_step": lab_bytes / max(args.steps, 1),
        "launches_per_step": lab_n / max(args.steps, 1),
        "share_of_step": (lab_ms / args.steps) / t_ms if t_ms > 0 else None,
        "note": "achieved = algorithmic GEMV bytes (8 sum_k [(m'-k)(n'-k-1) + (m'-k-1)(n'-k-1)] per panel) / time of "
                "the panel launches (CUDA events on their streams, recorded in an identical instrumented pass of the "
                "same K steps right after the uninstrumented timed pass)" + note_streams,
    }
    dmma_peak = 148 * 128 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12
    gem_achieved = (gem_flops / (gem_ms * 1e-3) / 1e12) if gem_ms > 0 else None
    roof_gem = {
        "kernel": "all DMMA GEMMs: dgemm_ws_kernel (TMA, long K: CWY inner products, TS U = Q U0), rankk_tile_kernel "
                  "(TMA, CWY rank-128 updates), rankk_stream_kernel (GEBRD rank-64 trailing update), "
                  "dgemm_ws_gather_kernel (TMA gather4, BDC merge products), dgemm_kernel (fallback)",
        "bound": "tensor", "achieved": gem_achieved, "peak": dmma_peak, "unit": "TFLOP/s",
        "frac": (gem_achieved / dmma_peak) if gem_achieved else None,
        "peak_source": "FP64 DMMA peak 148 SMs x 128 flop/clk at sm_max_mhz (MEASURED_PEAKS.json); cuBLAS DGEMM "
                       "8192^3 measured 35.4 TFLOP/s on this pool (tools/cublas_probe.py)",
        "traffic": None,
        "algorithmic_flops_per_step": gem_flops / max(args.steps, 1),
        "launches_per_step": gem_n / max(args.steps, 1),
        "share_of_step": (gem_ms / args.steps) / t_ms if t_ms > 0 else None,
        "note": "achieved = sum 2mnk / time of the GEMM launches (CUDA events on their streams, identical "
                "instrumented pass of the same K steps after the timed pass)" + note_streams,
    }
    roof, roof2 = (roof_lab, roof_gem) if lab_ms >= gem_ms else (roof_gem, roof_lab)
    if c5:
        svd_s = args.c5_total / (t_ms * 1e-3)
        metric, val, unit = f"batched fp64 SVD (U,S,V) throughput, {args.c5_total} x {m}x{n}", svd_s, "SVD/s"
        e2e_val = args.c5_total / (e2e_ms * 1e-3)
    else:
        metric, val, unit = "fp64 SVD (U,S,V) GFLOP/s (28/3 n^3 convention)", value, "GFLOP/s"
        e2e_val = e2e_value
    line = {
        "metric": metric,
        "value": val,
        "unit": unit,
        "gflops": value,
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_ms,
        "seconds_per_svd": t_ms * 1e-3 / (args.c5_total if c5 else 1),  # whole job (c5) / one replica
        "higher_is_better": True,
        "scaling": "strong" if c5 else "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (Philox MatrixSpec('random') inputs, BASELINE.md §3)",
        "config": {"workload": desc, "m": m, "n": n, "batch_per_gpu": batch,
                   **({"batch_total": args.c5_total, "shard_rank0": [lo, hi]} if c5 else {}),
                   "parallelism": f"batch shards x{ws} ({dist.get_backend() if ws > 1 else 'single process'})"
                   if c5 else f"replicas x{ws}",
                   "l2": "input 512 MiB > 126 MB L2 (no flush needed)" if m * n * 8 > 2 ** 28 else "input fits L2; timed back-to-back"},
        "phases_s": dict(prof.phases),
        "accuracy": {"sigma_rel_vs_reference": sig_rel, "sigma_tol": 1e-12 * k,
                     "sigma_reference": (f"tests/golden/{args.workload}_sigma.npz: reference dcsvd.gesdd values-only on "
                                         f"the same MatrixSpec('random',{m},{n},seed=...) bytes, {sig_items} item(s)")
                     if fx is not None else None,
                     "resid_scaled": resid, "orth_u_scaled": orth_u, "orth_v_scaled": orth_v, "tol": 1e-14,
                     "pass": bool((sig_rel is None or sig_rel <= 1e-12 * k) and resid <= 1e-14 and orth_u <= 1e-14
                                  and orth_v <= 1e-14)},
        "gpu_launches": int(launches),
        "roofline": roof,
        "roofline_secondary": roof2,
        "clocks": clk.summary(),
        "e2e": {"value": e2e_val, "unit": unit, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_ms},
    }
    if not args.no_cpu_baseline and ws == 1:
        kind = ref_kind()
        who = "reference dcsvd 0.1.0 (baseline/_ref)" if kind == "reference" else "oracle port (numpy restatement)"
        if c5:
            procs = max(1, min(host_cores(), 64))
            t_cpu = cpu_parallel(n, procs, seed)
            line["cpu_baseline"] = {"value": procs / t_cpu, "unit": "SVD/s", "cores": procs, "kind": kind,
                                    "seconds": t_cpu,
                                    "sample": f"{who}: {procs} concurrent single-thread processes, one full "
                                              f"{m}x{n} SVD with vectors each (seeds {seed}..{seed + procs - 1})"}
        else:
            n_s = 1536 if kind == "reference" else 2048
            t_cpu = cpu_sample(n_s, 1)
            line["cpu_baseline"] = {"value": flops_square(n_s) / t_cpu / 1e9, "unit": "GFLOP/s", "cores": 1,
                                    "kind": kind, "seconds": t_cpu,
                                    "sample": f"{who}, 1 BLAS thread (the reference's own pin, conftest.py), full "
                                              f"SVD with vectors of MatrixSpec('random',{n_s},{n_s},seed=1)"}
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
