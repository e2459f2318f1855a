"""Full-size CPU timing of the UNMODIFIED reference (baseline/_ref, dcsvd 0.1.0)
on the GPU box's host cores (BASELINE.md §3 plan):
phase_profile (driver.py:160-170) wall seconds for C1 (best of 3, 1 BLAS thread
and all cores), C3 (one run, all cores), C2 (one run, all cores), and C5
(one single-thread process per core, one 2048^2 item each, extrapolated to
512).  Inputs are the exact MatrixSpec bytes.  Writes JSON lines to stdout."""
import json, os, subprocess, sys, time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
CODE = ("import sys,time,json; sys.path.insert(0,%r); import dcsvd;"
        "a=dcsvd.generate_matrix(dcsvd.MatrixSpec('random',%d,%d,seed=%d));"
        "p=dcsvd.phase_profile(a); print(json.dumps({'total':p.total,'phases':dict(p.phases)}))")


def one(m, n, seed, threads):
    env = dict(os.environ, OPENBLAS_NUM_THREADS=str(threads), OMP_NUM_THREADS=str(threads), PYTHONDONTWRITEBYTECODE="1")
    r = subprocess.run([sys.executable, "-c", CODE % (REF, m, n, seed)], capture_output=True, text=True, env=env)
    if r.returncode:
        raise RuntimeError(r.stderr[-2000:])
    return json.loads(r.stdout.strip().splitlines()[-1])


def main(which):
    cores = len(os.sched_getaffinity(0))
    import platform
    info = {"host_cores": cores, "cpu": platform.processor() or open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": ")}
    print(json.dumps({"host": info}), flush=True)
    if "c1" in which:
        for th in (1, cores):
            runs = [one(1024, 1024, 1, th) for _ in range(3)]
            best = min(runs, key=lambda r: r["total"])
            print(json.dumps({"config": "C1 1024^2 seed 1", "threads": th, "best_of_3": best,
                              "all_totals": [r["total"] for r in runs]}), flush=True)
    if "c5" in which:
        import concurrent.futures as cf
        procs = min(cores, 64)
        t0 = time.perf_counter()
        with cf.ThreadPoolExecutor(max_workers=procs) as ex:
            res = list(ex.map(lambda i: one(2048, 2048, 1000 + i, 1), range(procs)))
        wall = time.perf_counter() - t0
        print(json.dumps({"config": "C5 2048^2 items, seeds 1000..", "processes": procs, "threads_each": 1,
                          "wall_s": wall, "svd_per_s": procs / wall, "extrapolated_512_s": 512 * wall / procs,
                          "item_totals": [r["total"] for r in res]}), flush=True)
    if "c3" in which:
        print(json.dumps({"config": "C3 65536x1024 seed 3", "threads": cores, "run": one(65536, 1024, 3, cores)}), flush=True)
    if "c2" in which:
        print(json.dumps({"config": "C2 8192^2 seed 2", "threads": cores, "run": one(8192, 8192, 2, cores)}), flush=True)


if __name__ == "__main__":
    main(set(sys.argv[1:]) or {"c1", "c5", "c3", "c2"})
