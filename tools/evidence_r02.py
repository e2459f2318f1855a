"""Round-2 ncu evidence on the GPU box (run under gpurun from the repo root):
  1. DRAM bytes + duration of EVERY LABRD / GEBD2 launch of one 8192^2 GEBRD
     (--cache-control none: the L2 state the pipeline leaves, not flushed)
  2. launch list of the BDC merge GEMMs (gathered grouped dgemm) of one
     8192 bdsdc, then a --set full capture of the longest one (the root merge)
  3. --set full capture of the TMA rank-128 kernel at the ORMBR shape
  4. the launch list of the C2 bench command (per-launch times)
Outputs gpurun_out/*_r02*."""
import csv, os, subprocess, sys

O = "gpurun_out"
NCU = ["ncu", "--clock-control", "none"]
py = sys.executable


def run(cmd):
    print("+", " ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        print(r.stdout[-2000:], r.stderr[-2000:], flush=True)
    return r


def launch_rows(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[i]
    return hdr, [dict(zip(hdr, r)) for r in rows[i + 1:] if len(r) == len(hdr)]


os.makedirs(O, exist_ok=True)
what = set(sys.argv[1:]) or {"labrd", "bdc", "ormbr", "launches"}
if "labrd" in what:
    run(NCU + ["--cache-control", "none", "--metrics", "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum",
               "-k", "regex:labrd|gebd2", "--csv", "--log-file", f"{O}/labrd_dram_r02.csv", py, "tools/gebrd_once.py", "8192"])
if "bdc" in what:
    sel = ["--kernel-name-base", "demangled", "-k", r"regex:dgemm_kernel<\(bool\)0, \(bool\)0, .*\(bool\)1>"]
    run(NCU + sel + ["--metrics", "gpu__time_duration.sum", "--csv", "--log-file", f"{O}/bdc_gemm_list_r02.csv",
                     py, "tools/bdc_once.py", "8192"])
    hdr, rows = launch_rows(f"{O}/bdc_gemm_list_r02.csv")
    durs = [float(r["Metric Value"].replace(",", "")) for r in rows if r["Metric Name"] == "gpu__time_duration.sum"]
    k = max(range(len(durs)), key=lambda i: durs[i])
    print("BDC merge GEMM launches (ns):", durs, "root =", k, flush=True)
    run(NCU + ["--set", "full", "--import-source", "on"] + sel + ["--launch-skip", str(k), "-c", "1",
                                                                   "-o", f"{O}/bdc_root_gemm_r02", py, "tools/bdc_once.py", "8192"])
if "ormbr" in what:
    run(NCU + ["--set", "full", "--import-source", "on", "-k", "regex:rankk_ws", "-s", "1", "-c", "1",
               "-o", f"{O}/rankk_ws128_r02", py, "tools/gemm_one.py", "8192", "8192", "128", "0", "0"])
    run(NCU + ["--set", "full", "--import-source", "on", "-k", "regex:rankk_stream", "-s", "1", "-c", "1",
               "-o", f"{O}/rankk_stream64_r02", py, "tools/gemm_one.py", "8160", "8160", "64", "0", "1"])
if "launches" in what:
    run(NCU + ["--metrics", "gpu__time_duration.sum", "--csv", "--log-file", f"{O}/launches_r02_c2.csv",
               py, "bench.py", "--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "1"])
print(os.listdir(O))
