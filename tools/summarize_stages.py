"""Per-stage roofline table from the stage captures of tools/stage_ncu.sh
(run in the build container: python tools/summarize_stages.py gpurun_out profiles/ncu_r01_stages.md)."""
import csv, glob, os, subprocess, sys

HBM = 6544.7e9      # MEASURED_PEAKS.json hbm_gbs (burst copy)
DMMA = 37.2e12      # 148 SMs x 128 flop/clk x 1965 MHz

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "%": 1, "": 1}

STAGE = {"stage_trailing": "GEBRD trailing update A -= P Q^T (rank 64, first panel of 8192^2)",
         "stage_bdc_gemm": "BDC root merge products (grouped, gathered), n = 8192 bidiagonal",
         "stage_bdc_secular": "BDC root secular solve (warp per root)",
         "stage_bdc_vectors": "BDC root Loewner vectors (warp per column)",
         "stage_ormbr": "ORMBR-shaped GEMMs at 8192 (rank-128 update / split-K Y^T C / rank-64)",
         "stage_geqr2": "TS GEQRF panel 65536 x 32 (cooperative, smem slab)"}


def rows(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    if len(r) < 3:
        return []
    hdr, units = r[0], r[1]
    out = []
    for row in r[2:]:
        d = {}
        for k in ("Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                  "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
                  "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                  "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"):
            if k in hdr:
                j = hdr.index(k)
                v = row[j]
                try:
                    d[k] = float(v.replace(",", "")) * UNITS.get(units[j], 1)
                except ValueError:
                    d[k] = v
        out.append(d)
    return out


def main():
    src, dst = sys.argv[1], sys.argv[2]
    lines = ["## Per-stage ncu captures (`ncu --set full`, one launch each; tools/stage_ncu.sh)\n",
             "Peaks: HBM 6544.7 GB/s (MEASURED_PEAKS.json), FP64 DMMA 37.2 TFLOP/s (148 SMs x 128 flop/clk x 1965 MHz).\n",
             "| stage | kernel | time | DRAM R+W | DRAM BW (% of peak) | DMMA pipe active | L2 hit | SM throughput |",
             "|---|---|---|---|---|---|---|---|"]
    for f in sorted(glob.glob(os.path.join(src, "stage_*.ncu-rep"))):
        tag = os.path.basename(f).replace(".ncu-rep", "")
        for d in rows(f):
            t = d.get("gpu__time_duration.sum", 0.0)
            by = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
            bw = by / t if t else 0.0
            name = str(d.get("Kernel Name", "?")).split("(")[0].replace("void ", "")[:60]
            lines.append(f"| {STAGE.get(tag, tag)} | `{name}` | {t * 1e6:.1f} us | {by / 1e6:.1f} MB | "
                         f"{bw / 1e9:.0f} GB/s ({100 * bw / HBM:.0f} %) | "
                         f"{d.get('sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active', 0):.0f} % | "
                         f"{d.get('lts__t_sector_hit_rate.pct', 0):.0f} % | "
                         f"{d.get('sm__throughput.avg.pct_of_peak_sustained_elapsed', 0):.0f} % |")
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
