"""Summarize ncu outputs into profiles/ (run in the build container).

usage: python tools/summarize_ncu.py launches.csv [full.ncu-rep ...] --out profiles/ncu_r01
Writes <out>_launches.md (per-kernel share of one step) and <out>_full.md with
the key metrics of each full capture, plus profiles/ncu_summary.json
(labrd dram bytes per launch, consumed by bench.py as roofline.traffic)."""
import collections, csv, json, os, re, subprocess, sys


def launches(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[i]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0.0, 0])
    for r in rows[i + 1:]:
        if len(r) <= vi:
            continue
        name = re.sub(r"<.*", "", re.sub(r"\(.*", "", r[ki])).replace("void ", "").strip()
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r[ui], 1e-6)
        agg[name][0] += v * scale
        agg[name][1] += 1
    return agg


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct"]
    out = []
    for r in rows[2:]:
        d = {}
        for w in want:
            if w in hdr:
                j = hdr.index(w)
                d[w] = (r[j], units[j])
        out.append(d)
    return out


def main():
    args = sys.argv[1:]
    out = args[args.index("--out") + 1]
    args = args[: args.index("--out")]
    os.makedirs(os.path.dirname(out), exist_ok=True)
    summ = {}
    lines = []
    for a in args:
        if a.endswith(".csv"):
            agg = launches(a)
            tot = sum(v[0] for v in agg.values())
            lines.append(f"## Launch list `{os.path.basename(a)}` (ncu gpu__time_duration, cold-cache, serialised)\n")
            lines.append(f"total kernel time {tot:.1f} ms, {sum(v[1] for v in agg.values())} launches\n")
            lines.append("| kernel | ms | share | launches |\n|---|---|---|---|")
            for k, (ms, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
                lines.append(f"| `{k}` | {ms:.2f} | {100 * ms / tot:.1f}% | {c} |")
                summ.setdefault("launch_share", {})[k] = ms / tot
            lines.append("")
        else:
            for d in full(a):
                name = d.get("Kernel Name", ("?", ""))[0]
                lines.append(f"## Full capture `{os.path.basename(a)}`: {name[:120]}\n")
                for k, (v, u) in d.items():
                    if k != "Kernel Name":
                        lines.append(f"- `{k}` = {v} {u}")
                lines.append("")
                if "labrd" in name:
                    key = "labrd2" if "labrd2" in name else "labrd"
                    rd = float(d["dram__bytes_read.sum"][0].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[d["dram__bytes_read.sum"][1]]
                    wr = float(d["dram__bytes_write.sum"][0].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[d["dram__bytes_write.sum"][1]]
                    summ[key + "_dram_bytes_per_launch"] = rd + wr
                    summ[key + "_capture"] = os.path.basename(a)
    open(out + ".md", "w").write("\n".join(lines) + "\n")
    pj = os.path.join(os.path.dirname(out), "ncu_summary.json")
    old = json.load(open(pj)) if os.path.exists(pj) else {}
    old.update(summ)
    json.dump(old, open(pj, "w"), indent=1)
    print(open(out + ".md").read())


if __name__ == "__main__":
    main()
