"""Per-kernel SASS opcode counts of libdcsvd_b200.so (build container, no GPU):
DMMA (FP64 tensor), LDGSTS (Ampere-style cp.async), UBLKCP (1-D TMA bulk copy),
UTMALDG / UTMAPF (TMA tensor-map load / L2 prefetch), LDS/LDG/STG, SYNCS
(mbarrier).  Writes profiles/sass_<tag>.md."""
import collections, re, subprocess, sys, os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2508_11467_b200", "libdcsvd_b200.so")
OPS = ["DMMA", "DFMA", "LDGSTS", "UBLKCP", "UTMALDG", "UTMAPF", "UTMASTG", "SYNCS", "LDS", "LDG", "STG", "BAR", "MEMBAR"]


def main(tag):
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    per = collections.OrderedDict()
    name = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            name = m.group(1)
            per[name] = collections.Counter()
            continue
        if name is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m:
            per[name][m.group(1)] += 1
    dem = subprocess.run(["c++filt"], input="\n".join(per), capture_output=True, text=True).stdout.splitlines()
    rows = []
    tot = collections.Counter()
    for (mang, cnt), d in zip(per.items(), dem):
        short = re.sub(r"\(.*", "", d).replace("void ", "")
        rows.append((short, cnt))
        tot.update(cnt)
    out = [f"## SASS opcode counts per kernel ({tag}, `cuobjdump -sass` of libdcsvd_b200.so, sm_100a)", "",
           "Static instruction counts (not executed counts). DMMA = FP64 tensor core (`mma.sync ... f64`; tcgen05 has "
           "no f64 kind); LDGSTS = per-thread cp.async; UBLKCP = 1-D TMA bulk copy (`cp.async.bulk`); UTMALDG / "
           "UTMAPF = TMA tensor-map load / L2 prefetch (`cp.async.bulk.tensor`, `cp.async.bulk.prefetch.tensor`); "
           "SYNCS = mbarrier operations.", "",
           "| kernel | " + " | ".join(OPS) + " |", "|---|" + "---|" * len(OPS)]
    for short, cnt in rows:
        if not any(cnt[o] for o in OPS):
            continue
        out.append(f"| `{short}` | " + " | ".join(str(cnt[o]) if cnt[o] else "" for o in OPS) + " |")
    out.append("| **total** | " + " | ".join(str(tot[o]) for o in OPS) + " |")
    path = os.path.join(ROOT, "profiles", f"sass_{tag}.md")
    open(path, "w").write("\n".join(out) + "\n")
    print(path, {o: tot[o] for o in OPS})


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02")
