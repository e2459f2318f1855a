#!/bin/bash
# Round evidence on the GPU box: bench lines for C1-C5, ncu launch list of the
# C2 bench command, full ncu captures of both LABRD variants (dev tool).
# usage (from the repo root, under gpurun): bash tools/evidence.sh TAG
set -x
TAG=${1:-r01}
O=gpurun_out
python bench.py > $O/bench_${TAG}_c2.json 2> $O/bench_${TAG}_c2.err
for w in c1 c3 c4 c5; do python bench.py --workload $w > $O/bench_${TAG}_$w.json 2> $O/bench_${TAG}_$w.err; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_${TAG}_c2.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:labrd4 -c 1 -o $O/labrd4_full python tools/prof_svd.py 8192 8192 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:labrd2 -c 1 -o $O/labrd2_full python tools/prof_svd.py 2048 2048 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:gebd2_cluster -c 1 -o $O/gebd2c_full python tools/prof_svd.py 1024 1024 1 > /dev/null 2>&1
ls -la $O
