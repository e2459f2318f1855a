#!/bin/bash
# Round-2 evidence on the GPU box (run from the repo root under gpurun):
# bench lines for C1-C5 (C2 with the CPU baseline), the C5 2-rank run, the
# reference arm, and ncu captures of the round-2 GEMM kernels.
O=gpurun_out
mkdir -p $O
timeout 900 python bench.py > $O/bench_r02_c2.json 2> $O/bench_r02_c2.err
for w in c1 c3 c4; do timeout 600 python bench.py --workload $w > $O/bench_r02_$w.json 2> $O/bench_r02_$w.err; done
timeout 900 python bench.py --workload c5 --steps 3 > $O/bench_r02_c5.json 2> $O/bench_r02_c5.err
timeout 900 python bench.py --workload c5 --steps 3 --gpus 2 --no-cpu-baseline > $O/bench_r02_c5_ws2.json 2> $O/bench_r02_c5_ws2.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_r02_ref.json 2> $O/bench_r02_ref.err
NCU="ncu --set full --import-source on --clock-control none"
timeout 600 $NCU -k regex:rankk_tilec -s 1 -c 1 -o $O/rankk_tilec128_r02 python tools/gemm_one.py 8192 8192 128 0 0 > /dev/null 2>&1
timeout 600 $NCU -k regex:rankk_tilec -s 1 -c 1 -o $O/rankk_tilec64_r02 python tools/gemm_one.py 8160 8160 64 0 1 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_r02b_c2.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
ls -la $O
