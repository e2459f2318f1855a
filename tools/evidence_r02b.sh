#!/bin/bash
# Round-2 (final session) evidence on the GPU box: bench lines C1-C5 (C2 with
# the CPU baseline), the C5 2-rank run, the reference arm, and the C2 launch list.
O=gpurun_out
mkdir -p $O
timeout 900 python bench.py > $O/bench_r02_c2.json 2> $O/bench_r02_c2.err
for w in c1 c3 c4; do timeout 600 python bench.py --workload $w > $O/bench_r02_$w.json 2> $O/bench_r02_$w.err; done
timeout 900 python bench.py --workload c5 --steps 3 > $O/bench_r02_c5.json 2> $O/bench_r02_c5.err
timeout 900 python bench.py --workload c5 --steps 3 --gpus 2 --no-cpu-baseline > $O/bench_r02_c5_ws2.json 2> $O/bench_r02_c5_ws2.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_r02_ref.json 2> $O/bench_r02_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_r02_c2.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
ls -la $O
