python -m pytest tests -m gpu -x -q 2>&1 | tail -3
bash tools/replay_reference_suite.sh r02b | tail -8
python bench.py --steps 5 --warmup 3 > gpurun_out/c2.json 2> gpurun_out/c2.err; tail -3 gpurun_out/c2.err
python bench.py --workload c3 --steps 5 --warmup 3 > gpurun_out/c3.json 2> gpurun_out/c3.err; tail -3 gpurun_out/c3.err
python bench.py --workload c5 --steps 3 --warmup 3 > gpurun_out/c5.json 2> gpurun_out/c5.err; tail -3 gpurun_out/c5.err
python bench.py --workload c4 --steps 5 --warmup 3 > gpurun_out/c4.json 2> gpurun_out/c4.err; tail -3 gpurun_out/c4.err
