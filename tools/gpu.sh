#!/bin/bash
# build + CPU sanity (library loads, exports) + gpurun.  usage: tools/gpu.sh TIMEOUT 'command'
set -e
cd /root/repo
python -m paper_2508_11467_b200.build > /dev/null
python -m pytest tests -q -x -m "not gpu" -k "exports" 2>&1 | tail -1
T=$1; shift
timeout $((T + 1200)) /usr/local/graft/bin/gpurun --timeout $T -- "$@" 2>&1 | tail -60
