#!/bin/bash
# run the reference's own test-suite (staged, unmodified, in the
# git-ignored baseline/_ref/tests_pkg) against the GPU engine through the
# `dcsvd` shim (shim/dcsvd -> paper_2508_11467_b200).  Run on the GPU box:
#   bash tools/replay_reference_suite.sh [TAG]
# Stage first (build container): cp -r /root/reference/pkg/tests baseline/_ref/tests_pkg
TAG=${1:-r02}
O=gpurun_out
mkdir -p $O
R=$(pwd)
PYTHONPATH=$R/shim:$R/baseline/_ref/tests_pkg PYTHONDONTWRITEBYTECODE=1 python -m pytest baseline/_ref/tests_pkg \
  -p no:cacheprovider -q -rfE --durations=15 --junitxml $O/replay_${TAG}.xml > $O/replay_${TAG}.txt 2>&1
echo "replay rc=$?"
tail -40 $O/replay_${TAG}.txt
