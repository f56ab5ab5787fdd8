#!/bin/bash
# A/B timing of library variants (tools/ab_time.py) followed by a subset of
# the GPU tests on the product library.  Usage (GPU box, repo root):
#   bash tools/gpu_ab.sh "<pytest files>" variant...
set -u
mkdir -p gpurun_out
tests=$1; shift
timeout 1200 python tools/ab_time.py "$@" > gpurun_out/ab.log 2>&1; echo "ab rc=$?" >> gpurun_out/ab.log
cat gpurun_out/ab.log
if [[ -n $tests ]]; then
  timeout 1500 python -m pytest $tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_sub.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sub.log
  tail -5 gpurun_out/pytest_sub.log
fi
