#!/bin/bash
# One gpurun session: GPU tests, a bench line, the ncu capture behind its
# roofline.  Usage (from the repo root, on the GPU box):
#   bash tools/gpu_round.sh [tests|bench|ncu|all] [bench args...]
set -u
mkdir -p gpurun_out
what=${1:-all}; shift || true
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
if [[ $what == tests || $what == all ]]; then
  timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
if [[ $what == bench || $what == all ]]; then
  timeout 1800 python bench.py "$@" > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench rc=$?" >> gpurun_out/bench.err
fi
if [[ $what == ab || $what == abncu ]]; then
  timeout 2400 python tools/ab_time.py "$@" > gpurun_out/ab.log 2>&1
  echo "ab rc=$?" >> gpurun_out/ab.log; cat gpurun_out/ab.log
fi
if [[ $what == ncu || $what == all || $what == abncu ]]; then
  timeout 2400 python tools/ncu_capture.py > gpurun_out/ncu_capture.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_capture.log
fi
tail -3 gpurun_out/pytest_gpu.log 2>/dev/null; tail -c 3000 gpurun_out/bench.json 2>/dev/null; tail -5 gpurun_out/bench.err 2>/dev/null; tail -20 gpurun_out/ncu_capture.log 2>/dev/null
