#!/bin/bash
# compute-sanitizer over the device pipeline (race / sync / memory
# checking of the persistent set kernel: work queue spin-waits, cross-CTA
# atomics, shared-memory atomicOr bitmaps).  Run on the GPU box; logs to
# gpurun_out/san_*.log.
set -u
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # name, env, tool, args...
  local name=$1 envs=$2 tool=$3; shift 3
  ( export $envs; timeout 2400 $CS --tool $tool --print-limit 100 --kernel-name kns=3gvo "$@" \
      > gpurun_out/san_${name}.log 2>&1; echo "rc=$?" >> gpurun_out/san_${name}.log )
  tail -4 gpurun_out/san_${name}.log
}
run memcheck GVO_X=1 memcheck --leak-check full python tools/san_cases.py 40 48
run memcheck_split GVO_SMEM_ELEMS=96 memcheck python tools/san_cases.py 24 16
run racecheck GVO_X=1 racecheck --racecheck-report hazard python tools/san_cases.py 8 8
run synccheck GVO_X=1 synccheck python tools/san_cases.py 16 16
run initcheck GVO_X=1 initcheck python tools/san_cases.py 8 8
