#!/bin/bash
# Quick synccheck + racecheck over tools/san_cases.py (GPU box); optional
# library variant as $1 (GVO_LIB_VARIANT).
mkdir -p gpurun_out/san2
export GVO_LIB_VARIANT=${1:-}
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool synccheck --print-limit 10 --kernel-name kns=3gvo python tools/san_cases.py 16 16 > gpurun_out/san2/sync$1.log 2>&1
timeout 900 $CS --tool racecheck --racecheck-report hazard --print-limit 10 --kernel-name kns=3gvo python tools/san_cases.py 8 8 > gpurun_out/san2/race$1.log 2>&1
for f in gpurun_out/san2/sync$1.log gpurun_out/san2/race$1.log; do echo "== $f"; grep -E "SUMMARY|mismatches" $f; grep -m4 " at .*\.cu" $f; done
