#!/bin/bash
# Barrier-alignment check of the persistent set kernel (debug build with
# -DGVO_DEBUG_SYNC=1: every warp counts its passes through the item loop and
# thread 0 reports a warp on another pass).  Run on the GPU box.
set -u
mkdir -p gpurun_out/dbg
export GVO_LIB_VARIANT=dbgsync
timeout 600 python tools/san_cases.py 40 48 > gpurun_out/dbg/san_cases.log 2>&1; echo "rc=$?" >> gpurun_out/dbg/san_cases.log
timeout 900 python bench.py --workload C4 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/dbg/bench_c4.log 2>&1; echo "rc=$?" >> gpurun_out/dbg/bench_c4.log
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool synccheck --print-limit 10 --kernel-name kns=3gvo python tools/san_cases.py 16 16 > gpurun_out/dbg/sync.log 2>&1; echo "rc=$?" >> gpurun_out/dbg/sync.log
for f in gpurun_out/dbg/*.log; do echo "== $f"; grep -c GVO_DEBUG_SYNC $f; grep -m3 GVO_DEBUG_SYNC $f; tail -2 $f; done
