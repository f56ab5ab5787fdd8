#!/bin/bash
# ncu capture of the set kernel for the headline workload (committed under
# profiles/, tagged with the build id), then the default bench line that
# reads it.  Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
timeout 2400 python tools/ncu_capture.py > gpurun_out/ncu_capture.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_capture.log
timeout 1800 python bench.py "$@" > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
tail -c 1500 gpurun_out/bench.json; tail -3 gpurun_out/bench.err; tail -5 gpurun_out/ncu_capture.log
