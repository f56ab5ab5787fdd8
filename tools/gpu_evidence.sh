#!/bin/bash
# Round evidence on the GPU box: the ncu capture of the dominant kernel for
# the headline workload (committed under profiles/, tagged with the build
# id), then the default bench line that reads it, then the GPU tests and the
# sanitizers.  Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 2400 python tools/ncu_capture.py > gpurun_out/ncu_capture.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_capture.log
timeout 1800 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
if [[ ${1:-} == full ]]; then
  timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
  bash tools/sanitize.sh > gpurun_out/san_summary.txt 2>&1
fi
tail -c 1500 gpurun_out/bench.json; tail -3 gpurun_out/bench.err; tail -c 600 gpurun_out/bench_ref.json; tail -3 gpurun_out/pytest_gpu.log 2>/dev/null
