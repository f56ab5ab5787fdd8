#!/bin/bash
# Round-end evidence on one B200: ncu capture of the set kernel (committed
# under profiles/, build-id tagged) -> default bench line that reads it ->
# every GPU test -> smoke -> sanitizers.  Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 2400 python tools/ncu_capture.py > gpurun_out/ncu_capture.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_capture.log
timeout 1800 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1800 bash tools/sanitize.sh > gpurun_out/san_summary.txt 2>&1
tail -c 800 gpurun_out/bench.json; tail -2 gpurun_out/bench.err; tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; grep -E "SUMMARY|mismatch" gpurun_out/san_summary.txt
