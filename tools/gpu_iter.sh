#!/bin/bash
# Iteration run: GPU parity tests, C4 per-template probe, C2/C4 bench lines, phase profiles.
# usage: gpurun --timeout 1800 -- bash tools/gpu_iter.sh TAG
O=gpurun_out/${1:-iter}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python tools/wl_probe.py C4 --per-template > $O/probe_C4.log 2>&1; echo "rc=$?" >> $O/probe_C4.log
GVO_SEG=0 timeout 600 python tools/wl_probe.py C4 --per-template > $O/probe_C4_noseg.log 2>&1; echo "rc=$?" >> $O/probe_C4_noseg.log
timeout 300 python bench.py --no-cpu > $O/bench_C2.log 2>&1; echo "rc=$?" >> $O/bench_C2.log
for f in ${FILTERS:-D3Q27/zyxf/a0/2y D3Q27/zyxf/a0/none}; do
  n=$(echo $f | tr '/' '_')
  GVO_LIB_VARIANT=prof timeout 300 python tools/unit_profile.py C4 $f > $O/unit_$n.log 2>&1
done
echo done
