#!/bin/bash
# A/B: C2 bench with/without segment cover, C4 probe, phase profile of a C4 subset.
O=gpurun_out/${1:-ab}
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for i in 1 2; do
timeout 300 python bench.py --no-cpu > $O/bench_C2_$i.log 2>&1
GVO_SEG=0 timeout 300 python bench.py --no-cpu > $O/bench_C2_noseg_$i.log 2>&1
done
timeout 600 python tools/wl_probe.py C4 --per-template > $O/probe_C4.log 2>&1
GVO_LIB_VARIANT=prof timeout 300 python tools/unit_profile.py C4 ${F:-D3Q27/zyxf/a0/2y} > $O/unit.log 2>&1
echo done
