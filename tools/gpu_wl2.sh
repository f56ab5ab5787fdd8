#!/bin/bash
O=gpurun_out/${1:-wl2}
mkdir -p $O
timeout 600 python tools/wl_probe.py C4 --per-template > $O/probe_C4.log 2>&1
timeout 900 python -m pytest tests/test_workloads.py -m gpu -x -q > $O/pytest_wl.log 2>&1; echo "rc=$?" >> $O/pytest_wl.log
timeout 900 python bench.py --workload C4 --steps 3 --warmup 3 > $O/bench_C4.log 2>&1; echo "rc=$?" >> $O/bench_C4.log
timeout 1200 python bench.py --workload C5 --steps 1 --warmup 1 --no-cpu > $O/bench_C5.log 2>&1; echo "rc=$?" >> $O/bench_C5.log
