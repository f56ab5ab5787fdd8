#!/bin/bash
# Workload parity + per-workload bench lines (exploration; not the driver's bench).
TAG=${1:-wl}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests/test_workloads.py -m gpu -x -q > $O/pytest_wl.log 2>&1; echo "rc=$?" >> $O/pytest_wl.log
for W in C1 C3 C4; do
  timeout 900 python bench.py --workload $W --steps 5 --warmup 3 > $O/bench_$W.log 2>&1; echo "rc=$?" >> $O/bench_$W.log
done
timeout 1200 python bench.py --workload C5 --steps 2 --warmup 1 --no-cpu > $O/bench_C5.log 2>&1; echo "rc=$?" >> $O/bench_C5.log
echo done
