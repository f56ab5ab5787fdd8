#!/bin/bash
O=gpurun_out/${1:-wl3}
mkdir -p $O
timeout 300 python tools/wl_probe.py C4 --per-template > $O/probe_C4.log 2>&1; echo "rc=$?" >> $O/probe_C4.log
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_workloads.py tests/test_report.py -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python bench.py --workload C4 --steps 3 --warmup 3 > $O/bench_C4.log 2>&1; echo "rc=$?" >> $O/bench_C4.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > $O/bench_C2.log 2>&1; echo "rc=$?" >> $O/bench_C2.log
