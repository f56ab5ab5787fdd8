#!/bin/bash
O=gpurun_out/${1:-wl4}
mkdir -p $O
timeout 300 python tools/unit_profile.py C4 > $O/unit_C4.log 2>&1; echo "rc=$?" >> $O/unit_C4.log
timeout 300 python tools/unit_profile.py C2 > $O/unit_C2.log 2>&1; echo "rc=$?" >> $O/unit_C2.log
timeout 900 python bench.py --workload C5 --steps 1 --warmup 1 --no-cpu > $O/bench_C5.log 2>&1; echo "rc=$?" >> $O/bench_C5.log
