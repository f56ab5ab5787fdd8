#!/bin/bash
O=gpurun_out/${1:-c2}
mkdir -p $O
for v in ${VARIANTS:-"" orig}; do for r in 1 2; do GVO_LIB_VARIANT=$v timeout 300 python bench.py --no-cpu > $O/bench_${v:-prod}_$r.log 2>&1; done; done
timeout 300 python tools/wl_probe.py C4 > $O/probe_C4.log 2>&1
echo done
