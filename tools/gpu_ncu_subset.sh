#!/bin/bash
# ncu --set full capture of k_sets on a workload subset.
O=gpurun_out/${1:-ncusub}; WL=${2:-C4}; F=${3:-D3Q27/zyxf/a0/none}
mkdir -p $O
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_sets -s 1 -c 1 -o $O/k_sets_sub python tools/run_subset.py $WL $F 2 > $O/ncu.log 2>&1
echo "rc=$?" >> $O/ncu.log
