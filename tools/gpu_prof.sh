#!/bin/bash
# Phase profile of the set engine, segment cover on and off.
O=gpurun_out/${1:-prof}
mkdir -p $O
for f in ${FILTERS:-D3Q27/zyxf/a0/2y D3Q27/zyxf/a0/none}; do
  n=$(echo $f | tr '/' '_')
  timeout 300 python tools/unit_profile.py C4 $f > $O/unit_$n.log 2>&1
  GVO_SEG=0 timeout 300 python tools/unit_profile.py C4 $f > $O/unit_${n}_noseg.log 2>&1
done
echo done
