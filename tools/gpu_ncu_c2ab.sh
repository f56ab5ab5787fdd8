#!/bin/bash
O=gpurun_out/${1:-c2ab}
mkdir -p $O
for v in "" orig; do
  GVO_LIB_VARIANT=$v timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sets -s 3 -c 1 -o $O/k_sets_${v:-prod} python bench.py --steps 1 --warmup 3 --no-cpu > $O/ncu_${v:-prod}.log 2>&1
done
echo done
