#!/bin/bash
# C2 bench + C4 probe for each library variant, then an ncu source capture of a C4 subset.
O=gpurun_out/${1:-var}
mkdir -p $O
for v in ${VARIANTS:-"" inl orig}; do
  for i in 1 2; do
    GVO_LIB_VARIANT=$v timeout 300 python bench.py --no-cpu > $O/bench_C2_${v:-prod}_$i.log 2>&1
  done
  GVO_LIB_VARIANT=$v timeout 300 python tools/wl_probe.py C4 > $O/probe_C4_${v:-prod}.log 2>&1
done
if [ -n "$NCU_F" ]; then
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_sets -s 1 -c 1 -o $O/k_sets_sub python tools/run_subset.py C4 $NCU_F 2 > $O/ncu.log 2>&1
fi
echo done
