#!/bin/bash
# Round evidence in one gpurun call: GPU tests, smoke, default bench (+CPU
# baseline) and reference arm, per-workload bench lines, ncu launch list and
# full k_sets captures (C2 default residency, C4 batch residency).
TAG=${1:-ev}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.log 2>&1; echo "ref rc=$?" >> $O/bench_ref.log
for W in C1 C3 C4; do
  timeout 900 python bench.py --workload $W --steps 5 --warmup 3 > $O/bench_$W.log 2>&1; echo "rc=$?" >> $O/bench_$W.log
done
timeout 1200 python bench.py --workload C5 --steps 1 --warmup 1 --no-cpu > $O/bench_C5.log 2>&1; echo "rc=$?" >> $O/bench_C5.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > $O/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sets -s 3 -c 1 -o $O/k_sets python bench.py --steps 1 --warmup 3 --no-cpu > $O/ncu_full.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sets -s 3 -c 1 -o $O/k_sets_c4 python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu > $O/ncu_full_c4.log 2>&1
echo done
