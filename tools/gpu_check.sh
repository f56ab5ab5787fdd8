#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench (both arms), ncu launch list + full capture of k_sets.
# usage: gpurun --timeout 2400 -- bash tools/gpu_check.sh TAG
TAG=${1:-run}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.log 2>&1; echo "ref rc=$?" >> $O/bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > $O/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sets -s 3 -c 1 -o $O/k_sets python bench.py --steps 1 --warmup 3 --no-cpu > $O/ncu_full.log 2>&1
echo done
