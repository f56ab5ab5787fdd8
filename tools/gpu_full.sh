#!/bin/bash
# Full check: GPU tests under both set-kernel residencies, bench lines C1..C5.
O=gpurun_out/${1:-full}
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
GVO_BIG_BATCH=1 timeout 600 python -m pytest tests -m gpu -x -q > $O/pytest_sets1.log 2>&1; echo "rc=$?" >> $O/pytest_sets1.log
GVO_BIG_BATCH=1000000000 timeout 600 python -m pytest tests -m gpu -x -q > $O/pytest_sets2.log 2>&1; echo "rc=$?" >> $O/pytest_sets2.log
for w in ${WORKLOADS:-C2 C1 C3 C4 C5}; do
  case $w in C5) a="--steps 1 --warmup 1";; C3) a="--steps 2 --warmup 1";; C4) a="--steps 3";; *) a="";; esac
  timeout 1200 python bench.py --workload $w $a ${BENCH_ARGS:---no-cpu} > $O/bench_$w.log 2>&1
done
echo done
