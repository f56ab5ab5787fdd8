#!/bin/bash
# C2 bench under several environment settings (A/B of context knobs); list on stdin-less heredoc below via $ENVLIST
O=gpurun_out/${1:-envab}
mkdir -p $O
i=0
echo "$ENVLIST" | tr ';' '\n' | while read -r envs; do
  [ -z "$envs" ] && continue
  i=$((i+1))
  for r in 1 2; do env $envs timeout 300 python bench.py --no-cpu > $O/bench_${i}_$r.log 2>&1; done
  echo "$i: $envs" >> $O/index.txt
done
echo done
