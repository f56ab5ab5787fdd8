#!/bin/bash
set -u
mkdir -p gpurun_out/loc
CS=/usr/local/cuda/bin/compute-sanitizer
run() { local name=$1 envs=$2 tool=$3; shift 3
  ( export $envs; timeout 900 $CS --tool $tool --print-limit 20 --kernel-name kns=3gvo "$@" > gpurun_out/loc/${name}.log 2>&1; echo "rc=$?" >> gpurun_out/loc/${name}.log )
  echo "== $name"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|rc=|mismatches" gpurun_out/loc/${name}.log; grep -m3 " at .*\.cu" gpurun_out/loc/${name}.log; }
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/loc/build.log 2>&1
run sync_base GVO_X=1 synccheck python tools/san_cases.py 16 16
run sync_nofuse GVO_FUSE_WARP=0 synccheck python tools/san_cases.py 16 16
run sync_nodedup GVO_DEDUP=0 synccheck python tools/san_cases.py 16 16
run race_nofuse GVO_FUSE_WARP=0 racecheck --racecheck-report hazard python tools/san_cases.py 8 8
run race_nodedup GVO_DEDUP=0 racecheck --racecheck-report hazard python tools/san_cases.py 8 8
run memcheck GVO_X=1 memcheck --leak-check full python tools/san_cases.py 8 8
