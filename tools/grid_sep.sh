#!/bin/bash
out=gpurun_out/${1:-gridsep}
mkdir -p $out
timeout 300 python -m pytest tests/test_gpu_planner.py -x -q -k "capacity_partitions and separate" > $out/pytest_sep.log 2>&1; echo "rc=$?" >> $out/pytest_sep.log
timeout 600 python -m pytest tests/test_gpu_planner.py -x -q > $out/pytest_planner.log 2>&1; echo "rc=$?" >> $out/pytest_planner.log
for mode in "" "SPLITPLAN_GRID_SEPARATE=1"; do
  env $mode SPLITPLAN_GRID_PARTS=4 timeout 300 python tools/cfg5bench.py >> $out/cfg5.jsonl 2>> $out/cfg5.err
done
