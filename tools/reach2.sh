#!/bin/bash
out=gpurun_out/${1:-reach2}
mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "rc=$?" >> $out/pytest_gpu.log
SPLITPLAN_GRID_INPLACE=0 timeout 600 python -m pytest tests/test_gpu_planner.py tests/test_gpu_configs.py -x -q > $out/pytest_noinplace.log 2>&1; echo "rc=$?" >> $out/pytest_noinplace.log
for e in "SPLITPLAN_NO_REACH=0" "SPLITPLAN_NO_REACH=1"; do
  env $e timeout 300 python tools/cfg5bench.py >> $out/cfg5.jsonl 2>> $out/cfg5.err
  env $e timeout 120 python tools/k2bench.py --requests 3000 --reps 2 >> $out/k2.jsonl 2>> $out/k2.err
done
SPLITPLAN_GRID_INPLACE=0 timeout 300 python tools/cfg5bench.py >> $out/cfg5.jsonl 2>> $out/cfg5.err
