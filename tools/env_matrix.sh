#!/bin/bash
# The GPU planner/config suites under alternative kernel configurations.
out=gpurun_out/${1:-envmatrix}
mkdir -p $out
for e in "SPLITPLAN_STREAM_CFG=1" "SPLITPLAN_STREAM_CFG=0" "SPLITPLAN_STREAM_CFG=2" "SPLITPLAN_DP_SINGLE_E=4" "SPLITPLAN_DP_SINGLE_E=8" "SPLITPLAN_STREAM_BUFS=3" "SPLITPLAN_GRID_INPLACE=0" "SPLITPLAN_ROW_EVICT_LAST=1"; do
  env $e timeout 600 python -m pytest tests/test_gpu_planner.py tests/test_gpu_configs.py tests/test_gpu_montecarlo.py -x -q > $out/pytest_${e}.log 2>&1; echo "rc=$?" >> $out/pytest_${e}.log
done
