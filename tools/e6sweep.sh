#!/bin/bash
out=gpurun_out/${1:-e6}
mkdir -p $out
timeout 300 python -m pytest tests/test_gpu_planner.py -x -q -k "stream" > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
for cfg in "1 7 80" "4 6 90" "4 7 80" "4 5 110"; do set -- $cfg
  SPLITPLAN_STREAM_CFG=$1 SPLITPLAN_DP_CLUSTER=$2 SPLITPLAN_L2_BUDGET_MB=$3 timeout 120 python tools/k2bench.py --requests 3000 --reps 2 >> $out/k2.jsonl 2>> $out/k2.err
done
