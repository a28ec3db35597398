#!/bin/bash
out=gpurun_out/${1:-cfgx}
mkdir -p $out
for cfg in "4 6" "5 6" "6 7" "6 8" "7 8" "7 4" "5 11" "4 11"; do set -- $cfg
  SPLITPLAN_STREAM_CFG=$1 SPLITPLAN_DP_CLUSTER=$2 SPLITPLAN_L2_BUDGET_MB=200 timeout 120 python tools/k2bench.py --requests 3000 --reps 2 >> $out/k2.jsonl 2>> $out/k2.err
done
