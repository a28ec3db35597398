#!/bin/bash
out=gpurun_out/${1:-occsweep}
mkdir -p $out
for cfg in "1 7 80" "4 7 80" "4 10 80" "4 7 110" "5 7 80" "5 10 80" "5 14 80" "2 7 80"; do set -- $cfg
  SPLITPLAN_STREAM_CFG=$1 SPLITPLAN_DP_CLUSTER=$2 SPLITPLAN_L2_BUDGET_MB=$3 timeout 120 python tools/k2bench.py --requests 3000 --reps 2 >> $out/k2.jsonl 2>> $out/k2.err
done
