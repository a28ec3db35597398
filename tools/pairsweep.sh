#!/bin/bash
out=gpurun_out/${1:-pairsweep}
mkdir -p $out
for cfg in "0 1 7" "0 2 10" "0 2 14" "0 2 12" "1 1 7"; do set -- $cfg
  SPLITPLAN_STREAM_CFG=$1 SPLITPLAN_STREAM_PAIR=$2 SPLITPLAN_DP_CLUSTER=$3 timeout 120 python tools/k2bench.py --requests 3000 --reps 2 >> $out/k2.jsonl 2>> $out/k2.err
done
