#!/bin/bash
out=gpurun_out/${1:-occ1}
mkdir -p $out
for cfg in "1 7" "4 3" "4 4" "4 5" "5 3" "5 4" "5 5"; do set -- $cfg
  SPLITPLAN_STREAM_CFG=$1 SPLITPLAN_DP_CLUSTER=$2 timeout 120 python tools/k2bench.py --requests 3000 --reps 2 >> $out/k2.jsonl 2>> $out/k2.err
done
for cfg in "4 4" "5 4"; do set -- $cfg
  SPLITPLAN_STREAM_DIAG=1 SPLITPLAN_STREAM_CFG=$1 SPLITPLAN_DP_CLUSTER=$2 timeout 120 python tools/k2bench.py --requests 3000 --reps 2 >> $out/k2.jsonl 2>> $out/k2.err
done
