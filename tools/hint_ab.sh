#!/bin/bash
out=gpurun_out/${1:-hintab}
mkdir -p $out
for rep in 1 2; do for e in "SPLITPLAN_ROW_EVICT_LAST=0" "SPLITPLAN_ROW_EVICT_LAST=1"; do
  env $e timeout 120 python tools/k2bench.py --requests 3000 --reps 2 >> $out/k2.jsonl 2>> $out/k2.err
done; done
for e in "SPLITPLAN_L2_BUDGET_MB=100 SPLITPLAN_ROW_EVICT_LAST=1" "SPLITPLAN_L2_BUDGET_MB=100"; do
  env $e timeout 120 python tools/k2bench.py --requests 3000 --reps 2 >> $out/k2.jsonl 2>> $out/k2.err
done
