#!/bin/bash
out=gpurun_out/${1:-gridab}
mkdir -p $out
for rep in 1 2; do for e in "SPLITPLAN_GRID_INPLACE=1" "SPLITPLAN_GRID_INPLACE=0"; do
  env $e timeout 300 python tools/cfg5bench.py >> $out/cfg5.jsonl 2>> $out/cfg5.err
done; done
SPLITPLAN_GRID_INPLACE=0 SPLITPLAN_NO_REACH=1 timeout 300 python tools/cfg5bench.py >> $out/cfg5.jsonl 2>> $out/cfg5.err
