#!/bin/bash
out=gpurun_out/${1:-reachab}
mkdir -p $out
for rep in 1 2; do for e in "SPLITPLAN_NO_REACH=0" "SPLITPLAN_NO_REACH=1"; do
  env $e timeout 120 python tools/k2bench.py --requests 3000 --reps 2 >> $out/k2.jsonl 2>> $out/k2.err
  env $e timeout 600 python bench.py --no-cpu-baseline --steps 5 >> $out/bench.jsonl 2>> $out/bench.err
done; done
