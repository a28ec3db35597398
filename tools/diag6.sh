#!/bin/bash
out=gpurun_out/${1:-diag6}
mkdir -p $out
for D in 0 1 2 3; do
  SPLITPLAN_STREAM_DIAG=$D timeout 120 python tools/k2bench.py --requests 3000 --reps 2 >> $out/diag.jsonl 2>> $out/diag.err
done
