#!/bin/bash
out=gpurun_out/${1:-policy}
mkdir -p $out
for rep in 1 2; do for P in 0 1 2; do
  SPLITPLAN_CLUSTER_POLICY=$P timeout 120 python tools/k2bench.py --requests 3000 --reps 2 >> $out/k2.jsonl 2>> $out/k2.err
done; done
