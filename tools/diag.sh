#!/bin/bash
# Streaming-kernel bottleneck diagnosis: normal, no stage waits, no window copies, neither.
out=gpurun_out/${1:-diag}
mkdir -p $out
for C in ${CFGS:-0 1}; do for D in 0 1 2 3; do for G in ${GS:-5 7 16}; do
  SPLITPLAN_STREAM_CFG=$C SPLITPLAN_STREAM_DIAG=$D SPLITPLAN_DP_CLUSTER=$G timeout 120 python tools/k2bench.py --requests 3000 --reps 2 >> $out/diag.jsonl 2>> $out/diag.err
done; done; done
