#!/bin/bash
# One full ncu capture per auxiliary kernel of the bench step (K1, prep, K3)
# and of the Monte-Carlo passes (prefix planners, K4 replay).
out=gpurun_out/${1:-ncuk}
mkdir -p $out
for k in cost_table_kernel prep_kernel backtrack_kernel; do
  timeout 600 ncu --set full --clock-control none -k regex:$k -c 1 -o $out/$k python tools/k2bench.py --requests 10000 --reps 1 > $out/log_$k.txt 2>&1
done
for k in prefix_kernel sim_replay_kernel; do
  timeout 600 ncu --set full --clock-control none -k regex:$k -c 1 -o $out/$k python tools/mc_time.py 4096 > $out/log_$k.txt 2>&1
done
