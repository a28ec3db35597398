#!/bin/bash
out=gpurun_out/${1:-matrix2}
mkdir -p $out
timeout 120 python tools/dpbench.py --variant stream --W 100000 --n 148 --reps 1 > $out/sanity.log 2>&1 || exit 1
for G in 5 6 7 8 10 12; do
  SPLITPLAN_DP_CLUSTER=$G timeout 200 python tools/dpbench.py --variant stream --W 28000,50000,100000 --reps 2 > $out/T256_G${G}.log 2>&1
done
for G in 3 4 6; do
  SPLITPLAN_STREAM_T=128 SPLITPLAN_DP_CLUSTER=$G timeout 200 python tools/dpbench.py --variant stream --W 28000,50000,100000 --reps 2 > $out/T128_G${G}.log 2>&1
done
timeout 200 python tools/dpbench.py --variant stream --W 28000,50000,100000 --reps 2 > $out/default.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > $out/bench.json 2> $out/bench.err
