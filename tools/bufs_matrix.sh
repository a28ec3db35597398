#!/bin/bash
out=gpurun_out/${1:-bm}
mkdir -p $out
timeout 120 python tools/dpbench.py --variant stream --W 100000 --n 148 --reps 1 > $out/sanity.log 2>&1 || exit 1
for G in 4 5 6 7 10; do
  SPLITPLAN_STREAM_BUFS=2 SPLITPLAN_DP_CLUSTER=$G timeout 200 python tools/dpbench.py --variant stream --W 100000 --reps 2 > $out/b2_G${G}.log 2>&1
done
SPLITPLAN_STREAM_BUFS=2 timeout 200 python tools/dpbench.py --variant stream --W 28000,50000,100000 --reps 2 > $out/b2_default.log 2>&1
timeout 200 python tools/dpbench.py --variant stream --W 28000,50000,100000 --reps 2 > $out/b3_default.log 2>&1
SPLITPLAN_STREAM_BUFS=2 timeout 900 python -m pytest tests/test_gpu_planner.py -m gpu -x -q > $out/pytest_b2.log 2>&1; echo "rc=$?" >> $out/pytest_b2.log
