#!/bin/bash
# Streaming-kernel configuration x cluster-size sweep at the bench workload.
out=gpurun_out/${1:-cfgsweep}
mkdir -p $out
for C in ${CFGS:-0 1 2}; do
  SPLITPLAN_STREAM_CFG=$C timeout 300 python -m pytest tests/test_gpu_planner.py -x -q > $out/pytest_C$C.log 2>&1; echo "rc=$?" >> $out/pytest_C$C.log
  for G in ${GS:-auto 4 5 7}; do
    if [ $G = auto ]; then unset SPLITPLAN_DP_CLUSTER; else export SPLITPLAN_DP_CLUSTER=$G; fi
    SPLITPLAN_STREAM_CFG=$C timeout 300 python bench.py --no-cpu-baseline --steps 3 --warmup 3 > $out/bench_C${C}_G$G.json 2>&1
  done
  unset SPLITPLAN_DP_CLUSTER
done
