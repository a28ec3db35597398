#!/bin/bash
out=gpurun_out/${1:-bufsweep}
mkdir -p $out
SPLITPLAN_DP_VARIANT=stream timeout 120 python tools/k2bench.py --requests 300 --reps 1 > $out/sanity.log 2>&1; echo "rc=$?" >> $out/sanity.log
grep -q "rc=0" $out/sanity.log || exit 1
timeout 600 python -m pytest tests/test_gpu_planner.py tests/test_gpu_configs.py -x -q > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
for NB in ${BUFS:-2 3}; do for G in ${GS:-5 7 8 10}; do for D in ${DS:-0}; do
  SPLITPLAN_STREAM_DIAG=$D SPLITPLAN_STREAM_BUFS=$NB SPLITPLAN_DP_CLUSTER=$G timeout 120 python tools/k2bench.py --requests 3000 --reps 2 >> $out/k2.jsonl 2>> $out/k2.err
done; done; done
