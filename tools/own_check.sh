#!/bin/bash
# own-block kernel: bounded sanity, parity, then numbers.
out=gpurun_out/${1:-own}
mkdir -p $out
SPLITPLAN_DP_VARIANT=own timeout 120 python tools/k2bench.py --requests 300 --reps 1 > $out/sanity.log 2>&1; echo "rc=$?" >> $out/sanity.log
if grep -q "rc=0" $out/sanity.log; then
  timeout 600 python -m pytest tests/test_gpu_planner.py -x -q > $out/pytest_planner.log 2>&1; echo "rc=$?" >> $out/pytest_planner.log
  for O in ${OCCS:-1 2}; do for C in ${CFGS:-0 1 2}; do for NB in ${BUFS:-3}; do
    SPLITPLAN_OWN_OCC=$O SPLITPLAN_OWN_CFG=$C SPLITPLAN_OWN_BUFS=$NB timeout 120 python tools/k2bench.py --requests 3000 --reps 2 >> $out/k2.jsonl 2>> $out/k2.err
  done; done; done
  timeout 300 python tools/dpbench.py --variant own --W 10000,18000,36000,100000 --reps 2 > $out/dp_own.log 2>&1
fi
