#!/bin/bash
out=gpurun_out/${1:-owndiag}
mkdir -p $out
timeout 300 python tools/dpbench.py --variant own --W 10000,18000,36000,100000 --reps 2 > $out/dp_own.log 2>&1
timeout 300 python tools/dpbench.py --variant smem --W 10000,18000 --reps 2 > $out/dp_smem.log 2>&1
SPLITPLAN_DP_VARIANT=own timeout 600 ncu --set full --import-source on --clock-control none -k regex:dp_own -c 1 -o $out/own_cfg2 python tools/k2bench.py --requests 1000 --reps 1 > $out/ncu_log.txt 2>&1
