#!/bin/bash
out=gpurun_out/${1:-owng1}
mkdir -p $out
SPLITPLAN_OWN_OCC=2 SPLITPLAN_OWN_CFG=2 timeout 300 python tools/dpbench.py --variant own --W 8000,16000,32000,100000 --reps 2 > $out/own_occ2.log 2>&1
timeout 300 python tools/dpbench.py --variant smem --W 8000,16000 --reps 2 > $out/smem.log 2>&1
SPLITPLAN_OWN_OCC=2 SPLITPLAN_OWN_CFG=2 SPLITPLAN_DP_CLUSTER=2 timeout 300 python tools/dpbench.py --variant own --W 8000 --reps 2 > $out/own_occ2_G2.log 2>&1
SPLITPLAN_OWN_OCC=2 SPLITPLAN_OWN_CFG=2 SPLITPLAN_DP_CLUSTER=4 timeout 300 python tools/dpbench.py --variant own --W 8000 --reps 2 > $out/own_occ2_G4.log 2>&1
