#!/bin/bash
out=gpurun_out/${1:-ncuown}
mkdir -p $out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dp_own -c 1 -o $out/own_w1e4 python tools/dpbench.py --variant own --W 10000 --n 2000 --reps 1 > $out/log1.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dp_stage -c 1 -o $out/smem_w1e4 python tools/dpbench.py --variant smem --W 10000 --n 2000 --reps 1 > $out/log2.txt 2>&1
SPLITPLAN_OWN_CFG=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:dp_own -c 1 -o $out/own_cfg2 python tools/k2bench.py --requests 1000 --reps 1 > $out/log3.txt 2>&1
