#!/bin/bash
# Tuning matrix of the streaming DP kernel at cfg2 width (W = 1e5).
out=gpurun_out/${1:-matrix}
mkdir -p $out
timeout 120 python tools/dpbench.py --variant stream --W 100000 --n 148 --reps 1 > $out/sanity.log 2>&1 || exit 1
for T in 256 128; do
  for B in 24 40 64; do
    SPLITPLAN_STREAM_T=$T SPLITPLAN_L2_BUDGET_MB=$B timeout 120 python tools/dpbench.py --variant stream --W 100000 --n 1200 --reps 2 > $out/T${T}_B${B}.log 2>&1
  done
  for G in 4 8 16; do
    SPLITPLAN_STREAM_T=$T SPLITPLAN_DP_CLUSTER=$G timeout 120 python tools/dpbench.py --variant stream --W 100000 --n 1200 --reps 2 > $out/T${T}_G${G}.log 2>&1
  done
done
for T in 256 128; do SPLITPLAN_STREAM_T=$T timeout 200 python tools/dpbench.py --variant stream --W 28000,50000 --reps 2 > $out/T${T}_widths.log 2>&1; done
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> $out/pytest_gpu.log
