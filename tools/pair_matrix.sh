#!/bin/bash
out=gpurun_out/${1:-pm}
mkdir -p $out
timeout 120 python tools/dpbench.py --variant stream --W 100000 --n 148 --reps 1 > $out/sanity.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> $out/pytest_gpu.log
for P in 1 2; do
  SPLITPLAN_STREAM_PAIR=$P timeout 200 python tools/dpbench.py --variant stream --W 28000,50000,100000 --reps 2 > $out/pair${P}.log 2>&1
done
for G in 7 10 12 16; do
  SPLITPLAN_STREAM_PAIR=2 SPLITPLAN_DP_CLUSTER=$G timeout 200 python tools/dpbench.py --variant stream --W 100000 --reps 2 > $out/pair2_G${G}.log 2>&1
done
SPLITPLAN_STREAM_PAIR=2 SPLITPLAN_L2_BUDGET_MB=200 timeout 200 python tools/dpbench.py --variant stream --W 100000 --reps 2 > $out/pair2_B200.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > $out/bench.json 2> $out/bench.err
