#!/bin/bash
out=gpurun_out/${1:-e8}
mkdir -p $out
timeout 300 python -m pytest tests/test_gpu_planner.py -x -q -k "single_cta" > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
timeout 300 python tools/dpbench.py --variant smem --W 1000,4000,10000,18000,26000 --reps 2 > $out/e4.log 2>&1
SPLITPLAN_DP_SINGLE_E=8 timeout 300 python tools/dpbench.py --variant smem --W 1000,4000,10000,18000,26000 --reps 2 > $out/e8.log 2>&1
SPLITPLAN_DP_SINGLE_E=8 SPLITPLAN_DP_THREADS=256 timeout 300 python tools/dpbench.py --variant smem --W 1000,4000,10000 --reps 2 > $out/e8_t256.log 2>&1
