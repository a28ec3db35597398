#!/bin/bash
# A/B of compile-time variants of the breakpoint kernel (build/var_*.so, loaded
# through SPLITPLAN_LIB) on the cfg2 batch; the GPU planner suite on the last.
#   usage: bash tools/ab_steps.sh [tag]
out=gpurun_out/${1:-ab}
mkdir -p $out
for v in "" build/var_*.so; do
  for r in 1 2; do SPLITPLAN_LIB=$v timeout 120 python tools/k2bench.py --requests 10000 --reps 5 >> $out/k2_$(basename ${v:-default}).log 2>&1; done
  last=$v
done
SPLITPLAN_LIB=$last timeout 600 python -m pytest tests/test_gpu_planner.py tests/test_gpu_scale_parity.py -x -q > $out/pytest_$(basename $last).log 2>&1
