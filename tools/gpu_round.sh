#!/bin/bash
# One GPU-box pass: parity suite, smoke, DP micro-bench per variant, bench line.
# usage: bash tools/gpu_round.sh [tag]   (outputs under gpurun_out/<tag>/)
tag=${1:-run}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi.csv 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1
timeout 600 python tools/dpbench.py > $out/dpbench_auto.log 2>&1
for v in smem stream coop; do
  timeout 300 python tools/dpbench.py --variant $v --W 10000,28000,100000 > $out/dpbench_$v.log 2>&1
done
timeout 900 python bench.py --no-cpu-baseline > $out/bench.json 2> $out/bench.err
