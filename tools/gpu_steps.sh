#!/bin/bash
# GPU check after a dp_steps_kernel change: sanity run, GPU suite, bench line
# (headline only), one ncu --set full capture of the kernel at the benched
# batch.   usage: bash tools/gpu_steps.sh [tag]
tag=${1:-steps}
out=gpurun_out/$tag
mkdir -p $out
timeout 180 python tools/k2bench.py --requests 10000 --reps 3 > $out/sanity.log 2>&1
echo "sanity_rc=$?" >> $out/sanity.log
if grep -q "sanity_rc=0" $out/sanity.log; then
  timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> $out/pytest_gpu.log
  timeout 600 python bench.py --no-cpu-baseline --no-configs --no-dense > $out/bench.json 2> $out/bench.err
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:dp_steps -c 1 -o $out/dp_steps_full python tools/k2bench.py --requests 10000 --reps 1 > $out/ncu_full.log 2>&1
fi
