#!/bin/bash
# Fast GPU check after a kernel change: a bounded sanity run first, then parity + numbers.
tag=${1:-quick}
out=gpurun_out/$tag
mkdir -p $out
timeout 120 python tools/dpbench.py --variant stream --W 100000 --n 148 --reps 1 > $out/sanity.log 2>&1
echo "sanity_rc=$?" >> $out/sanity.log
if grep -q "sanity_rc=0" $out/sanity.log; then
  timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> $out/pytest_gpu.log
  timeout 600 python tools/dpbench.py > $out/dpbench_auto.log 2>&1
  timeout 900 python bench.py --no-cpu-baseline > $out/bench.json 2> $out/bench.err
fi
