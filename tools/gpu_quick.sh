#!/bin/bash
# Fast GPU check after a kernel change: a bounded sanity run of the bench's
# DP step first, then parity + numbers.   usage: bash tools/gpu_quick.sh [tag]
tag=${1:-quick}
out=gpurun_out/$tag
mkdir -p $out
timeout 180 python tools/k2bench.py --requests 10000 --reps 3 > $out/sanity.log 2>&1
echo "sanity_rc=$?" >> $out/sanity.log
if grep -q "sanity_rc=0" $out/sanity.log; then
  timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> $out/pytest_gpu.log
  timeout 600 python bench.py --no-cpu-baseline --no-configs --no-dense > $out/bench.json 2> $out/bench.err
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-configs --no-dense > $out/bench_under_ncu.log 2>&1
fi
