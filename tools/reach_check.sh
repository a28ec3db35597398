#!/bin/bash
out=gpurun_out/${1:-reach}
mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "rc=$?" >> $out/pytest_gpu.log
for e in "SPLITPLAN_STREAM_CFG=1" "SPLITPLAN_STREAM_CFG=0" "SPLITPLAN_STREAM_PAIR=2"; do
  env $e timeout 600 python -m pytest tests/test_gpu_planner.py tests/test_gpu_configs.py -x -q > $out/pytest_${e}.log 2>&1; echo "rc=$?" >> $out/pytest_${e}.log
done
timeout 120 python tools/k2bench.py --requests 3000 --reps 2 >> $out/k2.jsonl 2>> $out/k2.err
SPLITPLAN_STREAM_CFG=1 timeout 120 python tools/k2bench.py --requests 3000 --reps 2 >> $out/k2.jsonl 2>> $out/k2.err
timeout 600 python bench.py --no-cpu-baseline > $out/bench.json 2> $out/bench.err
