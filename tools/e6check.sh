#!/bin/bash
out=gpurun_out/${1:-e6b}
mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "rc=$?" >> $out/pytest_gpu.log
timeout 120 python tools/k2bench.py --requests 3000 --reps 2 >> $out/k2.jsonl 2>> $out/k2.err
SPLITPLAN_STREAM_CFG=1 timeout 120 python tools/k2bench.py --requests 3000 --reps 2 >> $out/k2.jsonl 2>> $out/k2.err
timeout 600 python bench.py --no-cpu-baseline > $out/bench.json 2> $out/bench.err
timeout 300 python tools/dpbench.py --variant stream --W 28000,50000,100000,200000 --reps 2 > $out/dp_stream.log 2>&1
