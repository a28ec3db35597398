#!/bin/bash
out=gpurun_out/${1:-gride6}
mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_planner.py tests/test_gpu_configs.py -x -q -k "grid or cfg5 or devices or large or reachable" > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
for rep in 1 2; do timeout 300 python tools/cfg5bench.py >> $out/cfg5.jsonl 2>> $out/cfg5.err; done
