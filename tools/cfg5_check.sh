#!/bin/bash
out=gpurun_out/${1:-cfg5}
mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_planner.py tests/test_gpu_configs.py -x -q -k "grid or cfg5 or devices or large" > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
timeout 300 python tools/cfg5bench.py >> $out/cfg5.jsonl 2>> $out/cfg5.err
SPLITPLAN_WS_GB=150 timeout 300 python tools/cfg5bench.py >> $out/cfg5.jsonl 2>> $out/cfg5.err
