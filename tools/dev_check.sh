#!/bin/bash
out=gpurun_out/${1:-devcheck}
mkdir -p $out
timeout 300 python -m pytest tests/test_gpu_planner.py -x -q -k "devices" > $out/pytest_dev.log 2>&1; echo "rc=$?" >> $out/pytest_dev.log
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "rc=$?" >> $out/pytest_gpu.log
