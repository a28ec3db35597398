#!/bin/bash
# GPU suite + config timings + headline bench (no CPU legs).  usage: bash tools/gpu_check.sh tag
tag=${1:-chk}
out=gpurun_out/$tag; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo rc=$? >> $out/pytest_gpu.log
SPLITPLAN_TRACE=1 timeout 600 python tools/solve_breakdown.py --config cfg4 --n 65536 > $out/cfg4.json 2> $out/cfg4_trace.txt
SPLITPLAN_TRACE=1 timeout 600 python tools/solve_breakdown.py --config cfg3 --n 1000000 > $out/cfg3.json 2> $out/cfg3_trace.txt
timeout 300 python tools/mc_time.py 65536 > $out/mc_time.json 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-dense > $out/bench.json 2> $out/bench.err
