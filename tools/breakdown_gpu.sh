#!/bin/bash
# host phases (SPLITPLAN_TRACE) and device launches of one Engine.solve at
# cfg3 and cfg4 scale.   usage: bash tools/breakdown_gpu.sh [tag]
tag=${1:-bd}
out=gpurun_out/$tag; mkdir -p $out
SPLITPLAN_TRACE=1 timeout 600 python tools/solve_breakdown.py --config cfg4 --n 65536 > $out/cfg4.json 2> $out/cfg4_trace.txt
SPLITPLAN_TRACE=1 timeout 600 python tools/solve_breakdown.py --config cfg3 --n 1000000 > $out/cfg3.json 2> $out/cfg3_trace.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/cfg4_launches.csv python tools/solve_breakdown.py --config cfg4 --n 65536 > /dev/null 2>&1
