#!/bin/bash
out=gpurun_out/${1:-inphint}
mkdir -p $out
for H in 0 1; do
SPLITPLAN_ROW_EVICT_LAST=$H timeout 300 python tools/cfg5bench.py >> $out/cfg5.jsonl 2>> $out/cfg5.err
SPLITPLAN_ROW_EVICT_LAST=$H timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:dp_grid -c 1 --csv python tools/cfg5bench.py --L 50000 > $out/ncu_$H.csv 2>&1
done
