#!/bin/bash
out=gpurun_out/${1:-hm}
mkdir -p $out
timeout 120 python tools/dpbench.py --variant stream --W 100000 --n 148 --reps 1 > $out/sanity.log 2>&1 || exit 1
for H in 0 1; do
  for BUF in 2 3; do
    SPLITPLAN_ROW_EVICT_LAST=$H SPLITPLAN_STREAM_BUFS=$BUF timeout 200 python tools/dpbench.py --variant stream --W 28000,100000 --reps 2 > $out/h${H}_b${BUF}.log 2>&1
    SPLITPLAN_ROW_EVICT_LAST=$H SPLITPLAN_STREAM_BUFS=$BUF timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:dp_stream -c 1 --csv python tools/dpbench.py --variant stream --W 100000 --n 1000 --reps 1 > $out/ncu_h${H}_b${BUF}.csv 2>&1
  done
done
