#!/bin/bash
# Stream-kernel sweep over cluster size G at the bench workload (cfg2):
# bench speed without a profiler, then DRAM / L2 bytes of one K2 launch under ncu.
out=gpurun_out/${1:-l2sweep}
mkdir -p $out
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,lts__t_sectors.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum
for G in ${GS:-3 5 7 10 16}; do
  SPLITPLAN_DP_CLUSTER=$G timeout 300 python bench.py --no-cpu-baseline --requests 10000 --steps 3 --warmup 3 > $out/bench_G$G.json 2>&1
  SPLITPLAN_DP_CLUSTER=$G timeout 300 ncu --metrics $M --clock-control none -k regex:dp_stream -c 1 --csv \
     python bench.py --no-cpu-baseline --requests 3000 --steps 1 --warmup 0 > $out/ncu_G$G.csv 2>&1
done
