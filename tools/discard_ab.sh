#!/bin/bash
out=gpurun_out/${1:-discard}
mkdir -p $out
SPLITPLAN_ROW_DISCARD=2 timeout 600 python -m pytest tests/test_gpu_planner.py tests/test_gpu_configs.py -x -q > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
for rep in 1 2; do for D in 0 2; do
  SPLITPLAN_ROW_DISCARD=$D timeout 120 python tools/k2bench.py --requests 3000 --reps 2 >> $out/k2.jsonl 2>> $out/k2.err
done; done
for D in 0 2; do
  SPLITPLAN_ROW_DISCARD=$D timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:dp_stream -c 1 --csv python tools/k2bench.py --requests 1000 --reps 1 > $out/ncu_$D.csv 2>&1
done
