#!/bin/bash
out=gpurun_out/${1:-inplace}
mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_planner.py tests/test_gpu_configs.py -x -q -k "grid or cfg5 or devices or large" > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
if grep -q "rc=0" $out/pytest.log; then
  timeout 300 python tools/cfg5bench.py >> $out/cfg5.jsonl 2>> $out/cfg5.err
  SPLITPLAN_GRID_INPLACE=0 timeout 300 python tools/cfg5bench.py >> $out/cfg5.jsonl 2>> $out/cfg5.err
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:dp_grid -c 1 --csv python tools/cfg5bench.py --L 50000 > $out/ncu.csv 2>&1
fi
