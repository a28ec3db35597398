#!/bin/bash
out=gpurun_out/${1:-ncumore}
mkdir -p $out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dp_grid -c 1 -o $out/dp_grid python tools/cfg5bench.py --L 2000 --W 10000000 > $out/log_grid.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dp_stage -c 1 -o $out/dp_smem_e8 python tools/dpbench.py --variant smem --W 10000 --n 2000 --reps 1 > $out/log_smem.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:sim_replay --launch-skip 1 -c 1 -o $out/sim_replay python tools/mc_time.py 4096 > $out/log_sim.txt 2>&1
