#!/bin/bash
out=gpurun_out/${1:-ncugrid}
mkdir -p $out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dp_grid -c 1 -o $out/dp_grid python tools/cfg5bench.py --L 50000 --W 10000000 > $out/log_grid.txt 2>&1
