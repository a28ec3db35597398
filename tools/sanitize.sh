#!/bin/bash
# compute-sanitizer over every kernel (small instances): memcheck, racecheck,
# synccheck, initcheck.   usage: bash tools/sanitize.sh [outdir]
out=${1:-gpurun_out/sanitizer}
mkdir -p "$out"
for case in ${CASES:-smem stream grid grid_parts grid_devices steps steps_wide prefix sim cost tier0 tier1_waves async skeleton montecarlo}; do
  for tool in memcheck racecheck synccheck initcheck; do
    timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python tools/sanitize_cases.py --case $case > "$out/${case}_${tool}.log" 2>&1
    echo "$case $tool rc=$?" | tee -a "$out/summary.txt"
  done
done
