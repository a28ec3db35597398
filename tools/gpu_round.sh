#!/bin/bash
# One GPU-box pass: parity suite, smoke, bench line, reference arm, launch list,
# one full ncu capture of the bench's DP kernel, and the e2e step timeline.
#   usage: bash tools/gpu_round.sh [tag]
tag=${1:-run}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi.csv 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke_rc=$?" >> $out/smoke.log
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-configs --no-dense > $out/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dp_steps -c 1 -o $out/dp_steps_full python tools/k2bench.py --requests 10000 --reps 1 > $out/ncu_full.log 2>&1
timeout 300 python tools/e2e_profile.py --plain > $out/e2e_plain.log 2>&1
