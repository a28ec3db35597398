#!/bin/bash
out=gpurun_out/${1:-mc3}
mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_montecarlo.py tests/test_gpu_configs.py -x -q > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
for P in 1 16; do SPLITPLAN_SKELETON_PROCS=$P timeout 300 python tools/mc_time.py 16384 >> $out/mc.jsonl 2>> $out/mc.err; done
timeout 300 python tools/mc_time.py 65536 >> $out/mc.jsonl 2>> $out/mc.err
SPLITPLAN_SKELETON_PROCS=16 timeout 600 python tools/mc_profile.py > $out/prof.txt 2>&1
