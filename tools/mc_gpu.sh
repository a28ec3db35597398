out=gpurun_out/mc1; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_montecarlo.py -x -q > $out/pytest_mc.log 2>&1; echo "rc=$?" >> $out/pytest_mc.log
timeout 300 python tools/mc_time.py 65536 > $out/mc_time.json 2>&1
timeout 300 python tools/mc_time.py 65536 >> $out/mc_time.json 2>&1
timeout 600 python tools/mc_profile.py --scenarios 65536 > $out/mc_profile.txt 2>&1
