mkdir -p gpurun_out/ab3
for v in "" build/var_ev1_b8.so build/var_ev1_b10.so build/var_ev1_b12.so; do
  for r in 1 2; do SPLITPLAN_LIB=$v timeout 120 python tools/k2bench.py --requests 10000 --reps 5 >> gpurun_out/ab3/k2_${v##*/}.log 2>&1; done
done
SPLITPLAN_LIB=build/var_ev1_b10.so timeout 600 python -m pytest tests/test_gpu_planner.py tests/test_gpu_scale_parity.py -x -q > gpurun_out/ab3/pytest_ev1_b10.log 2>&1
