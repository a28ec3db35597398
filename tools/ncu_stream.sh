mkdir -p gpurun_out/ncu1
for D in 0 3; do
SPLITPLAN_STREAM_CFG=1 SPLITPLAN_STREAM_DIAG=$D SPLITPLAN_DP_CLUSTER=5 timeout 600 ncu --set full --import-source on --clock-control none -k regex:dp_stream -c 1 -o gpurun_out/ncu1/stream_C1_D$D python tools/k2bench.py --requests 1000 --reps 1 > gpurun_out/ncu1/log_D$D.txt 2>&1
done
