#!/bin/bash
# ncu --set full of this round's auxiliary kernels at Monte-Carlo / cfg2 scale:
# skeleton_kernel, sim_replay_kernel, t0_count / t0_scatter (tier-0 planning),
# prep_kernel, cost_table_kernel.   usage: bash tools/ncu_aux.sh [tag]
out=gpurun_out/${1:-aux}; mkdir -p $out
cat > $out/mc_small.py <<'PY'
import numpy as np, torch, sys
sys.path.insert(0, ".")
from paper_2410_10759_b200 import montecarlo as MC
MC.run(np.arange(0, 65536, 4))
torch.cuda.synchronize()
PY
for k in skeleton_kernel sim_replay_kernel; do
  timeout 900 ncu --set full --clock-control none -k regex:$k -c 1 -o $out/$k python $out/mc_small.py > $out/$k.log 2>&1
done
cat > $out/t0.py <<'PY'
import os, numpy as np, torch, sys
sys.path.insert(0, ".")
os.environ["SPLITPLAN_STEPS_MIN_COLS"] = str(1 << 30)  # tier 0 takes the narrow rows
from paper_2410_10759_b200 import montecarlo as MC
MC.run(np.arange(0, 65536, 4))
torch.cuda.synchronize()
PY
for k in t0_count_kernel t0_scatter_kernel; do
  timeout 900 ncu --set full --clock-control none -k regex:$k -c 1 -o $out/$k python $out/t0.py > $out/$k.log 2>&1
done
python tools/ncu_brief.py $out/*.ncu-rep > $out/brief.jsonl 2>&1
