"""K2 (DP stage kernel) alone on the bench workload (cfg2 request instances).

    python tools/k2bench.py [--requests 10000] [--reps 3]

Builds the cfg2 instances once through the engine (K1), then times
`batch.plan_dp` (prep -> K2 -> K3) with the library's per-launch CUDA-event
profile and prints K2 cells/s.  Environment knobs of the planner
(SPLITPLAN_STREAM_CFG, SPLITPLAN_DP_CLUSTER, SPLITPLAN_STREAM_DIAG, ...) apply.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=10_000)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch
    from paper_2410_10759_b200 import _native as N
    from paper_2410_10759_b200 import batch as B
    from paper_2410_10759_b200 import cost_model as cm
    from paper_2410_10759_b200 import workloads as W
    from paper_2410_10759_b200.requests import Engine, RequestBatch
    lib = N.library()
    N.workspace(int(float(os.environ.get("K2BENCH_WS_GB", "48")) * (1 << 30)))  # one wave from the first call
    req = RequestBatch.from_numpy(**W.cfg2(args.requests, 2000)[0]).to("cuda")
    layers = cm.build_preset("gpt2-24", 128).layers
    engine = Engine([layers])
    sol = engine.solve(req, args.requests * len(layers), engine.layer_offsets(req))
    inst = sol.instances
    B.plan_dp(inst)
    torch.cuda.synchronize()
    lib.sp_profile_enable(1)
    lib.sp_profile_collect(None, None, None, None, None, None)
    for _ in range(args.reps):
        B.plan_dp(inst)
    torch.cuda.synchronize()
    ms, nl, cells, byts, al, var = (C.c_double(), C.c_int64(), C.c_double(), C.c_double(),
                                    C.c_int64(), C.c_int32())
    lib.sp_profile_collect(C.byref(ms), C.byref(nl), C.byref(cells), C.byref(byts), C.byref(al),
                           C.byref(var))
    lib.sp_profile_enable(0)
    env = {k: v for k, v in os.environ.items() if k.startswith("SPLITPLAN_")}
    print(json.dumps({"env": env, "cells_per_s": cells.value / (ms.value / 1e3),
                      "kernel_ms": ms.value / max(nl.value, 1), "launches": nl.value,
                      "variant": var.value}), flush=True)


if __name__ == "__main__":
    main()
