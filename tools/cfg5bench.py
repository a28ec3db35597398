"""Time the cfg5 single huge instance (L = 1e5 stages x W = 1e7 columns) on one GPU.

    python tools/cfg5bench.py [--L 100000] [--W 10000000]

Prints one JSON line: wall time of plan_dp (forward pass with checkpoints +
recompute/backtrack), DP-kernel time and cells/s from sp_profile_*.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=100_000)
    ap.add_argument("--W", type=int, default=10_000_000)
    ap.add_argument("--devices", type=int, default=0,
                    help="capacity partitions through sp_plan_dp_devices with this GPU listed N times "
                         "(one workspace per partition)")
    args = ap.parse_args()
    import os
    # the whole-GPU path keeps as many back-pointer stages as the workspace
    # holds (the rest is recomputed from checkpoints): give it most of HBM
    os.environ.setdefault("SPLITPLAN_WS_GB", "150")
    import torch
    from paper_2410_10759_b200 import _native as N
    from paper_2410_10759_b200 import batch as B
    from paper_2410_10759_b200 import workloads as W
    x = W.cfg5(args.L, args.W)
    b = B.InstanceBatch.from_arrays(x["layer_off"], x["i"], x["s"], x["u"], x["d"], x["r"],
                                    x["budget"], x["sac"])
    lib = N.library()
    devs = [torch.cuda.current_device()] * args.devices if args.devices else None
    B.plan_dp(b, devices=devs)
    torch.cuda.synchronize()
    lib.sp_profile_enable(1)
    lib.sp_profile_collect(None, None, None, None, None, None)
    t0 = time.perf_counter()
    p = B.plan_dp(b, devices=devs)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ms, nl, cells, byts, al, var = (C.c_double(), C.c_int64(), C.c_double(), C.c_double(),
                                    C.c_int64(), C.c_int32())
    lib.sp_profile_collect(C.byref(ms), C.byref(nl), C.byref(cells), C.byref(byts), C.byref(al),
                           C.byref(var))
    problem_cells = float(args.L) * (args.W + 1)
    print(json.dumps({"L": args.L, "W": args.W, "partitions": args.devices or 1, "wall_s": wall, "problem_cells": problem_cells,
                      "problem_cells_per_s": problem_cells / wall, "dp_kernel_s": ms.value / 1e3,
                      "dp_cells_computed": cells.value, "dp_launches": nl.value,
                      "kernel_cells_per_s": cells.value / (ms.value / 1e3),
                      "feasible": bool(p.feasible.item()),
                      "integer_latency": int(p.integer_latency.item()),
                      "client_value": float(p.client_value.item())}))


if __name__ == "__main__":
    main()
