"""Where the time of one Engine.solve goes (device kernels vs host planning).

    python tools/solve_breakdown.py --config cfg3 --n 1000000
    python tools/solve_breakdown.py --config cfg4 --n 65536     (scenarios)

Runs a warm-up solve (the workspace grows to its useful size), then one
timed solve with the library's per-launch DP profile, CUDA events around the
whole solve and around the K1 cost table, and the host wall time.
"""
import argparse
import ctypes as C
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--n", type=int, default=1_000_000)
    args = ap.parse_args()
    import torch
    from paper_2410_10759_b200 import _native as N
    from paper_2410_10759_b200 import batch as B
    from paper_2410_10759_b200 import workloads as W
    from paper_2410_10759_b200.requests import Engine, RequestBatch
    if args.config == "cfg4":  # n scenarios of 64 requests each
        import numpy as np
        req, layers, _ = W.cfg4(np.arange(args.n))
    else:
        req, layers = getattr(W, args.config)(args.n)
    eng = Engine(layers)
    dev = RequestBatch.from_numpy(**req).to(N.device())
    total = int(eng.n_layers[req["model"]].sum())
    off = eng.layer_offsets(dev)
    eng.solve(dev, total, off)
    torch.cuda.synchronize()
    lib = N.library()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    lib.sp_profile_enable(1)
    lib.sp_profile_collect(None, None, None, None, None, None)
    t0 = time.perf_counter()
    ev[0].record()
    inst, status, f = eng.cost_table(dev, total, off)
    ev[1].record()
    B.plan_dp(inst)
    ev[2].record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ms, n, cells, byts, al, var = (C.c_double(), C.c_int64(), C.c_double(), C.c_double(), C.c_int64(), C.c_int32())
    lib.sp_profile_collect(C.byref(ms), C.byref(n), C.byref(cells), C.byref(byts), C.byref(al), C.byref(var))
    print(json.dumps({"config": args.config, "n": args.n, "wall_s": wall,
                      "k1_ms": ev[0].elapsed_time(ev[1]), "plan_dp_ms": ev[1].elapsed_time(ev[2]),
                      "dp_kernel_ms": ms.value, "dp_launches": n.value, "all_launches": al.value,
                      "dp_cells": cells.value, "variant": var.value,
                      "workspace_gb": N._ws[torch.cuda.current_device()].numel() / 2 ** 30,
                      "dense_fallbacks": int(lib.sp_last_dense_fallbacks())}))


if __name__ == "__main__":
    main()
