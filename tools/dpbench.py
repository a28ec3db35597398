"""Micro-benchmark of the K2 DP stage kernel variants over budget widths.

    python tools/dpbench.py [--L 98] [--W 1000,10000,100000] [--n 512] [--variant auto]

Instances are seeded `from_costs` chains with integer r (int32 value domain)
sized so W_eff == W.  Prints one JSON line per width with DP cells/s of the
stage kernel (CUDA events around each launch, via sp_profile_*).
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def make(n, L, W, seed, r_kind):
    rng = np.random.default_rng(seed)
    hi = max(2, 4 * W // L)
    i = rng.integers(0, hi, (n, L))
    s = rng.integers(0, max(2, hi // 16), (n, L))
    u = rng.integers(0, hi, (n, L))
    d = rng.integers(0, hi, (n, L))
    if r_kind == "int":
        r = rng.integers(0, 10_000, (n, L)).astype(float)
    else:
        r = rng.random((n, L)) * 1e6
    off = np.arange(n + 1, dtype=np.int64) * L
    return off, i.ravel(), s.ravel(), u.ravel(), d.ravel(), r.ravel(), np.full(n, W), np.ones(n)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=98)
    ap.add_argument("--W", default="1000,4000,10000,28000,50000,100000")
    ap.add_argument("--n", type=int, default=0, help="instances (default: ~2e10 cells)")
    ap.add_argument("--variant", default="auto")
    ap.add_argument("--r", default="int", choices=("int", "float"))
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    if args.variant != "auto":
        os.environ["SPLITPLAN_DP_VARIANT"] = args.variant
    import torch
    from paper_2410_10759_b200 import _native as N
    from paper_2410_10759_b200 import batch as B
    lib = N.library()
    names = {0: "smem", 2: "global", 4: "stream", 5: "grid", 7: "steps"}
    for W in [int(w) for w in args.W.split(",")]:
        n = args.n or max(148, int(1.2e10 / (args.L * (W + 1))))
        b = B.InstanceBatch.from_arrays(*make(n, args.L, W, 1, args.r))
        B.plan_dp(b)  # warm-up
        torch.cuda.synchronize()
        lib.sp_profile_enable(1)
        lib.sp_profile_collect(None, None, None, None, None, None)
        for _ in range(args.reps):
            B.plan_dp(b)
        torch.cuda.synchronize()
        ms, nl, cells, byts, al, var = (C.c_double(), C.c_int64(), C.c_double(), C.c_double(),
                                        C.c_int64(), C.c_int32())
        lib.sp_profile_collect(C.byref(ms), C.byref(nl), C.byref(cells), C.byref(byts), C.byref(al),
                               C.byref(var))
        lib.sp_profile_enable(0)
        print(json.dumps({"W": W, "L": args.L, "n": n, "variant": names.get(var.value, str(var.value)),
                          "cells_per_s": cells.value / (ms.value / 1e3),
                          "kernel_ms": ms.value / max(nl.value, 1), "launches": nl.value,
                          "hbm_GBps_algorithmic": byts.value / (ms.value / 1e3) / 1e9}), flush=True)


if __name__ == "__main__":
    main()
