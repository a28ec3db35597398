"""Small instances of every kernel for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck).  Results are checked for self-consistency only
(sanitizer runs are slow and the parity suite covers values).

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py --case stream
"""
import argparse
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

CASES = ("smem", "stream", "grid", "grid_parts", "grid_devices", "steps", "steps_wide", "prefix", "sim", "cost")


def instances(seed, n, L, W, hi, float_r=False):
    from paper_2410_10759_b200 import batch as B
    rng = np.random.default_rng(seed)
    off = np.arange(n + 1, dtype=np.int64) * L
    r = rng.random(n * L) * 50 if float_r else rng.integers(0, 9, n * L).astype(float)
    return B.InstanceBatch.from_arrays(off, rng.integers(0, hi, n * L), rng.integers(0, hi, n * L),
                                       rng.integers(0, hi, n * L), rng.integers(0, hi, n * L), r,
                                       np.full(n, W), (np.arange(n) % 2).astype(np.uint8))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", choices=CASES, required=True)
    args = ap.parse_args()
    import torch
    from paper_2410_10759_b200 import _native as N
    from paper_2410_10759_b200 import batch as B
    c = args.case
    if c in ("smem", "stream", "grid", "steps"):
        os.environ["SPLITPLAN_DP_VARIANT"] = c
        b = instances(1, 3, 12, 5000 if c != "smem" else 900, 400)
        p = B.plan_dp(b)
    elif c == "steps_wide":  # rows that outgrow the tier-1 lists: wide tier and dense fallback
        b = instances(2, 2, 300, 30000, 60, float_r=True)
        p = B.plan_dp(b)
    elif c == "grid_parts":
        os.environ.update(SPLITPLAN_DP_VARIANT="grid", SPLITPLAN_GRID_PARTS="2", SPLITPLAN_GRID_SEGMENT="5")
        b = instances(3, 1, 16, 20000, 400)
        p = B.plan_dp(b)
    elif c == "grid_devices":
        os.environ.update(SPLITPLAN_DP_VARIANT="grid", SPLITPLAN_GRID_SEGMENT="5")
        b = instances(4, 1, 16, 20000, 400)
        p = B.plan_dp(b, devices=[torch.cuda.current_device()] * 2)
    elif c == "prefix":
        b = instances(5, 4, 20, 3000, 400)
        p = B.plan_prefix(b, N.SP_GREEDY)
    elif c == "sim":
        from paper_2410_10759_b200 import throughput_sim as ts
        rng = np.random.default_rng(6)
        arr = np.cumsum(rng.exponential(5.0, 300))
        res = ts.simulate_stream(ts.Stream(arr, np.zeros(300, int), np.ones(300, int),
                                           rng.uniform(0.5, 3.0, 300), rng.uniform(5.0, 60.0, 300)), 6.0)
        print("sim ok", res.served_count)
        return
    elif c == "cost":
        from paper_2410_10759_b200 import workloads as W
        from paper_2410_10759_b200.requests import Engine, RequestBatch
        req, layers = W.cfg2(8, 7)
        eng = Engine(layers)
        s = eng.solve(RequestBatch.from_numpy(**req).to(N.device()))
        p = s.policies
    torch.cuda.synchronize()
    h = p.to_host()
    print(c, "ok", int(h["feasible"].sum()), int(np.abs(h["status"]).sum()))


if __name__ == "__main__":
    main()
