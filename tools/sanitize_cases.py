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

CASES = ("smem", "stream", "grid", "grid_parts", "grid_devices", "steps", "steps_wide", "prefix", "sim", "cost",
         "tier0", "tier1_waves", "async", "skeleton", "montecarlo")


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
    elif c == "tier0":  # the device-planned SMEM tier: classes of both domains, NaN domain
        os.environ["SPLITPLAN_STEPS_MIN_COLS"] = str(1 << 30)
        b = instances(7, 40, 10, 700, 120, float_r=False)
        p = B.plan_dp(b)
        b2 = instances(8, 40, 10, 3000, 500, float_r=True)
        p = B.plan_dp(b2)
    elif c == "tier1_waves":  # breakpoint lists in waves of a small workspace
        b = instances(9, 64, 12, 2000, 300)
        mn, full = B.dp_workspace_bytes(b)
        size = mn + (full - mn) // 4
        ws = torch.empty(size, dtype=torch.uint8, device=N.device())
        p = B.PolicyBatch.empty(b.n, b.total_layers, b.r.device)
        assert N.library().sp_plan_dp(b.struct(), p.struct(), N.ptr(ws), size, N.stream_ptr()) == 0
    elif c == "async":
        b = instances(10, 16, 12, 5000, 400)
        p = B.plan_dp_async(b).finish()
    elif c == "skeleton":
        from paper_2410_10759_b200.throughput_sim import skeletons_device
        arr, rows, ex = skeletons_device(np.arange(64), np.zeros(64, np.int64), np.arange(64) % 7 + 1, 500, 0.057)
        torch.cuda.synchronize()
        print("skeleton ok", float(arr[:, -1].sum()))
        return
    elif c == "montecarlo":
        from paper_2410_10759_b200 import montecarlo as MC
        res = MC.run(np.arange(0, 4096, 257), horizon=300)
        print("montecarlo ok", int((res.status == 0).sum()))
        return
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
