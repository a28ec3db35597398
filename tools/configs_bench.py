"""Measure every BASELINE.json config (beyond the cfg2 headline in bench.py).

    python tools/configs_bench.py [--configs cfg1,cfg3,cfg4,cfg5] [--cfg3-n 100000] [--cfg4-scenarios 4096]

One JSON line per config, timed with CUDA events after a warm-up:
  cfg1  bert-12 SLA sweep: 1,200 request scenarios x 4 planners (requests/s)
  cfg3  Llama-2-7B-like long sequences, W = 1e4 (DP cells/s, requests/s)
  cfg4  Monte-Carlo grid slice: plan + replay (scenarios/s, end to end incl. host table/skeleton work)
  cfg5  one 1e5 x 1e7 chain (problem cells/s; checkpoint/recompute)
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def _events():
    import torch
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def bench_requests(name, req, layers, reps=3):
    import torch
    from paper_2410_10759_b200 import _native as N
    from paper_2410_10759_b200 import batch as B
    from paper_2410_10759_b200.requests import Engine, RequestBatch
    eng = Engine(layers)
    dev = RequestBatch.from_numpy(**req).to(N.device())
    total = int(eng.n_layers[req["model"]].sum())
    off = eng.layer_offsets(dev)

    def step():
        s = eng.solve(dev, total, off)
        for which in (N.SP_GREEDY, N.SP_ALL_SERVER, N.SP_ALL_CLIENT):
            B.plan_prefix(s.instances, which)
        return s

    s = step()
    w = B.effective_budget(s.instances).cpu().numpy()
    lens = np.diff(s.layer_off.cpu().numpy())
    cells = float((lens * (w + 1)).sum())
    torch.cuda.synchronize()
    e0, e1 = _events()
    e0.record()
    for _ in range(reps):
        step()
    e1.record()
    torch.cuda.synchronize()
    sec = e0.elapsed_time(e1) / 1e3 / reps
    n = len(req["seq_len"])
    return {"config": name, "requests": n, "dp_cells": cells, "step_s": sec,
            "requests_per_s": n / sec, "dp_cells_per_s": cells / sec,
            "planners": "dp + greedy + all_server + all_client", "timing": "CUDA events, device-resident"}


def bench_cfg4(n_scen):
    import torch
    from paper_2410_10759_b200 import montecarlo as MC
    sids = np.arange(0, 65536, max(1, 65536 // n_scen))[:n_scen]
    MC.run(sids[:64])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = MC.run(sids)
    torch.cuda.synchronize()
    sec = time.perf_counter() - t0
    return {"config": "cfg4", "scenarios": len(sids), "requests": res.requests,
            "dp_cells": res.dp_cells, "wall_s": sec, "scenarios_per_s": len(sids) / sec,
            "simulated": int((res.table_size > 0).sum()),
            "timing": "wall clock of montecarlo.run (host generation, tables and skeletons included)"}


def bench_cfg5():
    import torch
    from paper_2410_10759_b200 import batch as B
    from paper_2410_10759_b200 import workloads as W
    x = W.cfg5()
    b = B.InstanceBatch.from_arrays(x["layer_off"], x["i"], x["s"], x["u"], x["d"], x["r"],
                                    x["budget"], x["sac"])
    B.plan_dp(b)
    torch.cuda.synchronize()
    e0, e1 = _events()
    e0.record()
    p = B.plan_dp(b)
    e1.record()
    torch.cuda.synchronize()
    sec = e0.elapsed_time(e1) / 1e3
    cells = 1e5 * (1e7 + 1)
    return {"config": "cfg5", "L": 100000, "W": 10000000, "problem_cells": cells, "solve_s": sec,
            "problem_cells_per_s": cells / sec, "feasible": bool(p.feasible.item()),
            "method": "grid wave kernel, checkpoint/recompute (the last segment keeps its back-pointers: 2L - K stages of DP work)", "timing": "CUDA events"}


def main():
    ap = argparse.ArgumentParser()
    import os
    os.environ.setdefault("SPLITPLAN_WS_GB", "150")  # cfg5 keeps more back-pointer stages (less recompute)
    ap.add_argument("--configs", default="cfg1,cfg3,cfg4,cfg5")
    ap.add_argument("--cfg3-n", type=int, default=100_000)
    ap.add_argument("--cfg4-scenarios", type=int, default=4096)
    args = ap.parse_args()
    from paper_2410_10759_b200 import workloads as W
    for c in args.configs.split(","):
        if c == "cfg1":
            req, layers = W.cfg1()
            out = bench_requests("cfg1", req, layers, reps=10)
        elif c == "cfg3":
            req, layers = W.cfg3(args.cfg3_n)
            out = bench_requests("cfg3", req, layers, reps=2)
        elif c == "cfg4":
            out = bench_cfg4(args.cfg4_scenarios)
        elif c == "cfg5":
            out = bench_cfg5()
        else:
            raise SystemExit(f"unknown config {c}")
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
