"""Per-call latency of the reference-facing Python API, and the sweep driver.

    python tools/api_latency.py --impl ours          (GPU box: the B200 drop-in)
    python tools/api_latency.py --impl reference     (build container: the live reference)

* plan_dp / plan_greedy on the reference's 600-instance acceptance battery
  (tests/golden/battery_acceptance.npz: L <= 24, small budgets), one call per
  instance, as a user of the scalar API makes them;
* run_sweep over the acceptance grid (3 models x 3 seq lens x 4 deadlines x 3
  links x 4 planners = 432 cells), jobs = 1 and jobs = all host cores.
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--impl", choices=("ours", "reference"), required=True)
    args = ap.parse_args()
    if args.impl == "reference":
        sys.path.insert(0, "/root/reference/pkg/src")
        import splitplan as P  # noqa: F401
        from splitplan import cost_model as cm, evaluator as ev, planner as pl, problem as pr
    else:
        sys.path.insert(0, str(ROOT))
        from paper_2410_10759_b200 import cost_model as cm, evaluator as ev, planner as pl, problem as pr
    z = np.load(ROOT / "tests" / "golden" / "battery_acceptance.npz")
    off = z["off"]
    probs = [pr.PlanProblem.from_costs(z["i"][off[k]:off[k + 1]], z["s"][off[k]:off[k + 1]],
                                       z["u"][off[k]:off[k + 1]], z["d"][off[k]:off[k + 1]],
                                       z["r"][off[k]:off[k + 1]], int(z["budget"][k]),
                                       source_at_client=bool(z["sac"][k])) for k in range(len(off) - 1)]
    out = {"impl": args.impl, "instances": len(probs)}
    for name, fn in (("plan_dp", pl.plan_dp), ("plan_greedy", pl.plan_greedy)):
        for p in probs[:20]:
            fn(p)  # warm-up (library load, kernels, workspace)
        t0 = time.perf_counter()
        for p in probs:
            fn(p)
        dt = time.perf_counter() - t0
        out[name] = {"calls": len(probs), "ms_per_call": 1e3 * dt / len(probs)}
    client = cm.calibrate(cm.build_preset("bert-12", 4096), 4096, 7.727)
    server = cm.calibrate(cm.build_preset("bert-12", 4096), 4096, 0.0979)
    grid = ev.SweepGrid(models=("bert-12", "gpt2-24", "vanilla-6x6"), seq_lens=(256, 1024, 4096),
                        deadlines_s=(32.0, 16.0, 8.0, 4.0),
                        links=tuple(pr.LinkSpec(b, b, 0.01) for b in (3e7, 2e8, 1e9)),
                        client=client, server=server)
    ev.run_sweep(grid)  # warm-up
    for jobs in (1, os.cpu_count() or 1):
        t0 = time.perf_counter()
        cells = ev.run_sweep(grid, jobs=jobs)
        dt = time.perf_counter() - t0
        scen = len(cells) // 4
        out[f"run_sweep_jobs{jobs}"] = {"cells": len(cells), "scenarios": scen, "s": dt,
                                        "scenarios_per_s": scen / dt}
    out["cpus"] = os.cpu_count()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
