"""Where one scalar plan_dp call's time goes (GPU box): host phases of
planner.plan_many on the acceptance battery, one instance per call.

    python tools/api_breakdown.py
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch
    from paper_2410_10759_b200 import _native as N, batch as B, planner as pl, problem as pr
    z = np.load(ROOT / "tests" / "golden" / "battery_acceptance.npz")
    off = z["off"]
    probs = [pr.PlanProblem.from_costs(z["i"][off[k]:off[k + 1]], z["s"][off[k]:off[k + 1]],
                                       z["u"][off[k]:off[k + 1]], z["d"][off[k]:off[k + 1]],
                                       z["r"][off[k]:off[k + 1]], int(z["budget"][k]),
                                       source_at_client=bool(z["sac"][k])) for k in range(len(off) - 1)]
    for p in probs[:20]:
        pl.plan_dp(p)
    ph = dict(upload=0.0, struct=0.0, plan=0.0, sync=0.0, download=0.0, policies=0.0)
    lib = N.library()
    for p in probs:
        t0 = time.perf_counter()
        b = B.InstanceBatch.from_problems([p])
        t1 = time.perf_counter()
        out = B.PolicyBatch.empty(b.n, b.total_layers, b.r.device)
        s, o = b.struct(), out.struct()
        ws = N.workspace()
        t2 = time.perf_counter()
        rc = lib.sp_plan_dp(s, o, N.ptr(ws), ws.numel(), N.stream_ptr())
        t3 = time.perf_counter()
        torch.cuda.synchronize()
        t4 = time.perf_counter()
        host = out.to_host()
        t5 = time.perf_counter()
        pl._policies("dp", host, np.array([0, p.n_layers]))
        t6 = time.perf_counter()
        assert rc == 0
        for k, (a, c) in zip(ph, ((t0, t1), (t1, t2), (t2, t3), (t3, t4), (t4, t5), (t5, t6))):
            ph[k] += (c - a) * 1e3 / len(probs)
    print(json.dumps({"ms_per_call": ph, "total": sum(ph.values())}))


if __name__ == "__main__":
    main()
