"""Golden vectors for the cfg4 Monte-Carlo path, produced by RUNNING the reference.

    python tests/golden/gen_montecarlo.py      (build container only)

For a handful of scenario ids of the cfg4 grid, the request parameters come
from `paper_2410_10759_b200.workloads.cfg4` (plain numbers); everything after
that is the live reference `splitplan` (`/root/reference/pkg/src`):
profile -> build_problem -> run_planner(dp / greedy / all_server) ->
SweepCell -> scenarios_from_cells -> capacity_for_requests(500) ->
SimConfig(beta 0.057, horizon 2000, seed = scenario id) -> compare_variants.
The per-scenario table sizes, capacities and per-variant max / mean waits go
to tests/golden/montecarlo.json.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

REF = Path("/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2410_10759_b200 import workloads as W  # noqa: E402  (inputs only)

sys.path.insert(0, str(REF))
import splitplan.cost_model as rcm  # noqa: E402
from splitplan.evaluator import SweepCell  # noqa: E402
from splitplan.planner import run_planner  # noqa: E402
from splitplan.problem import LinkSpec, build_problem  # noqa: E402
from splitplan.throughput_sim import (CapacityDeadlockError, SimConfig,  # noqa: E402
                                      capacity_for_requests, compare_variants,
                                      scenarios_from_cells)

# 8 hand-picked corners of the grid + 56 seeded draws: 64 scenarios, 4,096 requests
SIDS = [0, 17, 130, 255, 4095, 21845, 40000, 65535] + sorted(
    int(x) for x in __import__("numpy").random.default_rng(64).choice(
        [x for x in range(65536) if x not in (0, 17, 130, 255, 4095, 21845, 40000, 65535)], 56, replace=False))
OUT = Path(__file__).resolve().parent / "montecarlo.json"


def main():
    req, _layers, off = W.cfg4(SIDS)
    client = rcm.DeviceSpec("client", float(req["client_fps"][0]))
    server = rcm.DeviceSpec("server", float(req["server_fps"][0]))
    out = []
    for s, sid in enumerate(SIDS):
        cells = []
        for k in range(off[s], off[s + 1]):
            name = W.CFG4_MODELS[int(req["model"][k])]
            seq = int(req["seq_len"][k])
            dl = float(req["deadline_s"][k])
            link = LinkSpec(float(req["uplink_bps"][k]), float(req["downlink_bps"][k]),
                            float(req["propagation_s"][k]))
            layers = rcm.profile(rcm.build_preset(name, seq), client, server)
            prob = build_problem(layers, link, dl, unit_s=float(req["unit_s"][k]))
            for planner in ("dp", "greedy", "all_server"):
                pol = run_planner(planner, prob)
                cells.append(SweepCell(model=name, seq_len=seq, deadline_s=dl,
                                       uplink_bps=link.uplink_bps, downlink_bps=link.downlink_bps,
                                       planner=planner, feasible=pol.feasible,
                                       server_load=pol.server_load))
        scen = scenarios_from_cells(cells)
        rec = dict(sid=sid, table_size=len(scen))
        if scen:
            cap = capacity_for_requests(scen, 500)
            rec["capacity"] = cap
            cfg = SimConfig(beta_per_ms=0.057, capacity=cap, seed=sid, policy_variant="dp",
                            horizon=2000, scenarios=tuple(scen))
            try:
                res = compare_variants(cfg)
                rec["max_wait_ms"] = [res[v].max_wait_ms for v in ("dp", "greedy", "nosplit")]
                rec["mean_wait_ms"] = [res[v].mean_wait_ms for v in ("dp", "greedy", "nosplit")]
            except CapacityDeadlockError as exc:
                rec["deadlock"] = str(exc)
        out.append(rec)
        print(rec)
    OUT.write_text(json.dumps(dict(sids=SIDS, beta_per_ms=0.057, horizon=2000, omega=500,
                                   scenarios=out), indent=1))


if __name__ == "__main__":
    main()
