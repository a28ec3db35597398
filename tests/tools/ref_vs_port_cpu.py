"""CPU calibration in the build container (needs /root/reference): the live
reference's profile -> build_problem -> plan_dp against the oracle port on the
same cfg2 requests, one process each.  Run only where the reference exists.

    PYTHONPATH=/root/reference/pkg/src python tests/tools/ref_vs_port_cpu.py [--n 8]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=6)
    args = ap.parse_args()
    from splitplan import cost_model as rcm, planner as rpl, problem as rpr  # the reference
    from oracle import splitplan_oracle as O
    from paper_2410_10759_b200 import workloads as W
    req = W.cfg2(args.n, 2000)[0]
    spec = rcm.build_preset("gpt2-24", 128) if hasattr(rcm, "build_preset") else None
    layers = O.preset_layers("gpt2-24")
    t_ref = t_port = 0.0
    cells = 0
    for k in range(args.n):
        s = int(req["seq_len"][k])
        client = rcm.DeviceSpec("c", float(req["client_fps"][k]))
        server = rcm.DeviceSpec("s", float(req["server_fps"][k]))
        t0 = time.perf_counter()
        prof = rcm.profile(rcm.build_preset("gpt2-24", s), client, server)
        prob = rpr.build_problem(prof, rpr.LinkSpec(float(req["uplink_bps"][k]), float(req["uplink_bps"][k]),
                                                    float(req["propagation_s"][k])),
                                 float(req["deadline_s"][k]), unit_s=float(req["unit_s"][k]))
        pol = rpl.plan_dp(prob)
        t_ref += time.perf_counter() - t0
        t0 = time.perf_counter()
        r, cs, ss, tau = O.profile_arrays(layers, s, req["client_fps"][k], req["server_fps"][k])
        inst = O.instance_from_profile(r, cs, ss, tau, req["uplink_bps"][k], req["uplink_bps"][k],
                                       req["propagation_s"][k], req["deadline_s"][k], req["unit_s"][k])
        p = O.plan_dp(inst)
        t_port += time.perf_counter() - t0
        assert tuple(p["pi"]) == tuple(pol.pi) and p["integer_latency"] == pol.integer_latency
        cells += len(r) * (O.effective_budget(inst) + 1)
    print(json.dumps({"requests": args.n, "cells": cells, "reference_cells_per_s_1core": cells / t_ref,
                      "port_cells_per_s_1core": cells / t_port, "port_over_reference": t_ref / t_port,
                      "placements_identical": True}))


if __name__ == "__main__":
    main()
