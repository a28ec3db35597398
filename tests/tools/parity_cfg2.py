"""Bench-workload parity at scale: the bench's own cfg2 batch (10k requests,
seed 2000) solved on the GPU exactly as bench.py does, and a sample of its
placements recomputed by the oracle on every host core.

    python tests/tools/parity_cfg2.py [--sample 400]
"""
import argparse
import json
import os
import sys
from multiprocessing import get_context
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))


def _oracle(args):
    from oracle import splitplan_oracle as O
    layers, s, cf, sf, bw, prop, dl, unit = args
    r, cs, ss, tau = O.profile_arrays(layers, int(s), cf, sf)
    inst = O.instance_from_profile(r, cs, ss, tau, bw, bw, prop, dl, unit)
    p = O.plan_dp(inst)
    return (tuple(int(x) for x in p["pi"]), float(p["client_value"]), float(p["server_load"]),
            int(p["integer_latency"]), bool(p["feasible"]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sample", type=int, default=400)
    args = ap.parse_args()
    import torch
    import bench
    from oracle import splitplan_oracle as O
    from paper_2410_10759_b200 import cost_model as cm
    from paper_2410_10759_b200.requests import Engine, RequestBatch
    req = bench.cfg2_requests(10_000, 2000)
    layers = cm.build_preset("gpt2-24", 128).layers
    L = len(layers)
    eng = Engine([layers])
    dev = RequestBatch.from_numpy(**req).to("cuda")
    sol = eng.solve(dev, 10_000 * L, eng.layer_offsets(dev))
    pol = sol.policies
    pi = pol.pi.cpu().numpy().reshape(10_000, L)
    cv, sl = pol.client_value.cpu().numpy(), pol.server_load.cpu().numpy()
    il, fe = pol.integer_latency.cpu().numpy(), pol.feasible.cpu().numpy()
    idx = np.random.default_rng(7).choice(10_000, args.sample, replace=False)
    ol = O.preset_layers("gpt2-24")
    jobs = [(ol, req["seq_len"][k], req["client_fps"][k], req["server_fps"][k], req["uplink_bps"][k],
             req["propagation_s"][k], req["deadline_s"][k], req["unit_s"][k]) for k in idx]
    with get_context("fork").Pool(min(32, os.cpu_count() or 1)) as pool:
        exp = pool.map(_oracle, jobs, chunksize=1)
    bad = 0
    for k, e in zip(idx, exp):
        got = (tuple(int(x) for x in pi[k]), float(cv[k]), float(sl[k]), int(il[k]), bool(fe[k]))
        if got != e:
            bad += 1
    print(json.dumps({"workload": "bench cfg2 batch (10k requests, seed 2000)", "checked": len(idx),
                      "mismatches": bad, "feasible_in_sample": int(sum(e[4] for e in exp))}))


if __name__ == "__main__":
    main()
