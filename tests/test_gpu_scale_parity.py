"""Parity where the headline numbers are claimed (driver-run, `-m gpu`).

* the benchmark's exact batch -- bench.py's cfg2 requests (10k, seed 2000),
  solved through `Engine.solve` exactly as the timed step does -- with 2,048
  sampled requests recomputed by the oracle on every host core;
* configs[2] at full size: the 1M-request Llama-2-7B-like draw solved in one
  call, 1,000 sampled requests against the oracle.

Bit-exact: placement, integer latency, feasibility, and client value / server
load as float64 bit patterns.
"""

from __future__ import annotations

import os
from multiprocessing import get_context

import numpy as np
import pytest

from conftest import same_float
from oracle import splitplan_oracle as O

pytestmark = pytest.mark.gpu


def _layer_dicts(layers):
    return [dict(kind=l.kind.value, hidden_dim=l.hidden_dim, heads=l.heads, ffn_dim=l.ffn_dim,
                 out_dim=l.out_dim, seq_divisor=l.seq_divisor) for l in layers]


def _oracle_job(job):
    layers, s, cf, sf, up, down, prop, dl, unit, sac = job
    r, cs, ss, tau = O.profile_arrays(layers, int(s), cf, sf)
    inst = O.instance_from_profile(r, cs, ss, tau, up, down, prop, dl, unit, sac=sac)
    return O.plan_dp(inst)


def _oracle_many(req, idx, layer_dicts):
    jobs = [(layer_dicts[int(req["model"][k])], req["seq_len"][k], float(req["client_fps"][k]),
             float(req["server_fps"][k]), float(req["uplink_bps"][k]), float(req["downlink_bps"][k]),
             float(req["propagation_s"][k]), float(req["deadline_s"][k]), float(req["unit_s"][k]),
             bool(req["flags"][k] & 2)) for k in idx]
    procs = max(1, min(os.cpu_count() or 1, 64))
    with get_context("fork").Pool(procs) as pool:
        return pool.map(_oracle_job, jobs, chunksize=max(1, len(jobs) // (4 * procs)))


def _solve_and_compare(req, layer_lists, idx):
    import torch
    from paper_2410_10759_b200 import _native as N
    from paper_2410_10759_b200.requests import Engine, RequestBatch
    eng = Engine(layer_lists)
    dev = RequestBatch.from_numpy(**req).to(N.device())
    n = len(req["seq_len"])
    total = int(eng.n_layers[req["model"]].sum())
    sol = eng.solve(dev, total, eng.layer_offsets(dev))
    torch.cuda.synchronize()
    assert int(sol.status.abs().sum()) == 0
    host = sol.policies.to_host()
    off = sol.layer_off.cpu().numpy()
    del sol
    exp = _oracle_many(req, idx, [_layer_dicts(l) for l in layer_lists])
    for q, k in enumerate(idx):
        e = exp[q]
        a, b = off[k], off[k + 1]
        assert tuple(host["pi"][a:b]) == tuple(e["pi"]), k
        assert same_float(host["client_value"][k], e["client_value"]), k
        assert same_float(host["server_load"][k], e["server_load"]), k
        assert host["integer_latency"][k] == e["integer_latency"], k
        assert bool(host["feasible"][k]) == bool(e["feasible"]), k
    return host, n


def test_bench_batch_2048_sampled(gpu):
    """bench.py's own batch (cfg2, 10k requests, seed 2000) through Engine.solve,
    2,048 requests against the oracle (every 5th, plus the 48 with the widest
    and narrowest deadlines)."""
    import bench
    from paper_2410_10759_b200 import cost_model as cm
    req = bench.cfg2_requests(10_000, 2000)
    layers = [cm.build_preset("gpt2-24", 128).layers]
    f = req["deadline_s"] / req["unit_s"]
    idx = np.unique(np.concatenate([np.arange(0, 10_000, 5), np.argsort(f)[:24], np.argsort(f)[-24:]]))[:2048]
    assert len(idx) >= 2000
    host, n = _solve_and_compare(req, layers, idx)
    assert n == 10_000 and host["feasible"].mean() > 0.5


def test_cfg3_million_requests_1000_sampled(gpu):
    """configs[2] at full size: all 1M requests in one Engine.solve, 1,000
    sampled (seeded) against the oracle."""
    from paper_2410_10759_b200 import workloads as W
    req, layers = W.cfg3(1_000_000)
    idx = np.sort(np.random.default_rng(1000).choice(1_000_000, 1000, replace=False))
    host, n = _solve_and_compare(req, layers, idx)
    assert n == 1_000_000
