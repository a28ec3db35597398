"""Generate the golden fixtures under tests/golden/ by RUNNING the reference.

Usage (build container only -- /root/reference does not exist on the GPU box):

    python tests/golden/gen_golden.py

Every fixture is the live reference's own output (`splitplan` imported from
/root/reference/pkg/src) on seeded inputs; nothing here is computed by the
oracle or by the CUDA engine.  The files are committed so the GPU-box tests
and the oracle self-check can use them without the reference.
"""

from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.path.insert(0, "/root/reference/pkg/tests")

from splitplan import cost_model as cm  # noqa: E402
from splitplan import throughput_sim as ts  # noqa: E402
from splitplan.evaluator import SweepGrid, latency_of, run_sweep, sweep_csv_text  # noqa: E402
from splitplan.planner import (build_dp_tables, plan_dp, plan_greedy,  # noqa: E402
                               plan_oracle, plan_trivial, _effective_budget)
from splitplan.problem import (LinkSpec, PlanProblem, budget_units,  # noqa: E402
                               build_problem, to_units)
from conftest import random_problem  # noqa: E402

OUT = Path(__file__).resolve().parent


# ---------------------------------------------------------------------------
# encoding helpers


def pack_instances(problems, must=None):
    off = np.zeros(len(problems) + 1, dtype=np.int64)
    for k, p in enumerate(problems):
        off[k + 1] = off[k] + p.n_layers
    cat = lambda f: np.concatenate([np.asarray(f(p)) for p in problems]) if problems else np.zeros(0)
    return dict(
        off=off,
        i=cat(lambda p: p.client_units).astype(np.int64),
        s=cat(lambda p: p.server_units).astype(np.int64),
        u=cat(lambda p: p.up_units).astype(np.int64),
        d=cat(lambda p: p.down_units).astype(np.int64),
        r=cat(lambda p: p.r).astype(np.float64),
        budget=np.array([p.budget for p in problems], dtype=np.int64),
        sac=np.array([p.source_at_client for p in problems], dtype=np.uint8),
        must=np.array([-1 if m is None else (1 if m == "client" else 0)
                       for m in (must or [None] * len(problems))], dtype=np.int8),
        w_eff=np.array([_effective_budget(p) for p in problems], dtype=np.int64),
    )


def pack_policies(prefix, policies, problems):
    out = {}
    out[prefix + "_pi"] = np.concatenate([np.array(p.pi, dtype=np.uint8) if p is not None
                                          else np.zeros(q.n_layers, np.uint8)
                                          for p, q in zip(policies, problems)])
    out[prefix + "_cv"] = np.array([p.client_value if p else np.nan for p in policies])
    out[prefix + "_sl"] = np.array([p.server_load if p else np.nan for p in policies])
    out[prefix + "_lat"] = np.array([p.integer_latency if p else -1 for p in policies], np.int64)
    out[prefix + "_feas"] = np.array([p.feasible if p else False for p in policies], np.uint8)
    return out


def run_dp(prob, must=None):
    try:
        return plan_dp(prob, must_end_at=must), ""
    except AssertionError as exc:
        return None, "AssertionError: " + str(exc)


def save_battery(name, problems, must=None, with_oracle=False, planners=True):
    arrs = pack_instances(problems, must)
    dps, errs = zip(*[run_dp(p, m) for p, m in zip(problems, must or [None] * len(problems))])
    arrs.update(pack_policies("dp", dps, problems))
    arrs["dp_err"] = np.array([1 if e else 0 for e in errs], np.uint8)
    if planners:
        arrs.update(pack_policies("greedy", [plan_greedy(p) for p in problems], problems))
        arrs.update(pack_policies("all_server", [plan_trivial(p, "all_server") for p in problems],
                                  problems))
        arrs.update(pack_policies("all_client", [plan_trivial(p, "all_client") for p in problems],
                                  problems))
    if with_oracle:
        arrs.update(pack_policies("oracle", [plan_oracle(p) for p in problems], problems))
    np.savez_compressed(OUT / f"{name}.npz", **arrs)
    print(name, len(problems), "instances")


# ---------------------------------------------------------------------------
# planner batteries


def gen_planner():
    # conftest.random_problem battery, same seed as the reference acceptance test
    rng = np.random.default_rng(20240817)
    probs = [random_problem(rng) for _ in range(600)]
    save_battery("battery_acceptance", probs, with_oracle=True)

    # hand fixtures (reference tests/test_planner.py) + survey-found vectors
    F = PlanProblem.from_costs
    special = [
        (F([4, 4, 4], [0, 0, 0], [1, 1, 1], [1, 1, 1], [5.0, 1.0, 5.0], 9), None),   # instance_a
        (F([4, 4, 4], [0, 0, 0], [1, 1, 1], [1, 1, 1], [1.0, 1.0, 10.0], 9), None),  # instance_b
        (F([4, 4, 4], [0, 0, 0], [1, 1, 1], [1, 1, 1], [1.0, 1.0, 10.0], 9), "server"),
        (F([4, 4, 4], [0, 0, 0], [1, 1, 1], [1, 1, 1], [1.0, 1.0, 10.0], 9), "client"),
        (F([4, 4, 4], [0, 0, 0], [1, 1, 1], [1, 1, 1], [5.0, 1.0, 5.0], 9, source_at_client=False), None),
        (F([2, 2, 2], [0, 0, 0], [5, 5, 5], [5, 5, 5], [1.0, 2.0, 3.0], 6), None),
        (F([9, 9, 9], [0, 0, 0], [0, 0, 0], [0, 0, 0], [1.0, 1.0, 1.0], 8), None),
        (F([9], [9], [9], [9], [1.0], 5), None),                                       # infeasible
        (F([5, 5, 0], [0, 0, 0], [0, 0, 0], [0, 0, 0], [1.0, 0.0, 2.0 ** 53], 9), None),  # fp absorption
        (F([0, 0], [0, 0], [0, 0], [0, 0], [3.0, 4.0], 0), None),
        (F([0, 0], [0, 0], [0, 0], [0, 0], [1.0, 0.0], 0), None),
        (F([3], [0], [0], [0], [1.0], 0), None),
        (F([4, 4, 4], [0, 0, 0], [2, 2, 2], [0, 0, 0], [1.0, 1.0, 1.0], 9), None),
        (F([3, 4, 5], [9, 9, 9], [7, 7, 7], [7, 7, 7], [1.0, 1.0, 1.0], 12), None),
        (F([3, 4, 5], [9, 9, 9], [7, 7, 7], [7, 7, 7], [1.0, 1.0, 1.0], 11), None),
        (F([1, 2, 3], [1, 1, 1], [100, 100, 100], [100, 100, 100], [1.0, -0.0, 2.0], 50), None),
        (F([0], [0], [0], [0], [0.0], 0), None),
        (F([7, 1], [1, 7], [0, 0], [0, 0], [1.0, 1.0], 10 ** 12), None),              # W clamp
        (F([1, 1, 1], [1, 1, 1], [1, 1, 1], [1, 1, 1], [math.inf, 1.0, 2.0], 5), None),  # r = inf
        (F([1, 1, 1], [1, 1, 1], [1, 1, 1], [1, 1, 1], [1.0, math.inf, 2.0], 2), None),
        (F([1, 1, 1], [1, 1, 1], [1, 1, 1], [1, 1, 1], [math.nan, 1.0, 2.0], 5), None),  # r = NaN
        (F([2, 0, 3], [0, 2, 0], [1, 0, 5], [4, 4, 0], [0.1, 0.2, 0.30000000000000004], 7), None),
    ]
    save_battery("battery_special", [p for p, _ in special], must=[m for _, m in special],
                 with_oracle=False)

    # wider/float battery: non-integral r, larger L and W, both origins
    rng = np.random.default_rng(7)
    probs = []
    for t in range(300):
        L = int(rng.integers(1, 60))
        scale = int(rng.choice([1, 5, 40]))
        i = rng.integers(0, 21 * scale, L)
        s = rng.integers(0, 6 * scale, L)
        u = rng.integers(0, 31 * scale, L)
        d = rng.integers(0, 31 * scale, L)
        kind = t % 4
        if kind == 0:
            r = rng.random(L) * 100.0
        elif kind == 1:
            r = rng.random(L) * 10.0 ** rng.integers(-3, 17, L)
        elif kind == 2:
            r = rng.integers(0, 1000, L).astype(float) * 0.1
        else:
            r = np.round(rng.random(L) * 50) / 8.0
        W = int(rng.integers(0, max(1, int(i.sum()) + 40 * scale)))
        probs.append(PlanProblem.from_costs(i, s, u, d, r, W, source_at_client=bool(rng.integers(0, 2))))
    save_battery("battery_float", probs)

    # oracle-sized battery with float r and ties for the exhaustive planner
    rng = np.random.default_rng(11)
    probs = []
    for t in range(120):
        L = int(rng.integers(1, 12))
        r = rng.integers(0, 4, L).astype(float) * (0.5 if t % 2 else 1.0)
        probs.append(PlanProblem.from_costs(rng.integers(0, 6, L), rng.integers(0, 6, L),
                                            rng.integers(0, 6, L), rng.integers(0, 6, L), r,
                                            int(rng.integers(0, 30)),
                                            source_at_client=bool(rng.integers(0, 2))))
    save_battery("battery_oracle_ties", probs, with_oracle=True)

    gen_oracle_float()

    # medium integer battery: big W with many layers (exercises tiled rows)
    rng = np.random.default_rng(13)
    probs = []
    for t in range(24):
        L = int(rng.integers(20, 140))
        W = int(rng.choice([3000, 15000, 40000, 70000]))
        hi = max(2, W // 20)
        probs.append(PlanProblem.from_costs(rng.integers(0, hi, L), rng.integers(0, hi // 8 + 1, L),
                                            rng.integers(0, hi, L), rng.integers(0, hi, L),
                                            rng.integers(0, 1000, L).astype(float)
                                            if t % 3 else rng.random(L) * 1e6,
                                            W, source_at_client=bool(t % 2)))
    save_battery("battery_wide", probs, planners=True)


def gen_oracle_float():
    """battery_oracle_float (see the comment below)."""
    # oracle battery with decimal r (0.1 + 0.2 != 0.3): subsets whose sums tie
    # in exact arithmetic differ by rounding, so the argmax depends on the
    # order numpy's x @ r (BLAS dgemv) sums in (planner.py:253); L up to 20
    # crosses the 65,536-mask chunks; a few r = inf (0 * inf = NaN values)
    rng = np.random.default_rng(29)
    vals = np.array([0.1, 0.2, 0.3, 0.7, 1.1, 0.05, 0.15, 2.2, 0.45, 3.3])
    probs = []
    for t in range(160):
        L = int(rng.integers(1, 15)) if t < 140 else int(rng.integers(17, 21))
        r = rng.choice(vals, L) * rng.choice([1.0, 1.0, 1.7], L)
        if t % 53 == 52:
            r[int(rng.integers(0, L))] = math.inf
        i = rng.integers(0, 6, L)
        probs.append(PlanProblem.from_costs(i, rng.integers(0, 6, L), rng.integers(0, 6, L),
                                            rng.integers(0, 6, L), r, int(rng.integers(0, 4 * L + 8)),
                                            source_at_client=bool(rng.integers(0, 2))))
    save_battery("battery_oracle_float", probs, with_oracle=True, planners=False)



def gen_tables():
    F = PlanProblem.from_costs
    rng = np.random.default_rng(3)
    probs = [F([4, 4, 4], [0, 0, 0], [1, 1, 1], [1, 1, 1], [5.0, 1.0, 5.0], 9),
             F([4, 4, 4], [0, 0, 0], [1, 1, 1], [1, 1, 1], [5.0, 1.0, 5.0], 9, source_at_client=False),
             F([1, 1, 1], [1, 1, 1], [1, 1, 1], [1, 1, 1], [math.inf, 1.0, 2.0], 5)]
    for _ in range(8):
        probs.append(random_problem(rng))
    arrs = pack_instances(probs)
    with np.errstate(invalid="ignore"):
        tabs = [build_dp_tables(p) for p in probs]
    arrs["C"] = np.concatenate([t.client.ravel() for t in tabs])
    arrs["S"] = np.concatenate([t.server.ravel() for t in tabs])
    np.savez_compressed(OUT / "dp_tables.npz", **arrs)
    print("dp_tables", len(probs))


# ---------------------------------------------------------------------------
# cost model, integerization, evaluator


ACCEPT_REF = cm.build_preset("bert-12", 4096)
CLIENT = cm.calibrate(ACCEPT_REF, 4096, 7.727, "client")
SERVER = cm.calibrate(ACCEPT_REF, 4096, 0.0979, "server")

LLAMA_LIKE = {
    "name": "llama2-7b-like",
    "layers": ([{"kind": "embedding", "hidden_dim": 4096, "out_dim": 32000}]
               + [{"kind": k, "hidden_dim": 4096, "heads": 32, "ffn_dim": 11008}
                  for _ in range(32) for k in ("attention", "layer_norm", "feed_forward", "layer_norm")]
               + [{"kind": "classifier", "hidden_dim": 4096, "out_dim": 32000}]),
}
CUSTOM_SPEC = {
    "name": "custom-mix",
    "layers": [
        {"kind": "embedding", "hidden_dim": 96},
        {"kind": "custom", "hidden_dim": 96, "flop_coeffs": [0.37, 1234.5, 17.25],
         "mem_coeffs": [0.5, 384.0, 3.0], "out_bytes_per_token": 192.5},
        {"kind": "attention", "hidden_dim": 96, "heads": 3, "seq_divisor": 2},
        {"kind": "custom", "hidden_dim": 48, "flop_coeffs": [1e-3, 0.1, 1e7]},
        {"kind": "feed_forward", "hidden_dim": 96, "ffn_dim": 300, "seq_divisor": 3},
        {"kind": "classifier", "hidden_dim": 96, "out_dim": 7, "seq_divisor": 5},
    ],
}


def spec_from_doc(doc, seq_len):
    layers = []
    for e in doc["layers"]:
        kw = dict(e)
        kind = cm.LayerKind(kw.pop("kind"))
        for key in ("flop_coeffs", "mem_coeffs"):
            if kw.get(key) is not None:
                kw[key] = tuple(float(v) for v in kw[key])
        layers.append(cm.LayerSpec(kind=kind, **kw))
    return cm.ModelSpec(doc["name"], tuple(layers), seq_len)


def gen_cost_model():
    docs = {"llama2-7b-like": LLAMA_LIKE, "custom-mix": CUSTOM_SPEC}
    cases = []
    for name in ("bert-12", "gpt2-24", "vanilla-6x6", "cmt-like", "llama2-7b-like", "custom-mix"):
        for s in (1, 3, 7, 64, 128, 1000, 2048, 4096, 32768):
            spec = cm.build_preset(name, s) if name in cm.PRESET_NAMES else spec_from_doc(docs[name], s)
            for metric in ("flop", "memory"):
                for cdev, sdev in ((CLIENT, SERVER), (cm.DeviceSpec("c", 1e9), cm.DeviceSpec("s", 3.3e12))):
                    prof = cm.profile(spec, cdev, sdev, metric)
                    cases.append(dict(model=name, seq_len=s, metric=metric,
                                      client_fps=cdev.flops_per_s, server_fps=sdev.flops_per_s,
                                      r=[p.r for p in prof],
                                      client_time_s=[p.client_time_s for p in prof],
                                      server_time_s=[p.server_time_s for p in prof],
                                      tau_bytes=[p.tau_bytes for p in prof],
                                      model_flops=float(cm.model_flops(spec, s))))
    cal = [dict(model=m, seq_len=s, target=t, fps=cm.calibrate(cm.build_preset(m, s), s, t).flops_per_s)
           for m in cm.PRESET_NAMES for s in (64, 4096) for t in (7.727, 0.0979, 1.0, 3e-7)]
    doc = dict(client_fps=CLIENT.flops_per_s, server_fps=SERVER.flops_per_s, cases=cases,
               calibrate=cal, specs=docs)
    (OUT / "cost_model.json").write_text(json.dumps(doc))
    print("cost_model", len(cases), "profiles")


def gen_units():
    rng = np.random.default_rng(99)
    times = np.concatenate([
        rng.uniform(0.0, 5.0, 2000),
        np.arange(0, 200) * 1e-3,
        (np.arange(0, 200) + 0.5) * 1e-3,
        np.arange(0, 50) * 0.1,
        (np.arange(1, 200) * 1e-3) * (1 + 1e-12),
        (np.arange(1, 200) * 1e-3) * (1 - 1e-12),
        (np.arange(1, 200) * 1e-3) * (1 + 1e-8),
        [0.0, 1e-300, 1e-20, 123456.789, 0.0034, 0.5, 2.5e-3, 3.5e-3, 1e6],
    ])
    out = {"times": times}
    for unit in (1e-3, 1e-4, 1e-2, 0.3, 7e-6):
        for mode in ("paper", "conservative"):
            key = f"{mode}_{unit!r}"
            out["units_" + key] = to_units(times, unit, mode)
            out["budget_" + key] = np.array([budget_units(t, unit, mode) for t in times], np.int64)
    np.savez_compressed(OUT / "units.npz", **out)
    print("units", len(times))


def gen_build_problem():
    rng = np.random.default_rng(5)
    rows = []
    for t in range(160):
        name = ["bert-12", "gpt2-24", "vanilla-6x6", "cmt-like"][t % 4]
        s = int(rng.integers(1, 5000))
        spec = cm.build_preset(name, s)
        prof = cm.profile(spec, CLIENT, SERVER, "flop" if t % 5 else "memory")
        bw_up = float(10 ** rng.uniform(6, 10))
        bw_dn = bw_up if t % 3 else float(10 ** rng.uniform(6, 10))
        prop = [0.0, 0.01, 0.002][t % 3]
        all_client = sum(p.client_time_s for p in prof)
        deadline = float(all_client * rng.uniform(0.01, 1.2))
        unit = [1e-3, deadline / 1e4, deadline / 1e5, 1e-4, 0.05][t % 5]
        mode = "paper" if t % 7 == 0 else "conservative"
        sac = bool(t % 6)
        zst = (t % 11 == 0)
        prob = build_problem(prof, LinkSpec(bw_up, bw_dn, prop), deadline, unit_s=unit,
                             source_at_client=sac, rounding=mode, zero_server_time=zst)
        pols = {k: (plan_dp(prob) if k == "dp" else plan_greedy(prob) if k == "greedy"
                    else plan_trivial(prob, k)) for k in ("dp", "greedy", "all_server", "all_client")}
        rows.append(dict(model=name, seq_len=s, metric="flop" if t % 5 else "memory",
                         up=bw_up, down=bw_dn, prop=prop, deadline=deadline, unit=unit, mode=mode,
                         sac=sac, zst=zst,
                         i=prob.client_units.tolist(), s=prob.server_units.tolist(),
                         u=prob.up_units.tolist(), d=prob.down_units.tolist(), budget=prob.budget,
                         up_s=prob.up_s.tolist(), down_s=prob.down_s.tolist(),
                         w_eff=_effective_budget(prob),
                         policies={k: dict(pi=list(p.pi), client_value=p.client_value,
                                           server_load=p.server_load,
                                           integer_latency=p.integer_latency, feasible=p.feasible,
                                           latency_s=latency_of(p.pi, prob))
                                   for k, p in pols.items()}))
    doc = dict(client_fps=CLIENT.flops_per_s, server_fps=SERVER.flops_per_s, rows=rows)
    (OUT / "build_problem.json").write_text(json.dumps(doc))
    print("build_problem", len(rows))


def gen_sweeps():
    grid = SweepGrid(models=("bert-12", "gpt2-24", "vanilla-6x6"), seq_lens=(256, 1024, 4096),
                     deadlines_s=(32.0, 16.0, 8.0, 4.0),
                     links=tuple(LinkSpec(b, b, 0.01) for b in (3e7, 2e8, 1e9)),
                     client=CLIENT, server=SERVER)
    cells = run_sweep(grid)
    (OUT / "sweep_acceptance.csv").write_text(sweep_csv_text(cells))
    small = SweepGrid(models=("bert-12", "cmt-like"), seq_lens=(64, 500),
                      deadlines_s=(2.0, 1.0, 0.5, 0.01),
                      links=(LinkSpec(1e7, 1e7, 0.01), LinkSpec(1e9, 5e8, 0.0)),
                      client=cm.DeviceSpec("client", 2e9), server=cm.DeviceSpec("server", 2e12),
                      rounding="paper", source_at_client=False, metric="memory")
    (OUT / "sweep_small.csv").write_text(sweep_csv_text(run_sweep(small)))
    print("sweeps", len(cells))
    return cells


def gen_sim(cells):
    table = tuple(ts.scenarios_from_cells(cells))
    cap = ts.capacity_for_requests(table, 500)
    out = dict(
        scen_deadline=np.array([s.deadline_s for s in table]),
        scen_dp=np.array([s.demand_dp for s in table]),
        scen_greedy=np.array([s.demand_greedy for s in table]),
        scen_nosplit=np.array([s.demand_nosplit for s in table]),
        capacity=np.array([cap]),
    )
    for beta in (0.057, 0.045):
        cfg = ts.SimConfig(beta_per_ms=beta, capacity=cap, seed=7, policy_variant="dp",
                           horizon=15000, scenarios=table)
        res = ts.compare_variants(cfg)
        arr, idx, ex = ts._skeleton(cfg)
        tag = f"b{int(beta * 1000)}"
        out[tag + "_arrival"] = arr
        out[tag + "_idx"] = idx
        out[tag + "_exec"] = ex
        for v, r in res.items():
            out[f"{tag}_{v}_admit"] = r.admit_ms
            out[f"{tag}_{v}_mean"] = np.array([r.mean_wait_ms])
            out[f"{tag}_{v}_max"] = np.array([r.max_wait_ms])
    # small seeded configs exercising stream generation across seeds/variants
    for k in range(12):
        cfg = ts.SimConfig(beta_per_ms=0.03 + 0.01 * k, capacity=cap * (0.5 + 0.05 * k),
                           seed=1000 + k, policy_variant=ts.VARIANTS[k % 3], horizon=400 + 37 * k,
                           scenarios=table)
        st = ts.generate_stream(cfg)
        res = ts.simulate_stream(st, cfg.capacity)
        out[f"cfg{k}_arrival"] = st.arrival_ms
        out[f"cfg{k}_idx"] = st.scenario_idx
        out[f"cfg{k}_exec"] = st.exec_count
        out[f"cfg{k}_admit"] = res.admit_ms
        out[f"cfg{k}_params"] = np.array([cfg.beta_per_ms, cfg.capacity, cfg.seed, k % 3, cfg.horizon])
    np.savez_compressed(OUT / "sim.npz", **out)
    print("sim")


def gen_large():
    """Full-size (W = 1e5) model-derived and cfg5-reduced instances."""
    rng = np.random.default_rng(2)
    probs = []
    for t in range(6):
        s = int(rng.integers(128, 2049))
        bw = float(np.exp(rng.uniform(np.log(3e7), np.log(1e9))))
        f = float(rng.uniform(0.05, 1.0))
        spec = cm.build_preset("gpt2-24", s)
        prof = cm.profile(spec, CLIENT, SERVER)
        dl = f * sum(p.client_time_s for p in prof)
        probs.append(build_problem(prof, LinkSpec(bw, bw, 0.01), dl, unit_s=dl / 1e5))
    rng = np.random.default_rng(5)
    L = 100_000
    probs.append(PlanProblem.from_costs(rng.integers(0, 201, L), rng.integers(0, 201, L),
                                        rng.integers(0, 201, L), rng.integers(0, 201, L),
                                        rng.integers(0, 101, L).astype(float), 1000))
    L = 1000
    probs.append(PlanProblem.from_costs(rng.integers(0, 201, L), rng.integers(0, 201, L),
                                        rng.integers(0, 201, L), rng.integers(0, 201, L),
                                        rng.integers(0, 101, L).astype(float), 100_000))
    # greedy in the reference is O(L^2) Python: only the model-derived ones get it
    save_battery("battery_large_model", probs[:6], planners=True)
    save_battery("battery_large_chain", probs[6:], planners=False)


if __name__ == "__main__":
    which = set(sys.argv[1:]) or {"planner", "tables", "cost", "units", "build", "sweep", "large"}
    if "planner" in which:
        gen_planner()
    if "oracle_float" in which and "planner" not in which:
        gen_oracle_float()
    if "tables" in which:
        gen_tables()
    if "cost" in which:
        gen_cost_model()
    if "units" in which:
        gen_units()
    if "build" in which:
        gen_build_problem()
    if "sweep" in which:
        gen_sim(gen_sweeps())
    if "large" in which:
        gen_large()
