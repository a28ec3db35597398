"""K1 cost table, integerization, Eq. (1), sweeps and the K4 replay on the GPU,
against the reference's golden vectors (bit-exact)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import GOLDEN, load_json, load_npz, same_float

pytestmark = pytest.mark.gpu


def _spec(case, docs):
    from paper_2410_10759_b200 import cost_model as cm
    if case["model"] in cm.PRESET_NAMES:
        return cm.build_preset(case["model"], case["seq_len"])
    doc = docs[case["model"]]
    layers = []
    for e in doc["layers"]:
        kw = dict(e)
        kind = cm.LayerKind(kw.pop("kind"))
        for key in ("flop_coeffs", "mem_coeffs"):
            if kw.get(key) is not None:
                kw[key] = tuple(float(v) for v in kw[key])
        layers.append(cm.LayerSpec(kind=kind, **kw))
    return cm.ModelSpec(doc["name"], tuple(layers), case["seq_len"])


def test_profile_matches_reference(gpu):
    from paper_2410_10759_b200 import cost_model as cm
    doc = load_json("cost_model.json")
    cases = doc["cases"]
    for metric in ("flop", "memory"):
        sub = [c for c in cases if c["metric"] == metric]
        specs = [_spec(c, doc["specs"]) for c in sub]
        profs = cm.profile_many(specs, [cm.DeviceSpec("c", c["client_fps"]) for c in sub],
                                [cm.DeviceSpec("s", c["server_fps"]) for c in sub], metric)
        for c, prof in zip(sub, profs):
            for key in ("r", "client_time_s", "server_time_s", "tau_bytes"):
                got = np.array([getattr(p, key) for p in prof])
                assert np.array_equal(got, np.array(c[key])), (c["model"], c["seq_len"], key)
    for c in doc["calibrate"]:
        assert cm.calibrate(cm.build_preset(c["model"], c["seq_len"]), c["seq_len"],
                            c["target"]).flops_per_s == c["fps"]


def test_to_units_matches_reference(gpu):
    from paper_2410_10759_b200.problem import budget_units, to_units
    z = load_npz("units")
    t = z["times"]
    for key in z:
        if not key.startswith("units_"):
            continue
        mode, unit = key[len("units_"):].split("_", 1)
        np.testing.assert_array_equal(to_units(t, float(unit), mode), z[key], err_msg=key)
        bk = "budget_" + key[len("units_"):]
        sample = range(0, len(t), 7)
        got = [budget_units(float(t[j]), float(unit), mode) for j in sample]
        assert got == [int(z[bk][j]) for j in sample], key


def test_build_problem_and_policies_match_reference(gpu):
    from paper_2410_10759_b200 import cost_model as cm
    from paper_2410_10759_b200.evaluator import latency_of
    from paper_2410_10759_b200.planner import plan_many
    from paper_2410_10759_b200.problem import LinkSpec, build_problem
    doc = load_json("build_problem.json")
    client = cm.DeviceSpec("client", doc["client_fps"])
    server = cm.DeviceSpec("server", doc["server_fps"])
    probs = []
    for row in doc["rows"]:
        spec = cm.build_preset(row["model"], row["seq_len"])
        prof = cm.profile(spec, client, server, row["metric"])
        p = build_problem(prof, LinkSpec(row["up"], row["down"], row["prop"]), row["deadline"],
                          unit_s=row["unit"], source_at_client=row["sac"], rounding=row["mode"],
                          zero_server_time=row["zst"])
        assert list(p.client_units) == row["i"] and list(p.server_units) == row["s"]
        assert list(p.up_units) == row["u"] and list(p.down_units) == row["d"]
        assert p.budget == row["budget"]
        assert list(p.up_s) == row["up_s"] and list(p.down_s) == row["down_s"]
        probs.append(p)
    for name in ("dp", "greedy", "all_server", "all_client"):
        pols = plan_many(name, probs)
        for row, p, pol in zip(doc["rows"], probs, pols):
            exp = row["policies"][name]
            assert list(pol.pi) == exp["pi"], (row["model"], name)
            assert same_float(pol.client_value, exp["client_value"])
            assert same_float(pol.server_load, exp["server_load"])
            assert pol.integer_latency == exp["integer_latency"] and pol.feasible == exp["feasible"]
        for row, p, pol in list(zip(doc["rows"], probs, pols))[::9]:
            assert same_float(latency_of(pol.pi, p), row["policies"][name]["latency_s"])


def test_sweeps_csv_byte_identical(gpu):
    from paper_2410_10759_b200 import cost_model as cm
    from paper_2410_10759_b200.evaluator import SweepGrid, run_sweep, sweep_csv_text
    from paper_2410_10759_b200.problem import LinkSpec
    ref = cm.build_preset("bert-12", 4096)
    grid = SweepGrid(models=("bert-12", "gpt2-24", "vanilla-6x6"), seq_lens=(256, 1024, 4096),
                     deadlines_s=(32.0, 16.0, 8.0, 4.0),
                     links=tuple(LinkSpec(b, b, 0.01) for b in (3e7, 2e8, 1e9)),
                     client=cm.calibrate(ref, 4096, 7.727, "client"),
                     server=cm.calibrate(ref, 4096, 0.0979, "server"))
    assert sweep_csv_text(run_sweep(grid)) == (GOLDEN / "sweep_acceptance.csv").read_text()
    small = SweepGrid(models=("bert-12", "cmt-like"), seq_lens=(64, 500),
                      deadlines_s=(2.0, 1.0, 0.5, 0.01),
                      links=(LinkSpec(1e7, 1e7, 0.01), LinkSpec(1e9, 5e8, 0.0)),
                      client=cm.DeviceSpec("client", 2e9), server=cm.DeviceSpec("server", 2e12),
                      rounding="paper", source_at_client=False, metric="memory")
    assert sweep_csv_text(run_sweep(small, jobs=8)) == (GOLDEN / "sweep_small.csv").read_text()


def test_simulator_matches_reference(gpu):
    from paper_2410_10759_b200 import throughput_sim as ts
    z = load_npz("sim")
    table = tuple(ts.Scenario(f"s{k}", float(z["scen_deadline"][k]), float(z["scen_dp"][k]),
                              float(z["scen_greedy"][k]), float(z["scen_nosplit"][k]))
                  for k in range(len(z["scen_dp"])))
    cap = float(z["capacity"][0])
    for tag, beta in (("b57", 0.057), ("b45", 0.045)):
        cfg = ts.SimConfig(beta_per_ms=beta, capacity=cap, seed=7, policy_variant="dp",
                           horizon=15000, scenarios=table)
        res = ts.compare_variants(cfg)
        for v in ts.VARIANTS:
            np.testing.assert_array_equal(res[v].admit_ms, z[f"{tag}_{v}_admit"])
            assert res[v].mean_wait_ms == float(z[f"{tag}_{v}_mean"][0])
            assert res[v].max_wait_ms == float(z[f"{tag}_{v}_max"][0])
            np.testing.assert_array_equal(res[v].cumulative_wait_ms,
                                          np.cumsum(z[f"{tag}_{v}_admit"] - z[f"{tag}_arrival"]))
    for k in range(12):
        beta, capk, seed, vi, hz = z[f"cfg{k}_params"]
        cfg = ts.SimConfig(beta_per_ms=float(beta), capacity=float(capk), seed=int(seed),
                           policy_variant=ts.VARIANTS[int(vi)], horizon=int(hz), scenarios=table)
        np.testing.assert_array_equal(ts.simulate(cfg).admit_ms, z[f"cfg{k}_admit"])


def test_simulator_reference_cases(gpu):
    """throughput_sim.py FIFO cases (reference tests/test_throughput_sim.py:128-156)."""
    from paper_2410_10759_b200 import throughput_sim as ts

    def stream(a, dmd, dur):
        n = len(a)
        return ts.Stream(np.asarray(a, float), np.zeros(n, int), np.ones(n, int),
                         np.asarray(dmd, float), np.asarray(dur, float))
    r = ts.simulate_stream(stream([0.0, 1.0], [1.0, 1.0], [5.0, 5.0]), 1.0)
    assert r.wait_ms[1] == 4.0 and r.admit_ms[1] == 5.0
    r = ts.simulate_stream(stream([0.0, 1.0, 2.0], [8.0, 5.0, 1.0], [10.0] * 3), 10.0)
    assert r.admit_ms[1] == 10.0 and r.admit_ms[2] == 10.0
    r = ts.simulate_stream(stream([0.0, 5.0], [1.0, 1.0], [5.0, 5.0]), 1.0)
    assert r.wait_ms[1] == 0.0
    with pytest.raises(ts.CapacityDeadlockError, match="demands 20"):
        ts.simulate_stream(stream([0.0], [20.0], [5.0]), 10.0)
    r = ts.simulate_stream(stream([], [], []), 1.0)
    assert r.served_count == 0 and r.mean_wait_ms == 0.0
