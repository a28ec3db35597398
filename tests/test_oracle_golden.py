"""Pin the CPU oracle (oracle/splitplan_oracle.py) to the reference's golden
vectors.  These run without a GPU; once green, the oracle is a trusted
checker for the CUDA engine on inputs the fixtures do not cover."""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import GOLDEN, Battery, assert_policy, load_json, load_npz, same_float
from oracle import splitplan_oracle as O

BATTERIES = ["battery_acceptance", "battery_special", "battery_float", "battery_oracle_ties",
             "battery_wide"]


@pytest.mark.parametrize("name", BATTERIES)
def test_oracle_planners_match_reference(name):
    bat = Battery(name)
    for k in range(bat.n):
        inst = bat.inst(k)
        assert O.effective_budget(inst) == int(bat.z["w_eff"][k])
        exp = bat.expected("dp", k)
        if exp is None:
            with pytest.raises(AssertionError):
                O.plan_dp(inst, bat.must(k))
        else:
            assert_policy(O.plan_dp(inst, bat.must(k)), exp, f"{name}[{k}] dp")
        if bat.has("greedy"):
            assert_policy(O.plan_greedy(inst), bat.expected("greedy", k), f"{name}[{k}] greedy")
            for side in ("all_server", "all_client"):
                assert_policy(O.plan_trivial(inst, side), bat.expected(side, k), f"{name}[{k}] {side}")


def test_oracle_exhaustive_matches_reference():
    for name in ("battery_acceptance", "battery_oracle_ties", "battery_oracle_float"):
        bat = Battery(name)
        for k in range(0, bat.n, 3 if name == "battery_acceptance" else 1):
            inst = bat.inst(k)
            assert_policy(O.plan_exhaustive(inst), bat.expected("oracle", k), f"{name}[{k}]")


def test_oracle_dp_tables_match_reference():
    z = load_npz("dp_tables")
    off = z["off"]
    pos = 0
    for k in range(len(off) - 1):
        a, b = off[k], off[k + 1]
        inst = dict(i=z["i"][a:b], s=z["s"][a:b], u=z["u"][a:b], d=z["d"][a:b], r=z["r"][a:b],
                    budget=int(z["budget"][k]), sac=bool(z["sac"][k]))
        C, S = O.dp_tables(inst)
        cnt = C.size
        np.testing.assert_array_equal(C.ravel(), z["C"][pos:pos + cnt])
        np.testing.assert_array_equal(S.ravel(), z["S"][pos:pos + cnt])
        pos += cnt
    assert pos == z["C"].size


def test_fp_absorption_vector():
    """the stay test is fl(a + r) == C[k][j], not a >= b."""
    inst = dict(i=np.array([5, 5, 0]), s=np.zeros(3, np.int64), u=np.zeros(3, np.int64),
                d=np.zeros(3, np.int64), r=np.array([1.0, 0.0, 2.0 ** 53]), budget=9, sac=True)
    p = O.plan_dp(inst)
    assert p["pi"] == (0, 1, 1) and p["client_value"] == 2.0 ** 53 and p["integer_latency"] == 5


def _layers_from_case(case, docs):
    if case["model"] in docs:
        return docs[case["model"]]["layers"]
    return O.preset_layers(case["model"])


def test_oracle_profiles_match_reference():
    doc = load_json("cost_model.json")
    for case in doc["cases"]:
        layers = _layers_from_case(case, doc["specs"])
        r, cs, ss, tau = O.profile_arrays(layers, case["seq_len"], case["client_fps"],
                                          case["server_fps"], case["metric"])
        for got, key in ((r, "r"), (cs, "client_time_s"), (ss, "server_time_s"), (tau, "tau_bytes")):
            exp = np.array(case[key], dtype=float)
            assert np.array_equal(got, exp), (case["model"], case["seq_len"], key)
    for c in doc["calibrate"]:
        assert O.calibrate_rate(O.preset_layers(c["model"]), c["seq_len"], c["target"]) == c["fps"]


def test_oracle_units_match_reference():
    z = load_npz("units")
    t = z["times"]
    for key in z:
        if not key.startswith("units_"):
            continue
        mode, unit = key[len("units_"):].split("_", 1)
        unit = float(unit)
        np.testing.assert_array_equal(O.units_of(t, unit, mode), z[key], err_msg=key)
        bud = np.array([O.budget_of(x, unit, mode) for x in t], dtype=np.int64)
        np.testing.assert_array_equal(bud, z["budget_" + key[len("units_"):]], err_msg=key)


def test_oracle_build_problem_matches_reference():
    doc = load_json("build_problem.json")
    for row in doc["rows"]:
        layers = O.preset_layers(row["model"])
        r, cs, ss, tau = O.profile_arrays(layers, row["seq_len"], doc["client_fps"],
                                          doc["server_fps"], row["metric"])
        inst = O.instance_from_profile(r, cs, ss, tau, row["up"], row["down"], row["prop"],
                                       row["deadline"], row["unit"], row["sac"], row["mode"],
                                       row["zst"])
        for k in ("i", "s", "u", "d"):
            assert list(inst[k]) == row[k], (row["model"], k)
        assert inst["budget"] == row["budget"]
        assert list(inst["up_s"]) == row["up_s"] and list(inst["down_s"]) == row["down_s"]
        assert O.effective_budget(inst) == row["w_eff"]
        pols = {"dp": O.plan_dp(inst), "greedy": O.plan_greedy(inst),
                "all_server": O.plan_trivial(inst, "all_server"),
                "all_client": O.plan_trivial(inst, "all_client")}
        for name, exp in row["policies"].items():
            got = pols[name]
            assert list(got["pi"]) == exp["pi"], (row["model"], name)
            assert same_float(got["client_value"], exp["client_value"])
            assert same_float(got["server_load"], exp["server_load"])
            assert got["integer_latency"] == exp["integer_latency"]
            lat = O.eq1_latency(got["pi"], inst["client_s"], inst["server_s"], inst["up_s"],
                                inst["down_s"], inst["sac"])
            assert same_float(lat, exp["latency_s"]), (row["model"], name)


def test_oracle_simulator_matches_reference():
    z = load_npz("sim")
    table = np.stack([z["scen_dp"], z["scen_greedy"], z["scen_nosplit"]])
    cap = float(z["capacity"][0])
    for tag in ("b57", "b45"):
        arr, idx, ex = z[f"{tag}_arrival"], z[f"{tag}_idx"], z[f"{tag}_exec"]
        beta = 0.057 if tag == "b57" else 0.045
        a2, i2, e2 = O.skeleton(7, len(arr), beta, len(z["scen_dp"]))
        assert np.array_equal(a2, arr) and np.array_equal(i2, idx) and np.array_equal(e2, ex)
        dur = (z["scen_deadline"] * 1000.0)[idx] * ex
        for v, row in zip(("dp", "greedy", "nosplit"), table):
            admit = O.fifo_replay(arr, row[idx], dur, cap)
            np.testing.assert_array_equal(admit, z[f"{tag}_{v}_admit"])
            w = admit - arr
            assert float(np.mean(w)) == float(z[f"{tag}_{v}_mean"][0])
            assert float(np.max(w)) == float(z[f"{tag}_{v}_max"][0])
    for k in range(12):
        beta, capk, seed, vi, hz = z[f"cfg{k}_params"]
        arr, idx, ex = O.skeleton(int(seed), int(hz), beta, len(z["scen_dp"]))
        assert np.array_equal(arr, z[f"cfg{k}_arrival"])
        dur = (z["scen_deadline"] * 1000.0)[idx] * ex
        admit = O.fifo_replay(arr, table[int(vi)][idx], dur, capk)
        np.testing.assert_array_equal(admit, z[f"cfg{k}_admit"])


def test_golden_files_present():
    for f in ("battery_acceptance.npz", "battery_special.npz", "battery_float.npz",
              "battery_oracle_ties.npz", "battery_oracle_float.npz", "battery_wide.npz", "dp_tables.npz", "cost_model.json",
              "units.npz", "build_problem.json", "sweep_acceptance.csv", "sweep_small.csv",
              "sim.npz", "gen_golden.py"):
        assert (GOLDEN / f).exists(), f
