"""Golden outputs of the reference CLI (`splitplan.cli.main`), produced by RUNNING it.

    python tests/golden/gen_cli.py      (build container only)

Each case is (argv, input files); the outputs (profile / policy JSON, sweep
CSV, simulation CSV + summary files) and the exit codes go under
tests/golden/cli/<case>/.  Manifests are kept without their wall-clock
`duration_s`.  tests/test_gpu_cli.py replays the same argv through
`paper_2410_10759_b200.cli.main` and compares byte for byte.
"""

from __future__ import annotations

import json
import os
import shutil
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
from splitplan.cli import main  # noqa: E402

OUT = Path(__file__).resolve().parent / "cli"

TOY_PROFILE = {"model": "toy", "seq_len": 4, "metric": "flop", "layers": [
    {"index": 0, "kind": "embedding", "r": 1.0, "client_time_s": 4.0, "server_time_s": 0.0, "tau_bytes": 12.5e6},
    {"index": 1, "kind": "attention", "r": 1.0, "client_time_s": 4.0, "server_time_s": 0.0, "tau_bytes": 12.5e6},
    {"index": 2, "kind": "classifier", "r": 10.0, "client_time_s": 4.0, "server_time_s": 0.0, "tau_bytes": 12.5e6}]}
SCENARIO = {"uplink_bps": 1e8, "downlink_bps": 1e8, "propagation_s": 0.0, "deadline_s": 9.0, "unit_s": 1.0,
            "source_at_client": True, "rounding": "conservative"}
TIGHT = dict(SCENARIO, deadline_s=0.5)
GRID = {"models": ["bert-12", "gpt2-24"], "seq_lens": [64, 512], "deadlines_s": [2.0, 1.0, 0.25],
        "links": [{"uplink_bps": 1e7, "downlink_bps": 1e7, "propagation_s": 0.01},
                  {"uplink_bps": 1e9, "downlink_bps": 1e9, "propagation_s": 0.01}],
        "client": {"calibrate_model": "bert-12", "calibrate_seq_len": 4096, "calibrate_s": 7.727},
        "server": {"calibrate_model": "bert-12", "calibrate_seq_len": 4096, "calibrate_s": 0.0979}}

INPUTS = {"profile.json": TOY_PROFILE, "scenario.json": SCENARIO, "tight.json": TIGHT, "grid.json": GRID}

CASES = {
    "profile_bert": ["profile", "--model", "bert-12", "--seq-len", "512", "--calibrate-client", "7.727",
                     "--calibrate-server", "0.0979", "--out", "{o}/p.json"],
    "profile_memory": ["profile", "--model", "vanilla-6x6", "--seq-len", "300", "--metric", "memory",
                       "--client-tput", "1e9", "--server-tput", "1e12", "--out", "{o}/p.json"],
    "plan_dp": ["plan", "--profile", "{i}/profile.json", "--scenario", "{i}/scenario.json", "--planner", "dp",
                "--out", "{o}/plan.json"],
    "plan_greedy": ["plan", "--profile", "{i}/profile.json", "--scenario", "{i}/scenario.json", "--planner",
                    "greedy", "--out", "{o}/plan.json"],
    "plan_oracle": ["plan", "--profile", "{i}/profile.json", "--scenario", "{i}/scenario.json", "--planner",
                    "oracle", "--out", "{o}/plan.json"],
    "plan_infeasible": ["plan", "--profile", "{i}/profile.json", "--scenario", "{i}/tight.json", "--planner",
                        "dp", "--out", "{o}/plan.json"],
    "sweep": ["sweep", "--grid", "{i}/grid.json", "--out", "{o}/sweep.csv"],
    "sweep_geometric": ["sweep", "--grid", "{i}/grid.json", "--deadline-max", "4.0", "--deadline-count", "3",
                        "--out", "{o}/sweep.csv"],
    "bad_model": ["profile", "--model", "nope", "--seq-len", "8", "--client-tput", "1", "--server-tput", "1",
                  "--out", "{o}/p.json"],
}
SIM = ["simulate", "--scenarios", "{s}", "--beta", "0.057", "--seed", "7", "--horizon", "1000",
       "--out-dir", "{o}/sim"]


def run(argv, i, o, s=""):
    argv = [a.format(i=i, o=o, s=s) for a in argv]
    return main(argv)


def scrub(d: Path):
    for m in d.rglob("*manifest.json"):
        doc = json.loads(m.read_text())
        doc.pop("duration_s", None)
        m.write_text(json.dumps(doc, indent=2, sort_keys=True) + "\n")


def main_gen():
    if OUT.exists():
        shutil.rmtree(OUT)
    OUT.mkdir(parents=True)
    inp = OUT / "inputs"
    inp.mkdir()
    for name, doc in INPUTS.items():
        (inp / name).write_text(json.dumps(doc))
    codes = {}
    with tempfile.TemporaryDirectory() as tmp:
        for case, argv in CASES.items():
            o = Path(tmp) / case
            o.mkdir()
            codes[case] = run(argv, inp, o)
            shutil.copytree(o, OUT / case)
        o = Path(tmp) / "simulate"
        o.mkdir()
        codes["simulate"] = run(SIM, inp, o, s=str(OUT / "sweep" / "sweep.csv"))
        shutil.copytree(o, OUT / "simulate")
    scrub(OUT)
    (OUT / "exit_codes.json").write_text(json.dumps(codes, indent=1, sort_keys=True) + "\n")
    print(codes)


if __name__ == "__main__":
    main_gen()
