"""Debug helper: run the DP on the golden build_problem rows under every forced
kernel variant and report mismatches against the reference outputs."""

import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    from paper_2410_10759_b200 import batch as B
    from paper_2410_10759_b200.problem import PlanProblem
    doc = json.loads((ROOT / "tests/golden/build_problem.json").read_text())
    rows = doc["rows"]
    probs = [PlanProblem.from_costs(r["i"], r["s"], r["u"], r["d"], np.ones(len(r["i"])), r["budget"],
                                    source_at_client=r["sac"]) for r in rows]
    from paper_2410_10759_b200 import cost_model as cm
    client = cm.DeviceSpec("c", doc["client_fps"])
    server = cm.DeviceSpec("s", doc["server_fps"])
    for p, r in zip(probs, rows):
        prof = cm.profile(cm.build_preset(r["model"], r["seq_len"]), client, server, r["metric"])
        p.r = np.array([x.r for x in prof])
    for variant in ("auto", "smem", "global", "stream", "steps"):
        os.environ["SPLITPLAN_DP_VARIANT"] = variant
        b = B.InstanceBatch.from_problems(probs)
        h = B.plan_dp(b).to_host()
        off = np.concatenate([[0], np.cumsum([p.n_layers for p in probs])])
        bad = []
        for k, r in enumerate(rows):
            if list(h["pi"][off[k]:off[k + 1]]) != r["policies"]["dp"]["pi"]:
                bad.append((k, r["model"], r["w_eff"], len(r["i"]), r["sac"]))
        print(variant, "mismatches:", len(bad), bad[:8], flush=True)


if __name__ == "__main__":
    main()
