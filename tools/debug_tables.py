"""Debug helper: full DP tables of battery instances under each forced kernel
variant vs the global-row variant; prints the first differing cell."""

import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    from conftest import Battery
    from paper_2410_10759_b200 import planner as P
    name = sys.argv[1] if len(sys.argv) > 1 else "battery_wide"
    bat = Battery(name)
    probs = bat.problems()
    for k, prob in enumerate(probs[: int(sys.argv[2]) if len(sys.argv) > 2 else 6]):
        tabs = {}
        for v in ("global", "cluster", "smem"):
            os.environ["SPLITPLAN_DP_VARIANT"] = v
            t = P.build_dp_tables(prob)
            tabs[v] = (t.client, t.server)
        ref = tabs["global"]
        for v in ("cluster", "smem"):
            for name_, a, b in (("C", tabs[v][0], ref[0]), ("S", tabs[v][1], ref[1])):
                diff = np.argwhere(~((a == b) | (np.isnan(a) & np.isnan(b))))
                if diff.size:
                    r, c = diff[0]
                    print(f"inst {k} L={prob.n_layers} W+1={a.shape[1]} {v} {name_}: {len(diff)} diffs, "
                          f"first at k={r} j={c}: {a[r, c]} vs {b[r, c]}", flush=True)
                else:
                    print(f"inst {k} W+1={a.shape[1]} {v} {name_}: equal", flush=True)


if __name__ == "__main__":
    main()
