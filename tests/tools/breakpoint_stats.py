"""Breakpoints per DP row on the BASELINE workloads (test infrastructure, CPU).

The breakpoint-list kernels (paper_2410_10759_b200/csrc/dp_steps.cuh) hold a
DP row as the columns where its value changes.  This script measures, with
the oracle's dense tables (oracle/splitplan_oracle.py, reference-pinned),
how many breakpoints the rows of seeded cfg1 / cfg2 / cfg3 instances have,
and checks on a sample that the list form reproduces the dense tables
exactly (a numpy restatement of the list recurrence).

    python tests/tools/breakpoint_stats.py [--n 40] > profiles/r02/steps/breakpoints.json
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

from oracle import splitplan_oracle as O  # noqa: E402

NEG = -np.inf


def _shift(row, h, W):
    c, v = row
    c = c + h
    keep = c <= W
    return c[keep], v[keep]


def _vmax(a, b):
    """Pointwise max of two non-decreasing step functions (cols asc, vals asc)."""
    ca, va = a
    cb, vb = b
    cols = np.union1d(ca, cb)
    xa = np.concatenate([[NEG], va])[np.searchsorted(ca, cols, side="right")]
    xb = np.concatenate([[NEG], vb])[np.searchsorted(cb, cols, side="right")]
    x = np.maximum(xa, xb)
    keep = np.ones(len(x), bool)
    keep[1:] = x[1:] != x[:-1]
    keep &= x != NEG
    return cols[keep], x[keep]


def list_rows(inst):
    """planner.py:139-142 on breakpoint lists: [(C_k, S_k)] for k = 0..L."""
    W = O.effective_budget(inst)
    z = (np.array([0], np.int64), np.array([0.0]))
    e = (np.zeros(0, np.int64), np.zeros(0))
    C, S = (z, e) if inst["sac"] else (e, z)
    rows = [(C, S)]
    for k in range(len(inst["r"])):
        i, s, u, d = (int(inst[x][k]) for x in "isud")
        cm = _vmax(_shift(C, i, W), _shift(S, i + d, W))
        cv = cm[1] + inst["r"][k]
        keep = np.ones(len(cv), bool)
        keep[1:] = cv[1:] != cv[:-1]
        C, S = (cm[0][keep], cv[keep]), _vmax(_shift(S, s, W), _shift(C, s + u, W))
        rows.append((C, S))
    return rows, W


def densify(row, W):
    c, v = row
    out = np.full(W + 1, NEG)
    for t in range(len(c)):
        out[c[t]:(c[t + 1] if t + 1 < len(c) else W + 1)] = v[t]
    return out


def instances(cfg: str, n: int):
    from paper_2410_10759_b200 import workloads as Wk
    req, _ = {"cfg1": lambda: Wk.cfg1(), "cfg2": lambda: Wk.cfg2(n, 2000), "cfg3": lambda: Wk.cfg3(n, 3)}[cfg]()
    names = {"cfg1": "bert-12", "cfg2": "gpt2-24"}
    layers = O.preset_layers(names[cfg]) if cfg in names else None
    out = []
    for k in range(min(n, len(req["seq_len"]))):
        if layers is None:  # cfg3: the Llama-2-7B-like chain as layer dicts
            from paper_2410_10759_b200 import workloads as Wk2
            layers = [dict(kind=l.kind.value, hidden_dim=l.hidden_dim, heads=l.heads, ffn_dim=l.ffn_dim,
                           out_dim=l.out_dim, seq_divisor=l.seq_divisor) for l in Wk2.llama2_7b_layers()]
        r, cs, ss, tau = O.profile_arrays(layers, int(req["seq_len"][k]), req["client_fps"][k], req["server_fps"][k])
        out.append(O.instance_from_profile(r, cs, ss, tau, req["uplink_bps"][k], req["downlink_bps"][k],
                                           req["propagation_s"][k], req["deadline_s"][k], req["unit_s"][k]))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=40)
    ap.add_argument("--check", type=int, default=4, help="instances per config checked against dense tables")
    args = ap.parse_args()
    doc = {}
    for cfg in ("cfg1", "cfg2", "cfg3"):
        mx = []
        for q, inst in enumerate(instances(cfg, args.n)):
            rows, W = list_rows(inst)
            mx.append(max(max(len(a[0]), len(b[0])) for a, b in rows))
            if q < args.check:
                C, S = O.dp_tables(inst)
                for k, (a, b) in enumerate(rows):
                    assert np.array_equal(densify(a, W), C[k]) and np.array_equal(densify(b, W), S[k]), (cfg, q, k)
        mx = np.array(mx)
        doc[cfg] = {"instances": int(mx.size), "max_breakpoints_per_row": {
            "median": float(np.median(mx)), "p90": float(np.percentile(mx, 90)), "max": int(mx.max())},
            "dense_tables_checked": min(args.check, int(mx.size))}
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()
