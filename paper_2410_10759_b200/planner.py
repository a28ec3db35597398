"""Placement planners -- drop-in for `splitplan.planner`.

Every planner runs on the GPU through the C ABI:

* `plan_dp`          -> `sp_plan_dp` (prep + K2 DP stage + K3 backtrack)
* `build_dp_tables`  -> `sp_build_dp_tables`
* `plan_greedy` / `plan_trivial` -> `sp_plan_prefix` (warp-scan split points)
* `plan_oracle`      -> `sp_plan_exhaustive`

`plan_many` / `plan_batch` are the batched forms used by sweeps.  Results are
bit-identical to the reference (planner.py) on the same integer instance.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path
from typing import Sequence

import numpy as np

from . import _native as N
from . import batch as B
from .problem import PlanProblem

ORACLE_MAX_LAYERS = 24
PLANNER_NAMES = ("dp", "greedy", "all_server", "all_client", "oracle")

__all__ = ["PlacementPolicy", "DpTables", "PLANNER_NAMES", "ORACLE_MAX_LAYERS", "plan_dp",
           "plan_greedy", "plan_trivial", "plan_oracle", "run_planner", "build_dp_tables",
           "policy_to_dict", "save_policy", "plan_many", "plan_batch"]

_BACKTRACE_MSG = "no predecessor reproduces the stored value"


@dataclass(frozen=True)
class PlacementPolicy:
    """pi (1 = client, 0 = server) with its client value, server load, unit
    latency and feasibility flag (planner.py:42-51)."""

    planner: str
    pi: tuple[int, ...]
    client_value: float
    server_load: float
    integer_latency: int
    feasible: bool


@dataclass
class DpTables:
    """Budget-indexed tables C (layer k on the client) and S (on the server),
    shape (L+1, W_eff+1), unreachable = -inf (planner.py:54-66)."""

    client: np.ndarray
    server: np.ndarray


def _policies(name: str, host: dict, layer_off: np.ndarray) -> list[PlacementPolicy]:
    out = []
    for k in range(len(layer_off) - 1):
        if host["status"][k] == N.SP_ERR_BACKTRACE:
            raise AssertionError(_BACKTRACE_MSG)
        pi = host["pi"][layer_off[k]:layer_off[k + 1]]
        out.append(PlacementPolicy(planner=name, pi=tuple(int(v) for v in pi),
                                   client_value=float(host["client_value"][k]),
                                   server_load=float(host["server_load"][k]),
                                   integer_latency=int(host["integer_latency"][k]),
                                   feasible=bool(host["feasible"][k])))
    return out


def _check_must(must_end_at):
    if must_end_at not in (None, "client", "server"):
        raise ValueError(f"must_end_at must be 'client' or 'server', got {must_end_at!r}")


def plan_batch(name: str, batch: B.InstanceBatch) -> B.PolicyBatch:
    """Run planner `name` over a device batch; results stay on the device."""
    key = name.replace("-", "_")
    if key == "dp":
        return B.plan_dp(batch)
    if key == "greedy":
        return B.plan_prefix(batch, N.SP_GREEDY)
    if key == "all_server":
        return B.plan_prefix(batch, N.SP_ALL_SERVER)
    if key == "all_client":
        return B.plan_prefix(batch, N.SP_ALL_CLIENT)
    if key == "oracle":
        lens = batch.n_layers_host
        if lens is None:  # e.g. a cost-table batch: lengths from the device offsets
            lens = np.diff(batch.layer_off.cpu().numpy())
        if lens.size and int(lens.max()) > ORACLE_MAX_LAYERS:
            raise ValueError(f"oracle limited to {ORACLE_MAX_LAYERS} layers, got {int(lens.max())}")
        return B.plan_exhaustive(batch)
    raise ValueError(f"unknown planner {name!r}")


def plan_many(name: str, problems: Sequence[PlanProblem],
              must_end_at: Sequence[str | None] | None = None) -> list[PlacementPolicy]:
    """One planner over many instances in a single batched GPU call."""
    problems = list(problems)
    if not problems:
        return []
    if must_end_at is not None:
        for m in must_end_at:
            _check_must(m)
    key = name.replace("-", "_")
    label = key if key in PLANNER_NAMES else name
    off = np.zeros(len(problems) + 1, dtype=np.int64)
    np.cumsum([p.n_layers for p in problems], out=off[1:])
    prefix = {"greedy": N.SP_GREEDY, "all_server": N.SP_ALL_SERVER, "all_client": N.SP_ALL_CLIENT}.get(key)
    if (key == "dp" or prefix is not None) and len(problems) <= SCALAR_BATCH and int(off[-1]) <= SCALAR_LAYERS:
        # a few problems (the scalar drop-in calls): one library call, host
        # arrays in and out (sp_plan_dp_host / sp_plan_prefix_host)
        cat = lambda f: np.concatenate([np.asarray(getattr(p, f)) for p in problems])
        must = None if must_end_at is None else \
            np.array([-1 if m is None else (1 if m == "client" else 0) for m in must_end_at], dtype=np.int8)
        host = B.plan_dp_host(off, cat("client_units"), cat("server_units"), cat("up_units"), cat("down_units"),
                              cat("r"), [p.budget for p in problems], [p.source_at_client for p in problems],
                              must, prefix=prefix)
        return _policies(label, host, off)
    batch = B.InstanceBatch.from_problems(problems, must_end_at)
    res = plan_batch(name, batch)
    return _policies(label, res.to_host(), off)


# problems per call (and their layers) below which plan_many("dp") takes the
# one-call host path
SCALAR_BATCH = 64
SCALAR_LAYERS = 1 << 16


def plan_dp(problem: PlanProblem, must_end_at: str | None = None) -> PlacementPolicy:
    """Maximum client value within the unit budget (planner.py:182-202).

    `must_end_at` pins the last layer's side; an infeasible instance returns
    the all-server placement with feasible=False."""
    _check_must(must_end_at)
    return plan_many("dp", [problem], None if must_end_at is None else [must_end_at])[0]


def build_dp_tables(problem: PlanProblem) -> DpTables:
    """The full (L+1) x (W_eff+1) tables, computed by the DP stage kernel."""
    C, S = B.build_dp_tables(B.InstanceBatch.from_problems([problem]))
    return DpTables(client=C.cpu().numpy(), server=S.cpu().numpy())


def plan_greedy(problem: PlanProblem) -> PlacementPolicy:
    """Longest client prefix whose split latency fits the budget (planner.py:205-214)."""
    return plan_many("greedy", [problem])[0]


def plan_trivial(problem: PlanProblem, side: str) -> PlacementPolicy:
    """All-server or all-client placement (planner.py:217-225)."""
    if side not in ("all_server", "all_client"):
        raise ValueError(f"side must be 'all_server' or 'all_client', got {side!r}")
    return plan_many(side, [problem])[0]


def plan_oracle(problem: PlanProblem, chunk: int = 1 << 16) -> PlacementPolicy:
    """Exhaustive search over all 2^L placements, L <= 24 (planner.py:228-268).

    `chunk` is accepted for signature compatibility; the GPU kernel strides
    the masks itself."""
    if problem.n_layers > ORACLE_MAX_LAYERS:
        raise ValueError(f"oracle limited to {ORACLE_MAX_LAYERS} layers, got {problem.n_layers}")
    return plan_many("oracle", [problem])[0]


def run_planner(name: str, problem: PlanProblem) -> PlacementPolicy:
    """Dispatch by name; '-' and '_' are interchangeable (planner.py:271-282)."""
    key = name.replace("-", "_")
    if key == "dp":
        return plan_dp(problem)
    if key == "greedy":
        return plan_greedy(problem)
    if key == "oracle":
        return plan_oracle(problem)
    if key in ("all_server", "all_client"):
        return plan_trivial(problem, key)
    raise ValueError(f"unknown planner {name!r}")


def policy_to_dict(policy: PlacementPolicy) -> dict:
    return {"planner": policy.planner, "pi": list(policy.pi), "server_load": policy.server_load,
            "client_value": policy.client_value, "integer_latency": policy.integer_latency,
            "feasible": policy.feasible}


def save_policy(path, policy: PlacementPolicy) -> None:
    Path(path).write_text(json.dumps(policy_to_dict(policy), indent=2, sort_keys=True) + "\n")
