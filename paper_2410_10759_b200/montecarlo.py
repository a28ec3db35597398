"""Monte-Carlo scenario sweeps (BASELINE.json configs[3]).

A scenario is a workload mix of independent requests under one SLA scale
and one link bandwidth.  For every scenario the reference's own pipeline
would run, per request, `build_problem` + `run_planner` for dp / greedy /
all_server (`evaluator.py:172-208`), turn the results into a scenario table
(`throughput_sim.scenarios_from_cells`, `throughput_sim.py:133-163`), size
the server (`capacity_for_requests`, `:172-176`) and replay the three
demand variants over one seeded arrival skeleton (`compare_variants`,
`:264-272`).  Here the whole grid runs as three batched device passes:

    K1 cost table + prep + K2 + K3   every request of every scenario (dp)
    prefix kernel                    greedy and all_server on the same instances
    skeleton kernel                  one seeded arrival skeleton per scenario
                                     (numpy's default_rng stream, bit for bit)
    K4 replay                        3 runs per scenario in one launch

with the table bookkeeping (filter, coordinate sort, normalisation) on the
host and the device, exactly as the reference computes them.
Scenarios are independent, so `run(..., group=...)` shards them over ranks
and gathers the per-scenario records once at the end.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import batch as B
from . import workloads as W
from .requests import Engine, RequestBatch
from .throughput_sim import VARIANTS, replay_arrays, skeletons_device

BETA_PER_MS = 0.057
HORIZON = 2000
OMEGA_REQUESTS = 500
EXEC_MAX = 10
SIM_BLOCK = 16384  # scenarios per replay launch (bounds device memory; larger blocks measured no faster)


@dataclass
class MonteCarloResult:
    scenario_ids: np.ndarray   # [S]
    table_size: np.ndarray     # [S] scenario-table rows after the feasibility filter
    capacity: np.ndarray       # [S]
    max_wait_ms: np.ndarray    # [S, 3] dp, greedy, nosplit
    mean_wait_ms: np.ndarray   # [S, 3]
    status: np.ndarray         # [S, 3] SP_OK, SP_ERR_DEADLOCK, or -1 (empty table: not simulated)
    requests: int              # requests planned
    dp_cells: float            # DP cells solved


def solve_requests(req, layer_lists) -> dict:
    """dp / greedy / all_server server loads and feasibility for every request
    (device tensors); `req` a host dict of arrays or a device RequestBatch."""
    eng = Engine(layer_lists)
    sol = eng.solve(req if isinstance(req, RequestBatch) else RequestBatch.from_numpy(**req).to(N.device()))
    out = {"dp": sol.policies}
    out["greedy"] = B.plan_prefix(sol.instances, N.SP_GREEDY)
    out["all_server"] = B.plan_prefix(sol.instances, N.SP_ALL_SERVER)
    w_eff = B.effective_budget(sol.instances)
    lens = (sol.layer_off[1:] - sol.layer_off[:-1]).to(torch.float64)
    valid = sol.status == 0  # cost-table errors are error cells, never kept
    host = {k: dict(load=v.server_load, ok=(v.feasible != 0) & valid) for k, v in out.items()}
    host["cells"] = (lens * (w_eff + 1).to(torch.float64)).sum()
    return host


def scenario_tables(req: dict, off: np.ndarray, model_names, solved: dict):
    """Per scenario, the reference's scenario table: coordinates whose dp,
    greedy and all_server rows are feasible, sorted by (model, seq_len,
    deadline, up, down), one row per coordinate, demands normalised by the
    mean nosplit load (throughput_sim.py:133-163).  On the device.

    Returns CSR offsets over rows (host), the per-row demands [rows, 3] and
    deadlines (device)."""
    dev = N.device()
    # rank of each request's model name in sorted name order (the reference
    # sorts coordinates by name): a per-model lookup, not a sort of strings
    uniq = sorted(set(model_names))
    rank_of = torch.tensor([uniq.index(x) for x in model_names], dtype=torch.int64, device=dev)
    if isinstance(req, RequestBatch):  # already on the device
        col = lambda k, dt: getattr(req, k).to(dev, {np.int64: torch.int64, np.float64: torch.float64}[dt])
    else:
        col = lambda k, dt: torch.from_numpy(np.ascontiguousarray(req[k], dtype=dt)).to(dev)
    name_rank = rank_of[col("model", np.int64)]
    seq, dl, up, down = (col("seq_len", np.int64), col("deadline_s", np.float64), col("uplink_bps", np.float64),
                         col("downlink_bps", np.float64))
    S = len(off) - 1
    counts = torch.from_numpy(np.diff(off)).to(dev)
    scen = torch.repeat_interleave(torch.arange(S, device=dev), counts)
    keep = solved["dp"]["ok"] & solved["greedy"]["ok"] & solved["all_server"]["ok"]
    order = lexsort_tensors((down, up, dl, seq, name_rank, scen))
    order = order[keep[order]]
    # identical coordinates collapse to one row (a dict keyed by coordinate)
    dup = torch.zeros(order.numel(), dtype=torch.bool, device=dev)
    if order.numel() > 1:
        same = torch.ones(order.numel() - 1, dtype=torch.bool, device=dev)
        for k in (scen, name_rank, seq, dl, up, down):
            v = k[order]
            same &= v[1:] == v[:-1]
        dup[1:] = same
    order = order[~dup]
    rows_scen = scen[order]
    row_off = torch.zeros(S + 1, dtype=torch.int64, device=dev)
    torch.cumsum(torch.bincount(rows_scen, minlength=S), 0, out=row_off[1:])
    loads = torch.stack([solved["dp"]["load"][order], solved["greedy"]["load"][order],
                         solved["all_server"]["load"][order]], dim=1)
    norm = segment_means_device(loads[:, 2].contiguous(), row_off)  # throughput_sim.py:156, numpy-order np.mean
    demand = loads / norm[rows_scen][:, None]
    return row_off.cpu().numpy(), demand, dl[order]


def lexsort_tensors(keys) -> torch.Tensor:
    """np.lexsort(keys) (last key primary) of device tensors as successive
    stable sorts, least significant key first -- the same permutation."""
    idx = torch.arange(keys[0].numel(), device=keys[0].device)
    for k in keys:
        idx = idx[torch.sort(k[idx], stable=True).indices]
    return idx


def lexsort_device(keys, device=None) -> np.ndarray:
    """np.lexsort of host arrays, computed on the device."""
    dev = device or N.device()
    return lexsort_tensors([torch.from_numpy(np.ascontiguousarray(k)).to(dev) for k in keys]).cpu().numpy()


def segment_means_device(values: torch.Tensor, row_off: torch.Tensor) -> torch.Tensor:
    """np.mean of every CSR segment in numpy's summation order (sp_segment_sum,
    then / n); NaN for empty segments."""
    from .evaluator import segment_sums
    return segment_sums(values, row_off) / (row_off[1:] - row_off[:-1]).to(torch.float64)


def segment_means(values: np.ndarray, row_off: np.ndarray) -> np.ndarray:
    """segment_means_device of host arrays."""
    dev = N.device()
    x = torch.from_numpy(np.ascontiguousarray(values, dtype=np.float64)).to(dev)
    off = torch.from_numpy(np.ascontiguousarray(row_off, dtype=np.int64)).to(dev)
    return segment_means_device(x, off).cpu().numpy()


def run(scenario_ids=None, beta_per_ms: float = BETA_PER_MS, horizon: int = HORIZON,
        omega_requests: float = OMEGA_REQUESTS, group=None) -> MonteCarloResult:
    """The cfg4 sweep over `scenario_ids` (default: all 65,536), sharded over
    the ranks of `group` when torch.distributed is initialised."""
    import torch.distributed as dist
    sids = np.arange(16 * 16 * W.CFG4_MIXES) if scenario_ids is None else np.asarray(scenario_ids)
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    if world > 1:
        from .shard import shard_bounds
        rank = dist.get_rank(group)
        b = shard_bounds(len(sids), world)
        local = run(sids[b[rank]:b[rank + 1]], beta_per_ms, horizon, omega_requests, group=None) \
            if b[rank + 1] > b[rank] else None
        return _gather(local, sids, b, group)

    req, layer_lists, off = W.cfg4_device(sids, N.device())  # the grid expanded on the device
    solved = solve_requests(req, layer_lists)
    row_off, demand_d, dl_d = scenario_tables(req, off, W.CFG4_MODELS, solved)
    S = len(sids)
    sizes = np.diff(row_off)
    capacity = np.zeros(S)
    sim = np.flatnonzero(sizes > 0)
    # throughput_sim.py:172-176: omega x numpy-order mean of the nosplit demands
    mean_ns = segment_means_device(demand_d[:, 2].contiguous(), torch.from_numpy(row_off).to(demand_d.device))
    capacity[sim] = float(omega_requests) * mean_ns.cpu().numpy()[sim]

    max_w = np.zeros((S, 3))
    mean_w = np.zeros((S, 3))
    status = np.full((S, 3), -1, dtype=np.int32)
    dev = N.device()
    # the scenario tables live on the device; each run's demand / duration
    # columns are gathered there from the skeleton's table-row indices
    # (throughput_sim.py:189-198: duration = deadline x execution count)
    dl_ms_d = dl_d * 1000.0
    for blk in range(0, len(sim), SIM_BLOCK):
        ids = sim[blk:blk + SIM_BLOCK]
        n = len(ids)
        # the seeded skeletons, drawn on the device (numpy's stream bit for bit)
        arr_d, gidx_d, ex_d = skeletons_device(sids[ids], row_off[ids], row_off[ids + 1], horizon, beta_per_ms,
                                               EXEC_MAX)
        gidx_d = gidx_d.long()
        arr3 = arr_d[:, None, :].expand(n, 3, horizon).reshape(-1)
        dur3 = (dl_ms_d[gidx_d] * ex_d.to(torch.float64))[:, None, :].expand(n, 3, horizon).reshape(-1)
        dem3 = demand_d[gidx_d].permute(0, 2, 1).reshape(-1)
        roff = np.arange(3 * n + 1, dtype=np.int64) * horizon
        o = replay_arrays(roff, arr3, dem3, dur3, np.repeat(capacity[ids], 3), per_request=False)
        max_w[ids] = o["mx"][:3 * n].cpu().numpy().reshape(-1, 3)
        mean_w[ids] = o["mean"][:3 * n].cpu().numpy().reshape(-1, 3)
        status[ids] = o["st"][:3 * n].cpu().numpy().reshape(-1, 3)
        del o, arr3, dur3, dem3, arr_d, gidx_d, ex_d
    return MonteCarloResult(sids, sizes, capacity, max_w, mean_w, status, int(off[-1]),
                            float(solved["cells"].item()))


def _gather(local, sids, bounds, group) -> MonteCarloResult:
    """One all_gather of the fixed-size per-scenario records (scenario order)."""
    import torch.distributed as dist
    from .shard import _all_gather_padded
    dev = N.device() if dist.get_backend(group) == "nccl" else torch.device("cpu")
    n_local = 0 if local is None else len(local.scenario_ids)
    rec = torch.zeros((n_local, 12), dtype=torch.float64)
    stats = torch.zeros(2, dtype=torch.float64)
    if local is not None:
        rec[:, 0] = torch.from_numpy(local.table_size.astype(np.float64))
        rec[:, 1] = torch.from_numpy(local.capacity)
        rec[:, 2:5] = torch.from_numpy(local.max_wait_ms)
        rec[:, 5:8] = torch.from_numpy(local.mean_wait_ms)
        rec[:, 8:11] = torch.from_numpy(local.status.astype(np.float64))
        stats[0], stats[1] = local.requests, local.dp_cells
    rows = [int(bounds[r + 1] - bounds[r]) for r in range(len(bounds) - 1)]
    parts = _all_gather_padded(rec.to(dev), rows, group)
    dist.all_reduce(stats_d := stats.to(dev), group=group)
    allrec = torch.cat(parts).cpu().numpy()
    st = stats_d.cpu().numpy()
    return MonteCarloResult(np.asarray(sids), allrec[:, 0].astype(np.int64), allrec[:, 1],
                            allrec[:, 2:5], allrec[:, 5:8], allrec[:, 8:11].astype(np.int32),
                            int(st[0]), float(st[1]))


__all__ = ["MonteCarloResult", "run", "solve_requests", "scenario_tables", "VARIANTS"]
