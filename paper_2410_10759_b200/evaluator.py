"""Policy evaluation and scenario sweeps -- drop-in for `splitplan.evaluator`.

`run_sweep` is the reference's data-parallel driver (evaluator.py:211-226).
Here the whole grid is one batched GPU pipeline instead of a per-scenario
Python loop: K1 builds every scenario's cost table, the planners run over
the batch, Eq. (1) latencies and the numpy-order sums come from kernels,
and only the SweepCell records are assembled on the host.  Output order and
every value are identical to the reference, independent of `jobs`.
"""

from __future__ import annotations

import csv
import io
import logging
from dataclasses import dataclass
from pathlib import Path
from typing import Iterable, Sequence

import numpy as np
import torch

from . import _native as N
from . import batch as B
from . import cost_model
from .cost_model import DeviceSpec
from .problem import LinkSpec, PlanProblem, raise_cost_status

logger = logging.getLogger(__name__)

SWEEP_COLUMNS = ("model", "seq_len", "deadline_s", "uplink_bps", "downlink_bps", "planner",
                 "feasible", "server_load", "offload_fraction", "latency_s", "improvement_pp",
                 "improvement_rel")
DEFAULT_PLANNERS = ("dp", "greedy", "all_server", "all_client")

__all__ = ["SweepGrid", "SweepCell", "SWEEP_COLUMNS", "DEFAULT_PLANNERS", "latency_of",
           "latency_units_of", "server_load_of", "client_value_of", "improvement_over_greedy",
           "geometric_deadlines", "run_sweep", "write_sweep_csv", "sweep_csv_text",
           "read_sweep_csv", "mean_over", "segment_sums"]


# ---------------------------------------------------------------------------
# device helpers


def segment_sums(values: torch.Tensor, off: torch.Tensor) -> torch.Tensor:
    """numpy-order np.sum of each CSR segment (sp_segment_sum)."""
    n = off.numel() - 1
    out = torch.empty(max(n, 0), dtype=torch.float64, device=values.device)
    N.check(N.library().sp_segment_sum(N.ptr(values), N.ptr(off), n, N.ptr(out), N.stream_ptr()),
            "sp_segment_sum")
    return out


def _total_r(problem: PlanProblem) -> float:
    dev = N.device()
    r = N.to_dev(problem.r, torch.float64, dev)
    off = torch.tensor([0, r.numel()], dtype=torch.int64, device=dev)
    return float(segment_sums(r, off)[0].item())


def _pi_vector(pi, problem: PlanProblem) -> np.ndarray:
    x = np.asarray(pi, dtype=float)
    if x.shape != (problem.n_layers,):
        raise ValueError(f"policy length {x.shape} does not match {problem.n_layers} layers")
    return x


def _eq1_one(x: np.ndarray, problem: PlanProblem, times) -> float:
    dev = N.device()
    batch = B.InstanceBatch.from_problems([problem])
    t = [N.to_dev(np.asarray(a, dtype=float), torch.float64, dev) for a in times]
    pi = N.to_dev((x != 0).astype(np.uint8), torch.uint8, dev)
    return float(B.latency_eq1(batch, *t, pi)[0].item())


def latency_of(pi, problem: PlanProblem) -> float:
    """Eq. (1) latency in seconds (evaluator.py:64-78), evaluated on the GPU."""
    x = _pi_vector(pi, problem)
    if not problem.has_real_times:
        raise ValueError("problem carries no real-valued times")
    return _eq1_one(x, problem, (problem.client_s, problem.server_s, problem.up_s, problem.down_s))


def latency_units_of(pi, problem: PlanProblem) -> int:
    """Eq. (1) on the integer costs (evaluator.py:81-87)."""
    x = _pi_vector(pi, problem)
    return int(round(_eq1_one(x, problem, (problem.client_units, problem.server_units,
                                           problem.up_units, problem.down_units))))


def _evaluate(pi, problem: PlanProblem) -> dict:
    x = np.asarray(pi, dtype=np.int64)
    if x.shape != (problem.n_layers,):
        raise ValueError(f"policy length {x.shape} does not match {problem.n_layers} layers")
    batch = B.InstanceBatch.from_problems([problem])
    out = B.PolicyBatch.empty(1, problem.n_layers)
    dev_pi = N.to_dev((x != 0).astype(np.uint8), torch.uint8)
    ws = N.workspace(4 * problem.n_layers)
    N.check(N.library().sp_evaluate_policy(batch.struct(), N.ptr(dev_pi), out.struct(), N.ptr(ws),
                                           ws.numel(), N.stream_ptr()), "sp_evaluate_policy")
    return out.to_host()


def server_load_of(pi, problem: PlanProblem) -> float:
    """Resource total left on the server (evaluator.py:90-95)."""
    return float(_evaluate(pi, problem)["server_load"][0])


def client_value_of(pi, problem: PlanProblem) -> float:
    return float(_evaluate(pi, problem)["client_value"][0])


def improvement_over_greedy(dp_load: float, greedy_load: float, total_r: float) -> float | None:
    """Greedy-minus-DP server load in percentage points of total r (evaluator.py:105-113)."""
    if greedy_load is None:
        return None
    if total_r <= 0:
        raise ValueError("total_r must be positive")
    return 100.0 * (greedy_load - dp_load) / total_r


def geometric_deadlines(deadline_max_s: float, count: int) -> list[float]:
    if deadline_max_s <= 0 or count < 1:
        raise ValueError("need a positive max deadline and count >= 1")
    return [deadline_max_s / (2.0 ** k) for k in range(count)]


# ---------------------------------------------------------------------------
# sweeps


@dataclass(frozen=True)
class SweepGrid:
    """Cross product models x seq_lens x deadlines x links plus fixed context."""

    models: tuple[str, ...]
    seq_lens: tuple[int, ...]
    deadlines_s: tuple[float, ...]
    links: tuple[LinkSpec, ...]
    client: DeviceSpec
    server: DeviceSpec
    planners: tuple[str, ...] = DEFAULT_PLANNERS
    metric: str = "flop"
    unit_s: float = 1e-3
    source_at_client: bool = True
    rounding: str = "conservative"

    def __post_init__(self):
        if not (self.models and self.seq_lens and self.deadlines_s and self.links
                and self.planners):
            raise ValueError("every sweep axis must be non-empty")
        if any(b >= a for a, b in zip(self.deadlines_s, self.deadlines_s[1:])):
            raise ValueError("deadlines must be strictly decreasing")


@dataclass(frozen=True)
class SweepCell:
    model: str
    seq_len: int
    deadline_s: float
    uplink_bps: float
    downlink_bps: float
    planner: str
    feasible: bool
    server_load: float | None = None
    offload_fraction: float | None = None
    latency_s: float | None = None
    improvement_pp: float | None = None
    improvement_rel: float | None = None
    error: str | None = None


def _error_text(fn) -> str | None:
    try:
        fn()
    except Exception as exc:  # mirrors the reference's flagged-cell capture
        return str(exc)
    return None


def run_sweep(grid: SweepGrid, jobs: int = 1) -> list[SweepCell]:
    """Every grid coordinate under every planner, as one batched GPU pipeline.

    `jobs` is accepted for compatibility; the result never depends on it."""
    scen = [(m, s, d, l) for m in grid.models for s in grid.seq_lens
            for d in grid.deadlines_s for l in grid.links]
    n = len(scen)
    errors: list[str | None] = [None] * n
    # model resolution (cost_model.load_model_spec); layers do not depend on seq_len
    layer_lists, model_idx, names = [], {}, {}
    req_model = np.zeros(n, dtype=np.int32)
    for k, (m, s, _d, _l) in enumerate(scen):
        try:
            spec = cost_model.load_model_spec(m, s)
        except Exception as exc:
            errors[k] = str(exc)
            continue
        if m not in model_idx:
            model_idx[m] = len(layer_lists)
            layer_lists.append(spec.layers)
            names[m] = spec
        req_model[k] = model_idx[m]
    if grid.metric not in ("flop", "memory"):
        errors = [e or f"metric must be 'flop' or 'memory', got {grid.metric!r}" for e in errors]
    unit_err = _error_text(lambda: _check_unit(grid))
    if unit_err:
        errors = [e or unit_err for e in errors]
    valid = np.array([e is None for e in errors])
    results = _sweep_valid(grid, scen, req_model, layer_lists, valid, errors) if valid.any() else {}

    cells = []
    for k, (m, s, d, l) in enumerate(scen):
        coords = dict(model=m, seq_len=s, deadline_s=d, uplink_bps=l.uplink_bps,
                      downlink_bps=l.downlink_bps)
        if errors[k] is not None:
            logger.warning("scenario %s failed: %s", coords, errors[k])
            cells += [SweepCell(planner=p, feasible=False, error=errors[k], **coords)
                      for p in grid.planners]
            continue
        cells += results[k](coords)
    cells.sort(key=lambda c: (c.model, c.seq_len, c.deadline_s, c.uplink_bps, c.downlink_bps,
                              c.planner))
    return cells


def _check_unit(grid: SweepGrid) -> None:
    if grid.unit_s <= 0:
        raise ValueError("unit_s must be positive")
    if grid.rounding not in ("paper", "conservative"):
        raise ValueError(f"unknown rounding mode {grid.rounding!r}")


def _sweep_valid(grid, scen, req_model, layer_lists, valid, errors) -> dict:
    dev = N.device()
    idx = np.flatnonzero(valid)
    n = idx.size
    models, keep = cost_model.encode_models(layer_lists, dev)
    f64 = lambda vals: N.to_dev(np.asarray(vals, dtype=np.float64), torch.float64, dev)
    flags = ((N.SP_REQ_PAPER_ROUNDING if grid.rounding == "paper" else 0)
             | (N.SP_REQ_SOURCE_CLIENT if grid.source_at_client else 0)
             | (N.SP_REQ_METRIC_MEMORY if grid.metric == "memory" else 0))
    rq = dict(model=N.to_dev(req_model[idx], torch.int32, dev),
              seq=N.to_dev(np.array([scen[k][1] for k in idx], np.int64), torch.int64, dev),
              cf=f64(np.full(n, grid.client.flops_per_s)), sf=f64(np.full(n, grid.server.flops_per_s)),
              up=f64([scen[k][3].uplink_bps for k in idx]),
              dn=f64([scen[k][3].downlink_bps for k in idx]),
              pr=f64([scen[k][3].propagation_s for k in idx]),
              dl=f64([scen[k][2] for k in idx]), un=f64(np.full(n, grid.unit_s)),
              fl=N.to_dev(np.full(n, flags, np.uint8), torch.uint8, dev))
    req = N.SpRequests(n, *[N.ptr(rq[k]).value for k in
                            ("model", "seq", "cf", "sf", "up", "dn", "pr", "dl", "un", "fl")])
    off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    N.check(N.library().sp_request_layer_offsets(models, req, N.ptr(off), N.stream_ptr()),
            "sp_request_layer_offsets")
    off_h = off.cpu().numpy()
    T = int(off_h[-1])
    ft = {k: torch.empty(T, dtype=torch.float64, device=dev)
          for k in ("r", "cs", "ss", "up_s", "dn_s")}
    it = {k: torch.empty(T, dtype=torch.int64, device=dev) for k in ("i", "s", "u", "d")}
    budget = torch.empty(n, dtype=torch.int64, device=dev)
    sac = torch.empty(n, dtype=torch.uint8, device=dev)
    status = torch.empty(n, dtype=torch.int32, device=dev)
    tab = N.SpCostTable(N.ptr(off).value, T, N.ptr(ft["r"]).value, N.ptr(ft["cs"]).value, None,
                        None, N.ptr(ft["ss"]).value, N.ptr(ft["up_s"]).value,
                        N.ptr(ft["dn_s"]).value, N.ptr(it["i"]).value, N.ptr(it["s"]).value,
                        N.ptr(it["u"]).value, N.ptr(it["d"]).value, N.ptr(budget).value,
                        N.ptr(sac).value, N.ptr(status).value)
    N.check(N.library().sp_build_cost_table(models, req, 1, tab, N.stream_ptr()),
            "sp_build_cost_table")
    st_h = status.cpu().numpy()
    ok = np.ones(n, dtype=bool)
    for q in np.flatnonzero(st_h):
        k = idx[q]
        errors[k] = _error_text(lambda: raise_cost_status(int(st_h[q]), scen[k][2]))
        ok[q] = False
    lens = np.diff(off_h)
    if "oracle" in [p.replace("-", "_") for p in grid.planners]:
        for q in np.flatnonzero(ok & (lens > 24)):
            errors[idx[q]] = f"oracle limited to 24 layers, got {int(lens[q])}"
            ok[q] = False
    for p in grid.planners:
        if p.replace("-", "_") not in ("dp", "greedy", "all_server", "all_client", "oracle"):
            for q in np.flatnonzero(ok):
                errors[idx[q]] = f"unknown planner {p!r}"
            ok[:] = False
    sel = np.flatnonzero(ok)
    if sel.size == 0:
        return {}
    # compact the valid requests into one instance batch (device gathers)
    sel_t = torch.from_numpy(sel).to(dev)
    lo = off[:-1][sel_t]
    ln = (off[1:] - off[:-1])[sel_t]
    new_off = torch.zeros(sel.size + 1, dtype=torch.int64, device=dev)
    new_off[1:] = torch.cumsum(ln, 0)
    Tn = int(new_off[-1].item())
    rep = torch.repeat_interleave(torch.arange(sel.size, device=dev), ln, output_size=Tn)
    gidx = lo[rep] + (torch.arange(Tn, device=dev) - new_off[:-1][rep])
    g = lambda t: t[gidx].contiguous()
    batch = B.InstanceBatch(new_off, g(it["i"]), g(it["s"]), g(it["u"]), g(it["d"]), g(ft["r"]),
                            budget[sel_t].contiguous(), sac[sel_t].contiguous(), None,
                            lens[sel].astype(np.int64))
    times = (g(ft["cs"]), g(ft["ss"]), g(ft["up_s"]), g(ft["dn_s"]))
    total = segment_sums(batch.r, batch.layer_off)
    from .planner import plan_batch  # late import: planner imports batch
    outs, lat = {}, {}
    for p in grid.planners:
        key = p.replace("-", "_")
        if key not in outs:
            outs[key] = plan_batch(key, batch)
            lat[key] = B.latency_eq1(batch, *times, outs[key].pi)
    # reference metrics (evaluator.py:187-207), elementwise IEEE on the device
    zero = torch.zeros_like(total)
    offload = {k: torch.where(total > 0, o.client_value / total, zero) for k, o in outs.items()}
    imp_pp = imp_rel = None
    have_greedy = "greedy" in outs
    if "dp" in outs and have_greedy:
        gl, dl = outs["greedy"].server_load, outs["dp"].server_load
        diff = (gl - dl) * 100.0
        imp_pp = diff / total
        imp_rel = torch.where(gl > 0, diff / gl, zero)
    H = {k: o.to_host() for k, o in outs.items()}
    Hoff = {k: v.cpu().numpy() for k, v in offload.items()}
    Hlat = {k: v.cpu().numpy() for k, v in lat.items()}
    tot_h = total.cpu().numpy()
    pp_h = imp_pp.cpu().numpy() if imp_pp is not None else None
    rel_h = imp_rel.cpu().numpy() if imp_rel is not None else None
    results = {}
    for q, pos in enumerate(sel):
        k = idx[pos]
        bt = [key for key in outs if H[key]["status"][q] == N.SP_ERR_BACKTRACE]
        if bt:
            errors[k] = "no predecessor reproduces the stored value"
            continue
        greedy_ok = have_greedy and bool(H["greedy"]["feasible"][q])
        if "dp" in outs and greedy_ok and not tot_h[q] > 0:
            raise ValueError("total_r must be positive")
        results[k] = _cell_builder(grid.planners, H, Hoff, Hlat, q, greedy_ok, pp_h, rel_h)
    del keep
    return results


def _cell_builder(planners, H, Hoff, Hlat, q, greedy_ok, pp_h, rel_h):
    def build(coords):
        cells = []
        for p in planners:
            key = p.replace("-", "_")
            h = H[key]
            pp = rel = None
            if p == "dp" and greedy_ok:
                pp, rel = float(pp_h[q]), float(rel_h[q])
            cells.append(SweepCell(planner=p, feasible=bool(h["feasible"][q]),
                                   server_load=float(h["server_load"][q]),
                                   offload_fraction=float(Hoff[key][q]),
                                   latency_s=float(Hlat[key][q]), improvement_pp=pp,
                                   improvement_rel=rel, **coords))
        return cells
    return build


# ---------------------------------------------------------------------------
# CSV (evaluator.py:229-288) -- host-side formatting


def _fmt(v) -> str:
    if v is None:
        return ""
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, float):
        return repr(v)
    return str(v)


def sweep_csv_text(cells: Iterable[SweepCell]) -> str:
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(SWEEP_COLUMNS)
    for c in cells:
        w.writerow([_fmt(getattr(c, col)) for col in SWEEP_COLUMNS])
    return buf.getvalue()


def write_sweep_csv(path, cells: Iterable[SweepCell]) -> None:
    Path(path).write_text(sweep_csv_text(cells))


def read_sweep_csv(path) -> list[SweepCell]:
    opt = lambda v: float(v) if v else None
    with open(path, newline="") as fh:
        return [SweepCell(model=r["model"], seq_len=int(r["seq_len"]),
                          deadline_s=float(r["deadline_s"]), uplink_bps=float(r["uplink_bps"]),
                          downlink_bps=float(r["downlink_bps"]), planner=r["planner"],
                          feasible=r["feasible"] == "true", server_load=opt(r["server_load"]),
                          offload_fraction=opt(r["offload_fraction"]),
                          latency_s=opt(r["latency_s"]), improvement_pp=opt(r["improvement_pp"]),
                          improvement_rel=opt(r["improvement_rel"]))
                for r in csv.DictReader(fh)]


def mean_over(cells: Sequence[SweepCell], axis: str, value: str, planner: str | None = None) -> dict:
    """Mean of `value` grouped by `axis` (reporting helper, evaluator.py:276-288)."""
    groups: dict = {}
    for c in cells:
        if planner is not None and c.planner != planner:
            continue
        v = getattr(c, value)
        if v is not None:
            groups.setdefault(getattr(c, axis), []).append(v)
    return {k: float(np.mean(v)) for k, v in sorted(groups.items())}
