"""FIFO capacity-queue simulator -- drop-in for `splitplan.throughput_sim`.

The admission loop (throughput_sim.py:207-256) runs in the K4 replay kernel,
one thread per run: `compare_variants` replays its three demand variants in
one launch, and `replay_many` takes any number of independent runs (the
Monte-Carlo sweeps of SURVEY.md cfg4).  Seeded arrival skeletons are drawn
with numpy's PCG64 `Generator` exactly as the reference does, so paired runs
see bit-identical streams.
"""

from __future__ import annotations

import csv
import io
import json
from dataclasses import dataclass
from pathlib import Path
from typing import Sequence

import numpy as np
import torch

from . import _native as N
from .evaluator import SweepCell, segment_sums

VARIANTS = ("dp", "greedy", "nosplit")
REQUEST_COLUMNS = ("request_id", "arrival_ms", "admit_ms", "wait_ms", "demand", "duration_ms")

__all__ = ["VARIANTS", "Scenario", "SimConfig", "Stream", "SimResult", "CapacityDeadlockError",
           "scenarios_from_cells", "scenarios_from_csv", "capacity_for_requests",
           "generate_stream", "simulate_stream", "simulate", "compare_variants", "replay_many",
           "requests_csv_text", "cumulative_csv_text", "summary_dict", "write_outputs"]


class CapacityDeadlockError(RuntimeError):
    """The FIFO head demands more than the whole capacity."""


@dataclass(frozen=True)
class Scenario:
    key: str
    deadline_s: float
    demand_dp: float
    demand_greedy: float
    demand_nosplit: float

    def demand(self, variant: str) -> float:
        if variant not in VARIANTS:
            raise ValueError(f"unknown variant {variant!r}")
        return getattr(self, f"demand_{variant}")


@dataclass(frozen=True)
class SimConfig:
    beta_per_ms: float
    capacity: float
    seed: int
    policy_variant: str
    horizon: int
    scenarios: tuple[Scenario, ...]
    exec_count_max: int = 10

    def __post_init__(self):
        checks = ((self.beta_per_ms <= 0, "beta_per_ms must be positive"),
                  (self.capacity <= 0, "capacity must be positive"),
                  (self.horizon < 0, "horizon must be >= 0"),
                  (not self.scenarios, "scenario table must be non-empty"),
                  (self.policy_variant not in VARIANTS,
                   f"unknown variant {self.policy_variant!r}"))
        for bad, msg in checks:
            if bad:
                raise ValueError(msg)
        object.__setattr__(self, "scenarios", tuple(self.scenarios))


@dataclass(frozen=True)
class Stream:
    arrival_ms: np.ndarray
    scenario_idx: np.ndarray
    exec_count: np.ndarray
    demand: np.ndarray
    duration_ms: np.ndarray


@dataclass(frozen=True)
class SimResult:
    """Per-request records plus queueing aggregates (throughput_sim.py:109-130).

    Replays (`replay_many`) attach the kernel-computed aggregates for the
    exact arrays they returned; a result built any other way (or copied with
    `dataclasses.replace`) computes them from `wait_ms` like the reference."""

    arrival_ms: np.ndarray
    admit_ms: np.ndarray
    wait_ms: np.ndarray
    demand: np.ndarray
    duration_ms: np.ndarray
    served_count: int

    def _cached(self):
        c = self.__dict__.get("_agg")
        return c[1] if c is not None and c[0] is self.wait_ms else None

    @property
    def max_wait_ms(self) -> float:
        if not len(self.wait_ms):
            return 0.0
        c = self._cached()
        return float(c[0]) if c is not None else float(np.max(self.wait_ms))

    @property
    def mean_wait_ms(self) -> float:
        if not len(self.wait_ms):
            return 0.0
        c = self._cached()
        return float(c[1]) if c is not None else float(np.mean(self.wait_ms))

    @property
    def cumulative_wait_ms(self) -> np.ndarray:
        c = self._cached()
        return c[2] if c is not None else np.cumsum(self.wait_ms)


def _attach(res: SimResult, max_w: float, mean_w: float, cum: np.ndarray) -> SimResult:
    """Attach the kernel's aggregates (not a dataclass field: copies recompute
    them), tied to the wait array they describe."""
    object.__setattr__(res, "_agg", (res.wait_ms, (max_w, mean_w, cum)))
    return res


# ---------------------------------------------------------------------------
# scenario table (throughput_sim.py:133-176)


def _device_mean(values: Sequence[float]) -> float:
    """np.mean on the device: numpy-order sum (sp_segment_sum) / n."""
    dev = N.device()
    x = N.to_dev(np.asarray(values, dtype=np.float64), torch.float64, dev)
    off = torch.tensor([0, x.numel()], dtype=torch.int64, device=dev)
    return float(segment_sums(x, off)[0].item()) / float(x.numel())


def scenarios_from_cells(cells: Sequence[SweepCell]) -> list[Scenario]:
    """Coordinates whose dp, greedy and all_server rows are all feasible,
    demands normalised by the mean nosplit (all_server) load."""
    by_coord: dict[tuple, dict[str, SweepCell]] = {}
    for c in cells:
        by_coord.setdefault((c.model, c.seq_len, c.deadline_s, c.uplink_bps, c.downlink_bps),
                            {})[c.planner] = c
    rows = []
    for coord in sorted(by_coord):
        g = by_coord[coord]
        trio = [g.get("dp"), g.get("greedy"), g.get("all_server")]
        if any(c is None or not c.feasible or c.server_load is None for c in trio):
            continue
        rows.append(("{}/s{}/d{:g}/u{:g}".format(*coord[:4]), coord[2],
                     trio[0].server_load, trio[1].server_load, trio[2].server_load))
    if not rows:
        return []
    norm = _device_mean([r[4] for r in rows])
    if norm <= 0:
        raise ValueError("nosplit demands are all zero; nothing to simulate")
    return [Scenario(key=k, deadline_s=dl, demand_dp=a / norm, demand_greedy=b / norm,
                     demand_nosplit=c / norm) for k, dl, a, b, c in rows]


def scenarios_from_csv(path) -> list[Scenario]:
    from .evaluator import read_sweep_csv
    return scenarios_from_cells(read_sweep_csv(path))


def capacity_for_requests(scenarios: Sequence[Scenario], n_requests: float) -> float:
    if not scenarios:
        raise ValueError("scenario table is empty")
    return float(n_requests) * _device_mean([s.demand_nosplit for s in scenarios])


# ---------------------------------------------------------------------------
# streams


def _skeleton(config: SimConfig):
    """Seeded arrivals / scenario picks / execution counts (throughput_sim.py:179-186)."""
    g = np.random.default_rng(config.seed)
    n = config.horizon
    arrivals = np.cumsum(g.exponential(scale=1.0 / config.beta_per_ms, size=n))
    idx = g.integers(0, len(config.scenarios), size=n)
    execs = g.integers(1, config.exec_count_max + 1, size=n)
    return arrivals, idx, execs


def skeletons_device(seeds, choice_lo, choice_hi, horizon: int, beta_per_ms: float,
                     exec_count_max: int = 10) -> tuple:
    """`_skeleton` of many seeded runs at once on the GPU (sp_sim_skeletons:
    numpy's default_rng(seed) stream bit for bit, one thread per run).  Run r
    picks table rows in [choice_lo[r], choice_hi[r]).  Returns device tensors
    [n, horizon]: arrivals (float64), rows (int32), execution counts (int32)."""
    dev = N.device()
    seeds_d = N.to_dev(np.asarray(seeds, dtype=np.int64), torch.int64, dev)
    lo_d = N.to_dev(np.asarray(choice_lo, dtype=np.int64), torch.int64, dev)
    hi_d = N.to_dev(np.asarray(choice_hi, dtype=np.int64), torch.int64, dev)
    n = seeds_d.numel()
    if bool(((hi_d - lo_d) < 1).any()) or bool((seeds_d < 0).any()):
        raise ValueError("skeletons need non-negative seeds and non-empty scenario ranges")
    arr = torch.empty((n, horizon), dtype=torch.float64, device=dev)
    rows = torch.empty((n, horizon), dtype=torch.int32, device=dev)
    execs = torch.empty((n, horizon), dtype=torch.int32, device=dev)
    N.check(N.library().sp_sim_skeletons(N.ptr(seeds_d), N.ptr(lo_d), N.ptr(hi_d), n, int(horizon),
                                         1.0 / beta_per_ms, int(exec_count_max), N.ptr(arr), N.ptr(rows),
                                         N.ptr(execs), None, N.stream_ptr()), "sp_sim_skeletons")
    return arr, rows, execs


def _project(config: SimConfig, arrivals, idx, execs, variant: str) -> Stream:
    dem = np.array([s.demand(variant) for s in config.scenarios])
    dl = np.array([s.deadline_s * 1000.0 for s in config.scenarios])
    return Stream(arrival_ms=arrivals, scenario_idx=idx, exec_count=execs, demand=dem[idx],
                  duration_ms=dl[idx] * execs)


def generate_stream(config: SimConfig) -> Stream:
    arrivals, idx, execs = _skeleton(config)
    return _project(config, arrivals, idx, execs, config.policy_variant)


# ---------------------------------------------------------------------------
# replay on the GPU


def replay_arrays(run_off, arrival_ms, demand, duration_ms, capacity, per_request: bool = True) -> dict:
    """K4 over independent runs given as CSR arrays (host numpy or device
    tensors): run k replays requests [run_off[k], run_off[k+1]) against
    capacity[k].  Returns the device outputs: admit / wait / cumulative wait
    per request (wait / cumulative only with `per_request`), max / mean wait,
    status and the deadlocked request per run."""
    dev = N.device()
    t = dict(off=N.to_dev(run_off, torch.int64, dev), arr=N.to_dev(arrival_ms, torch.float64, dev),
             dem=N.to_dev(demand, torch.float64, dev), dur=N.to_dev(duration_ms, torch.float64, dev),
             cap=N.to_dev(capacity, torch.float64, dev))
    nr = t["off"].numel() - 1
    total = t["arr"].numel()
    o = dict(admit=torch.empty(max(total, 1), dtype=torch.float64, device=dev),
             mx=torch.empty(max(nr, 1), dtype=torch.float64, device=dev),
             mean=torch.empty(max(nr, 1), dtype=torch.float64, device=dev),
             st=torch.zeros(max(nr, 1), dtype=torch.int32, device=dev),
             dead=torch.empty(max(nr, 1), dtype=torch.int64, device=dev))
    if per_request:
        o["wait"] = torch.empty(max(total, 1), dtype=torch.float64, device=dev)
        o["cum"] = torch.empty(max(total, 1), dtype=torch.float64, device=dev)
    b = N.SpSimBatch(nr, total, *[N.ptr(t[k]).value for k in ("off", "arr", "dem", "dur", "cap")])
    so = N.SpSimOut(*[N.ptr(o[k]).value if k in o else None for k in ("admit", "wait", "cum", "mx", "mean",
                                                                       "st", "dead")])
    lib = N.library()
    need = int(lib.sp_sim_workspace_bytes(b))
    ws = N.workspace(need)
    N.check(lib.sp_sim_replay(b, so, N.ptr(ws), ws.numel(), N.stream_ptr()), "sp_sim_replay")
    return o


def replay_many(streams: Sequence[Stream], capacities: Sequence[float],
                raise_on_deadlock: bool = True) -> list[SimResult | CapacityDeadlockError]:
    """Replay independent (stream, capacity) runs in one K4 launch."""
    lens = np.array([len(s.arrival_ms) for s in streams], dtype=np.int64)
    off = np.zeros(len(streams) + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    total = int(off[-1])
    cat = lambda f: (np.concatenate([np.asarray(f(s), dtype=np.float64) for s in streams])
                     if total else np.zeros(0))
    o = replay_arrays(off, cat(lambda s: s.arrival_ms), cat(lambda s: s.demand),
                      cat(lambda s: s.duration_ms), np.asarray(capacities, dtype=np.float64))
    h = {k: v.cpu().numpy() for k, v in o.items()}
    out = []
    for r, s in enumerate(streams):
        a, z = off[r], off[r + 1]
        if h["st"][r] == N.SP_ERR_DEADLOCK:
            q = int(h["dead"][r])
            err = CapacityDeadlockError(
                f"request {q} demands {s.demand[q]:.6g} > capacity {capacities[r]:.6g}; "
                f"the FIFO head can never be admitted")
            if raise_on_deadlock:
                raise err
            out.append(err)
            continue
        res = SimResult(arrival_ms=s.arrival_ms, admit_ms=h["admit"][a:z].copy(),
                        wait_ms=h["wait"][a:z].copy(), demand=s.demand,
                        duration_ms=s.duration_ms, served_count=int(z - a))
        out.append(_attach(res, float(h["mx"][r]), float(h["mean"][r]), h["cum"][a:z].copy()))
    return out


def simulate_stream(stream: Stream, capacity: float) -> SimResult:
    """FIFO admission over one prepared stream (throughput_sim.py:207-256)."""
    return replay_many([stream], [capacity])[0]


def simulate(config: SimConfig) -> SimResult:
    return simulate_stream(generate_stream(config), config.capacity)


def compare_variants(config: SimConfig) -> dict[str, SimResult]:
    """dp, greedy and nosplit over one shared skeleton, replayed in one launch."""
    arrivals, idx, execs = _skeleton(config)
    streams = [_project(config, arrivals, idx, execs, v) for v in VARIANTS]
    res = replay_many(streams, [config.capacity] * len(VARIANTS))
    return dict(zip(VARIANTS, res))


# ---------------------------------------------------------------------------
# outputs (throughput_sim.py:275-322) -- host-side formatting


def requests_csv_text(result: SimResult) -> str:
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(REQUEST_COLUMNS)
    cols = (result.arrival_ms, result.admit_ms, result.wait_ms, result.demand, result.duration_ms)
    for k in range(len(result.arrival_ms)):
        w.writerow([k, *(repr(float(c[k])) for c in cols)])
    return buf.getvalue()


def cumulative_csv_text(result: SimResult) -> str:
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(("request_id", "cumulative_wait_ms"))
    for k, v in enumerate(result.cumulative_wait_ms):
        w.writerow([k, repr(float(v))])
    return buf.getvalue()


def summary_dict(result: SimResult) -> dict:
    return {"max_wait_ms": result.max_wait_ms, "mean_wait_ms": result.mean_wait_ms,
            "served": result.served_count}


def write_outputs(out_dir, variant: str, result: SimResult) -> list[Path]:
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    files = ((f"requests_{variant}.csv", requests_csv_text(result)),
             (f"cumulative_{variant}.csv", cumulative_csv_text(result)),
             (f"summary_{variant}.json",
              json.dumps(summary_dict(result), indent=2, sort_keys=True) + "\n"))
    paths = []
    for name, text in files:
        p = out_dir / name
        p.write_text(text)
        paths.append(p)
    return paths
