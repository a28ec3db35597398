"""Integer placement instances -- drop-in for `splitplan.problem`.

Same public names and behaviour as the reference module (problem.py); the
arithmetic runs on the GPU: `to_units` / `budget_units` / `integerize` call
the elementwise `sp_to_units` kernel and `build_problem` the K1
`sp_integerize_profiles` kernel (problem.py:58-115, 188-222).  Argument
validation stays here so exception types and messages match the reference.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path
from typing import Mapping, Sequence

import numpy as np
import torch

from . import _native as N

ROUNDING_MODES = ("paper", "conservative")

__all__ = ["LinkSpec", "PlanProblem", "ROUNDING_MODES", "transfer_times", "to_units",
           "budget_units", "integerize", "build_problem", "load_scenario"]

_COST_ERRORS = {
    1: (ValueError, "times must be >= 0"),
    2: (ValueError, "r must be >= 0"),
    3: (ValueError, "cannot convert float NaN to integer"),
    4: (OverflowError, "cannot convert float infinity to integer"),
    5: (OverflowError, "Python int too large to convert to C long"),
}


def raise_cost_status(code: int, deadline_s: float | None = None) -> None:
    """Raise what the reference raises for a K1 status word, in its order:
    time arrays (problem.py:79-92), deadline (:95-104), then r (:151-153)."""
    code = int(code)
    for part in (code & 0xFF, None, (code >> 8) & 0xFF):
        if part is None:
            if deadline_s is not None and deadline_s < 0:
                raise ValueError("deadline must be >= 0")
        elif part:
            exc, msg = _COST_ERRORS.get(part, (RuntimeError, f"cost status {part}"))
            raise exc(msg)
    if code >> 16:
        raise ValueError("r must be >= 0")


@dataclass(frozen=True)
class LinkSpec:
    """Client<->server link: rates in bit/s, one-way propagation in s (problem.py:43-55)."""

    uplink_bps: float
    downlink_bps: float
    propagation_s: float = 0.0

    def __post_init__(self):
        if not (self.uplink_bps > 0 and self.downlink_bps > 0):
            raise ValueError("link rates must be positive")
        if self.propagation_s < 0:
            raise ValueError("propagation delay must be >= 0")


def transfer_times(tau_bytes: float, link: LinkSpec) -> tuple[float, float]:
    """(upload_s, download_s) of one boundary tensor (problem.py:58-65).

    Scalar convenience: the batched form is fused into the K1 kernel."""
    bits = 8.0 * tau_bytes
    return bits / link.uplink_bps + link.propagation_s, bits / link.downlink_bps + link.propagation_s


def _check_unit_mode(unit_s: float, mode: str) -> None:
    if unit_s <= 0:
        raise ValueError("unit_s must be positive")
    if mode not in ROUNDING_MODES:
        raise ValueError(f"unknown rounding mode {mode!r}")


def _units_gpu(values: np.ndarray, unit_s: float, kernel_mode: int) -> np.ndarray:
    dev = N.device()
    t = N.to_dev(values, torch.float64, dev)
    out = torch.empty(t.numel(), dtype=torch.int64, device=dev)
    st = torch.empty(t.numel(), dtype=torch.int32, device=dev)
    N.check(N.library().sp_to_units(N.ptr(t), t.numel(), float(unit_s), kernel_mode,
                                    N.ptr(out), N.ptr(st), N.stream_ptr()), "sp_to_units")
    status = st.cpu().numpy()
    bad = np.flatnonzero(status)
    if bad.size:
        raise_cost_status(status[bad[0]])
    return out.cpu().numpy()


def to_units(seconds, unit_s: float, mode: str = "conservative") -> np.ndarray:
    """Per-layer times -> integer units: ceil (conservative) or half-up (paper)."""
    _check_unit_mode(unit_s, mode)
    arr = np.atleast_1d(np.asarray(seconds, dtype=float))
    if np.any(arr < 0):
        raise ValueError("times must be >= 0")
    if arr.size == 0:
        return np.empty(arr.shape, dtype=np.int64)
    return _units_gpu(arr.ravel(), unit_s, 1 if mode == "paper" else 0).reshape(arr.shape)


def budget_units(deadline_s: float, unit_s: float, mode: str = "conservative") -> int:
    """Deadline -> integer budget W: floor (conservative) or half-up (paper)."""
    if deadline_s < 0:
        raise ValueError("deadline must be >= 0")
    _check_unit_mode(unit_s, mode)
    return int(_units_gpu(np.array([deadline_s], dtype=float), unit_s, 1 if mode == "paper" else 2)[0])


def integerize(times: Mapping[str, Sequence[float]], deadline_s: float,
               unit_s: float, mode: str = "conservative") -> tuple[dict[str, np.ndarray], int]:
    """Integer units for a bundle of time vectors plus the budget (problem.py:107-115)."""
    units = {key: to_units(vals, unit_s, mode) for key, vals in times.items()}
    return units, budget_units(deadline_s, unit_s, mode)


@dataclass
class PlanProblem:
    """A chain of L layers with integer costs, values r and a unit budget.

    Field meaning follows problem.py:118-185: client/server compute units,
    up/down transfer units of each layer's input tensor, `budget` (W), and the
    optional real-valued times the instance was built from.
    """

    client_units: np.ndarray
    server_units: np.ndarray
    up_units: np.ndarray
    down_units: np.ndarray
    r: np.ndarray
    budget: int
    source_at_client: bool = True
    unit_s: float = 1e-3
    rounding: str = "conservative"
    client_s: np.ndarray | None = None
    server_s: np.ndarray | None = None
    up_s: np.ndarray | None = None
    down_s: np.ndarray | None = None
    deadline_s: float | None = None

    def __post_init__(self):
        for field in ("client_units", "server_units", "up_units", "down_units"):
            vec = np.asarray(getattr(self, field), dtype=np.int64)
            if np.any(vec < 0):
                raise ValueError(f"{field} must be >= 0")
            setattr(self, field, vec)
        self.r = np.asarray(self.r, dtype=float)
        if np.any(self.r < 0):
            raise ValueError("r must be >= 0")
        sizes = {v.shape[0] if v.ndim else 1 for v in (self.client_units, self.server_units,
                                                       self.up_units, self.down_units, self.r)}
        if len(sizes) != 1 or 0 in sizes:
            raise ValueError("cost vectors must share one positive length")
        if self.budget < 0:
            raise ValueError("budget must be >= 0")
        for field in ("client_s", "server_s", "up_s", "down_s"):
            if getattr(self, field) is not None:
                setattr(self, field, np.asarray(getattr(self, field), dtype=float))

    @property
    def n_layers(self) -> int:
        return len(self.client_units)

    @property
    def total_r(self) -> float:
        """np.sum(r) in numpy's pairwise order, computed on the device once per
        r content (a cached value is reused while r's bytes are unchanged)."""
        r = np.asarray(self.r, dtype=np.float64)
        key = (id(self.r), hash(r.tobytes()))
        cached = self.__dict__.get("_total_r_cache")
        if cached is None or cached[0] != key:
            from .evaluator import _total_r
            cached = (key, _total_r(self))
            self.__dict__["_total_r_cache"] = cached
        return cached[1]

    @property
    def has_real_times(self) -> bool:
        return self.client_s is not None

    @classmethod
    def from_costs(cls, client, server, up, down, r, budget, source_at_client=True,
                   **kwargs) -> "PlanProblem":
        """Instance straight from integer cost vectors (problem.py:179-185)."""
        return cls(np.asarray(client), np.asarray(server), np.asarray(up), np.asarray(down),
                   np.asarray(r, dtype=float), int(budget), source_at_client=source_at_client,
                   **kwargs)


def _request_arrays(n, link: LinkSpec, deadline_s, unit_s, flags):
    dev = N.device()
    full = lambda v: torch.full((n,), float(v), dtype=torch.float64, device=dev)
    return dict(up=full(link.uplink_bps), down=full(link.downlink_bps),
                prop=full(link.propagation_s), deadline=full(deadline_s), unit=full(unit_s),
                flags=torch.full((n,), flags, dtype=torch.uint8, device=dev))


def build_problem(layers, link: LinkSpec, deadline_s: float, unit_s: float = 1e-3,
                  source_at_client: bool = True, rounding: str = "conservative",
                  zero_server_time: bool = False) -> PlanProblem:
    """Integer instance for a profiled model and one scenario (problem.py:188-222).

    The transfer times and every integerization run in the K1 kernel."""
    layers = list(layers)
    _check_unit_mode(unit_s, rounding)
    L = len(layers)
    if L == 0:
        raise ValueError("cost vectors must share one positive length")
    dev = N.device()
    col = lambda attr: N.to_dev(np.array([getattr(p, attr) for p in layers], dtype=float),
                                torch.float64, dev)
    r, cs, ss, tau = col("r"), col("client_time_s"), col("server_time_s"), col("tau_bytes")
    flags = ((N.SP_REQ_PAPER_ROUNDING if rounding == "paper" else 0)
             | (N.SP_REQ_SOURCE_CLIENT if source_at_client else 0)
             | (N.SP_REQ_ZERO_SERVER if zero_server_time else 0))
    q = _request_arrays(1, link, deadline_s, unit_s, flags)
    off = torch.tensor([0, L], dtype=torch.int64, device=dev)
    o = {k: torch.empty(L, dtype=torch.float64, device=dev) for k in ("server_s", "up_s", "down_s")}
    u = {k: torch.empty(L, dtype=torch.int64, device=dev) for k in ("i", "s", "u", "d")}
    budget = torch.empty(1, dtype=torch.int64, device=dev)
    sac = torch.empty(1, dtype=torch.uint8, device=dev)
    status = torch.empty(1, dtype=torch.int32, device=dev)
    req = N.SpRequests(1, None, None, None, None, N.ptr(q["up"]).value, N.ptr(q["down"]).value,
                       N.ptr(q["prop"]).value, N.ptr(q["deadline"]).value, N.ptr(q["unit"]).value,
                       N.ptr(q["flags"]).value)
    prof = N.SpProfiles(N.ptr(r).value, N.ptr(cs).value, N.ptr(ss).value, N.ptr(tau).value)
    tab = N.SpCostTable(N.ptr(off).value, L, None, None, None, None, N.ptr(o["server_s"]).value,
                        N.ptr(o["up_s"]).value, N.ptr(o["down_s"]).value, N.ptr(u["i"]).value,
                        N.ptr(u["s"]).value, N.ptr(u["u"]).value, N.ptr(u["d"]).value,
                        N.ptr(budget).value, N.ptr(sac).value, N.ptr(status).value)
    N.check(N.library().sp_integerize_profiles(prof, req, tab, N.stream_ptr()),
            "sp_integerize_profiles")
    raise_cost_status(int(status.item()), deadline_s)
    host = lambda t: t.cpu().numpy()
    return PlanProblem(client_units=host(u["i"]), server_units=host(u["s"]), up_units=host(u["u"]),
                       down_units=host(u["d"]), r=host(r), budget=int(budget.item()),
                       source_at_client=source_at_client, unit_s=unit_s, rounding=rounding,
                       client_s=host(cs), server_s=host(o["server_s"]), up_s=host(o["up_s"]),
                       down_s=host(o["down_s"]), deadline_s=deadline_s)


def load_scenario(path) -> dict:
    """Scenario JSON: link rates, deadline, unit and flags (problem.py:225-240)."""
    doc = json.loads(Path(path).read_text())
    return {
        "link": LinkSpec(float(doc["uplink_bps"]), float(doc["downlink_bps"]),
                         float(doc.get("propagation_s", 0.0))),
        "deadline_s": float(doc["deadline_s"]),
        "unit_s": float(doc.get("unit_s", 1e-3)),
        "source_at_client": bool(doc.get("source_at_client", True)),
        "rounding": str(doc.get("rounding", "conservative")),
        "zero_server_time": bool(doc.get("zero_server_time", False)),
    }
