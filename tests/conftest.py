"""Shared fixtures: golden-vector loaders and the `gpu` marker.

`-m "not gpu"` runs here (no GPU): the oracle against the golden vectors, the
host logic, and the C-ABI library's exports.  `-m gpu` runs on a B200 and
checks every CUDA entry point against the golden vectors and the oracle.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(ROOT))


# the reference's own suite is staged here by tests/tools/ref_tests.sh and run
# separately (it imports `splitplan`); never collected by this suite
collect_ignore = ["golden/_ref_tests", "golden/ref_shim", "tools"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    if not has_gpu():
        pytest.fail("GPU test selected but no CUDA device is visible")
    from paper_2410_10759_b200 import _native
    _native.library()
    return True


def load_npz(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def load_json(name: str) -> dict:
    return json.loads((GOLDEN / name).read_text())


class Battery:
    """CSR instance battery from tests/golden/*.npz with reference outputs."""

    def __init__(self, name: str):
        self.name = name
        self.z = load_npz(name)
        self.off = self.z["off"]
        self.n = len(self.off) - 1

    def inst(self, k: int) -> dict:
        a, b = self.off[k], self.off[k + 1]
        z = self.z
        return dict(i=z["i"][a:b], s=z["s"][a:b], u=z["u"][a:b], d=z["d"][a:b], r=z["r"][a:b],
                    budget=int(z["budget"][k]), sac=bool(z["sac"][k]))

    def must(self, k: int):
        m = int(self.z["must"][k])
        return None if m < 0 else ("client" if m == 1 else "server")

    def has(self, planner: str) -> bool:
        return f"{planner}_pi" in self.z

    def expected(self, planner: str, k: int) -> dict | None:
        z = self.z
        if planner == "dp" and z["dp_err"][k]:
            return None
        a, b = self.off[k], self.off[k + 1]
        return dict(pi=tuple(int(v) for v in z[f"{planner}_pi"][a:b]),
                    client_value=float(z[f"{planner}_cv"][k]),
                    server_load=float(z[f"{planner}_sl"][k]),
                    integer_latency=int(z[f"{planner}_lat"][k]),
                    feasible=bool(z[f"{planner}_feas"][k]))

    def problems(self):
        from paper_2410_10759_b200.problem import PlanProblem
        return [PlanProblem.from_costs(**{"client": x["i"], "server": x["s"], "up": x["u"],
                                          "down": x["d"], "r": x["r"], "budget": x["budget"],
                                          "source_at_client": x["sac"]})
                for x in (self.inst(k) for k in range(self.n))]


def same_float(a: float, b: float) -> bool:
    """Bit-level equality that also matches NaN with NaN."""
    return (a == b and np.signbit(a) == np.signbit(b)) or (a != a and b != b)


def assert_policy(got: dict, exp: dict, ctx: str = ""):
    assert tuple(got["pi"]) == exp["pi"], f"{ctx} pi {got['pi']} != {exp['pi']}"
    assert same_float(got["client_value"], exp["client_value"]), \
        f"{ctx} client_value {got['client_value']!r} != {exp['client_value']!r}"
    assert same_float(got["server_load"], exp["server_load"]), \
        f"{ctx} server_load {got['server_load']!r} != {exp['server_load']!r}"
    assert int(got["integer_latency"]) == exp["integer_latency"], ctx
    assert bool(got["feasible"]) == exp["feasible"], ctx
