"""Test-only alias: the reference's import name `splitplan` mapped onto the
drop-in package, so the reference's own test suite (pkg/tests, copied at run
time by tests/tools/ref_tests.sh into a git-ignored directory) runs against
the B200 engine unchanged.  Only the conformance run puts this on sys.path."""

import importlib
import sys

import paper_2410_10759_b200 as _pkg
from paper_2410_10759_b200 import *  # noqa: F401,F403

for _name in ("cost_model", "problem", "planner", "evaluator", "throughput_sim", "cli"):
    _mod = importlib.import_module(f"paper_2410_10759_b200.{_name}")
    sys.modules[f"splitplan.{_name}"] = _mod
    globals()[_name] = _mod

__version__ = getattr(_pkg, "__version__", "b200")
