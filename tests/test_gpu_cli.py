"""The CLI drop-in (`paper_2410_10759_b200.cli`) against the reference CLI's own
outputs (tests/golden/cli, produced by tests/golden/gen_cli.py running
`splitplan.cli.main`): same exit codes, byte-identical profile / policy JSON,
sweep CSV and simulation files, manifests with the same shape."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

sys.path.insert(0, str(GOLDEN))
CLI = GOLDEN / "cli"




@pytest.fixture(scope="module")
def gen(gpu):
    # the generator module imports splitplan at import time; load just its tables
    src = (GOLDEN / "gen_cli.py").read_text()
    start, end = src.index("TOY_PROFILE = "), src.index("\n\ndef run(")
    ns: dict = {}
    exec(src[start:end], ns)  # plain data: dicts and argv lists
    return ns


def _compare_tree(got: Path, exp: Path):
    for f in exp.rglob("*"):
        if f.is_dir():
            continue
        g = got / f.relative_to(exp)
        assert g.exists(), f"missing output {g.name}"
        if f.name.endswith("manifest.json"):
            a, b = json.loads(g.read_text()), json.loads(f.read_text())
            assert set(a) == set(b) | {"duration_s"} and a["command"] == b["command"], f.name
            assert a["seed"] == b["seed"] and set(a["inputs"]) == set(b["inputs"]), f.name
            assert [Path(p).name for p in a["outputs"]] == [Path(p).name for p in b["outputs"]]
        else:
            assert g.read_bytes() == f.read_bytes(), f"{f.relative_to(CLI)} differs"


def test_cli_matches_reference(gen, tmp_path):
    from paper_2410_10759_b200.cli import main
    codes = json.loads((CLI / "exit_codes.json").read_text())
    inp = CLI / "inputs"
    for case, argv in gen["CASES"].items():
        o = tmp_path / case
        o.mkdir()
        code = main([a.format(i=inp, o=o, s="") for a in argv])
        assert code == codes[case], case
        _compare_tree(o, CLI / case)
    o = tmp_path / "simulate"
    o.mkdir()
    sim = [a.format(i=inp, o=o, s=str(CLI / "sweep" / "sweep.csv")) for a in gen["SIM"]]
    assert main(sim) == codes["simulate"]
    _compare_tree(o, CLI / "simulate")
