"""Write csrc/np_ziggurat.inc: numpy's exponential ziggurat tables.

numpy's Generator draws exponentials with the ziggurat method of its
distributions library (numpy/random/src/distributions/distributions.c,
random_standard_exponential) over three 256-entry tables (ke_double,
we_double, fe_double).  They are not part of numpy's Python API, so this
script reads them out of the installed wheel's static library
(numpy/random/lib/libnpyrandom.a: the symbol offsets in .rodata come from
`nm`, the section's file offset from `readelf`) and writes them as exact
hex-float / integer literals.  Run once per numpy version (checked in CPU
tests: tests/test_skeleton.py regenerates and compares).

    python tools/gen_np_ziggurat.py [--check]
"""

from __future__ import annotations

import os
import re
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parents[1] / "paper_2410_10759_b200" / "csrc" / "np_ziggurat.inc"


def tables() -> dict:
    lib = Path(np.random.__file__).parent / "lib" / "libnpyrandom.a"
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["ar", "x", str(lib)], cwd=d, check=True)
        obj = next(p for p in Path(d).iterdir() if "distributions_distributions" in p.name)
        syms = {}
        for line in subprocess.run(["nm", str(obj)], capture_output=True, text=True, check=True).stdout.splitlines():
            parts = line.split()
            if len(parts) == 3 and parts[2] in ("ke_double", "we_double", "fe_double"):
                syms[parts[2]] = int(parts[0], 16)
        sec = subprocess.run(["readelf", "-S", "-W", str(obj)], capture_output=True, text=True, check=True).stdout
        m = re.search(r"\]\s+\.rodata\s+PROGBITS\s+[0-9a-f]+\s+([0-9a-f]+)", sec)
        base = int(m.group(1), 16)
        m8 = re.search(r"\]\s+\.rodata\.cst8\s+PROGBITS\s+[0-9a-f]+\s+([0-9a-f]+)\s+([0-9a-f]+)", sec)
        blob = obj.read_bytes()
    get = lambda name, dt: np.frombuffer(blob[base + syms[name]: base + syms[name] + 2048], dtype=dt)
    t = {"ke": get("ke_double", "<u8"), "we": get("we_double", "<f8"), "fe": get("fe_double", "<f8")}
    assert t["fe"][0] == 1.0 and np.all(np.diff(t["fe"]) < 0), "unexpected fe_double layout"
    # ziggurat_exp_r (the tail start): the one 8-byte literal of the object in
    # (7.6, 7.8); it is also the right edge of the last strip, we[255] * 2^53
    c8 = np.frombuffer(blob[int(m8.group(1), 16): int(m8.group(1), 16) + int(m8.group(2), 16)], dtype="<f8")
    r = [float(v) for v in c8 if 7.6 < v < 7.8]
    assert len(r) == 1 and abs(r[0] - float(t["we"][255]) * 2.0 ** 53) < 1e-12, r
    t["r"] = r[0]
    return t


def render(t: dict) -> str:
    lines = ["// numpy's exponential ziggurat tables (numpy " + np.__version__ + ",",
             "// numpy/random/src/distributions/ziggurat_constants.h: ke_double, we_double,",
             "// fe_double, ziggurat_exp_r), read from the installed wheel by",
             "// tools/gen_np_ziggurat.py.  Qualifier SP_ZIG_QUAL: device global memory",
             "// (divergent indices: not __constant__), or static const in host test code.",
             "// Generated file; do not edit."]
    def arr(name, ctype, vals, fmt):
        lines.append(f"SP_ZIG_QUAL {ctype} {name}[256] = {{")
        for i in range(0, 256, 4):
            lines.append("    " + ", ".join(fmt(v) for v in vals[i:i + 4]) + ",")
        lines.append("};")
    arr("np_zig_ke", "uint64_t", t["ke"], lambda v: f"{int(v)}ull")
    arr("np_zig_we", "double", t["we"], lambda v: float(v).hex())
    arr("np_zig_fe", "double", t["fe"], lambda v: float(v).hex())
    lines.append(f"constexpr double np_zig_exp_r = {t['r'].hex()};  // ziggurat_exp_r")
    return "\n".join(lines) + "\n"


if __name__ == "__main__":
    text = render(tables())
    if "--check" in sys.argv:
        sys.exit(0 if OUT.read_text() == text else 1)
    OUT.write_text(text)
    print(f"wrote {OUT}")
