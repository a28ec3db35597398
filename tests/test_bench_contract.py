"""The bench.py reference arm under torchrun (no GPU needed): rank 0 alone
prints exactly one JSON line with the contract's keys; the other rank exits 0
without output."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_reference_arm_under_torchrun_world2():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--requests", "8",
           "--cpu-sample", "2"]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["steps"] == 1
    for k in ("metric", "value", "unit", "higher_is_better", "cpu_baseline", "e2e", "config"):
        assert k in d
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "port"
    assert d["value"] > 0


def test_clock_sampler_samples_short_regions(monkeypatch):
    """bench.ClockSampler keeps only samples taken inside the timed region and
    always has at least the one taken as the region closes (a 20-step cfg2
    region lasts ~20 ms); throttle reasons map from NVML's bit mask."""
    import types

    nv = types.ModuleType("pynvml")
    nv.NVML_CLOCK_SM = 0
    nv.nvmlInit = lambda: None
    nv.nvmlDeviceGetHandleByIndex = lambda i: i
    nv.nvmlDeviceGetClockInfo = lambda h, c: 1965
    nv.nvmlDeviceGetMaxClockInfo = lambda h, c: 1965
    nv.nvmlDeviceGetCurrentClocksEventReasons = lambda h: 0x4
    nv.nvmlClocksEventReasonSwPowerCap = 0x4
    nv.nvmlClocksEventReasonHwSlowdown = 0x8
    monkeypatch.setitem(sys.modules, "pynvml", nv)
    sys.path.insert(0, str(ROOT))
    try:
        import bench
    finally:
        sys.path.remove(str(ROOT))
    with bench.ClockSampler(0) as clocks:
        clocks.sample_now()
    s = clocks.summary()
    assert s["samples"] >= 1 and s["sm_mhz"] == 1965.0 and s["sm_max_mhz"] == 1965.0
    assert s["reasons"] == ["sw_power_cap"]
