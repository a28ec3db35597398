"""Benchmark: DP cells/s and solved requests/s of the SplitLLM placement engine.

Workload (BASELINE.json configs[1]): gpt2-24 (L = 98
splittable entries), 10,000 requests per GPU, seq_len ~ U{128..2048}, symmetric
links log-uniform in [3e7, 1e9] bit/s with 10 ms propagation, deadline = f x
all-client time with f ~ U(0.05, 1), unit_s = deadline / 1e5 so every request
has W = W_eff = 100,000 budget columns.  Devices calibrated as the reference
acceptance suite (bert-12 @ 4096 tokens: 7.727 s client, 0.0979 s server).

One step = the hot path over the whole batch through the public engine
(`requests.Engine.solve`): K1 cost table -> prep -> K2 DP -> K3 backtrack, every
request gets its optimal placement.  A "DP cell" is one cell of the
reference's (L+1) x (W_eff+1) tables (planner.py:128-143): L x (W_eff+1) per
request, 9.8e10 per step.  The engine solves the wide cfg2 rows as breakpoint
lists (csrc/dp_steps.cuh: every row is a step function with <= ~130
breakpoints, the same table bit for bit); `dense_kernel` reports the same
batch forced onto the dense L2-streaming kernel for comparison.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun each rank solves its own 10k requests (weak scaling); the step
time is the max over ranks.  `--impl reference` times the CPU oracle port of
the reference path (profile -> build_problem -> plan_dp) on the host cores.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import platform
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "DP cells/sec and solved scenarios/sec at 1/2/4/8 B200; % HBM roofline"
L2_BYTES = 126 * 2 ** 20


# ---------------------------------------------------------------------------
# workload


def cfg2_requests(n: int, seed: int) -> dict:
    """Seeded cfg2 request parameters (host numpy arrays), workloads.cfg2."""
    from paper_2410_10759_b200 import workloads as W
    return W.cfg2(n, seed)[0]


def value_domains(r: np.ndarray, layer_off: np.ndarray) -> dict:
    """Instances per DP value domain, by the prep kernel's rule (dp_core.cuh):
    int32 when every r is integral, sum(r) < 2^53 and sum(r)/gcd <= 2^31 - 1;
    fp64 otherwise; fp64+NaN when some r is not finite."""
    out = {"int32": 0, "f64": 0, "f64_nan": 0}
    for k in range(len(layer_off) - 1):
        x = r[layer_off[k]:layer_off[k + 1]]
        if not np.all(np.isfinite(x)):
            out["f64_nan"] += 1
        elif np.all(x == np.floor(x)) and x.sum() < 2.0 ** 53:
            xi = x.astype(np.int64)
            g = max(int(np.gcd.reduce(xi)) if xi.size else 1, 1)
            out["int32" if int(xi.sum()) // g <= 2 ** 31 - 1 else "f64"] += 1
        else:
            out["f64"] += 1
    return out


def dtype_label(domains: dict) -> str:
    ran = [k for k in ("int32", "f64", "f64_nan") if domains.get(k)]
    return "+".join(ran) if ran else "int32"


# ---------------------------------------------------------------------------
# CPU side: the oracle port of the reference path, timed on host cores


def _cpu_one(args):
    from oracle import splitplan_oracle as O
    layers, s, cf, sf, bw, prop, dl, unit = args
    r, cs, ss, tau = O.profile_arrays(layers, int(s), cf, sf)
    inst = O.instance_from_profile(r, cs, ss, tau, bw, bw, prop, dl, unit)
    p = O.plan_dp(inst)
    return len(r) * (O.effective_budget(inst) + 1), p["integer_latency"]


def _cpu_jobs(req: dict, idx):
    from oracle import splitplan_oracle as O
    layers = O.preset_layers("gpt2-24")
    return [(layers, req["seq_len"][k], req["client_fps"][k], req["server_fps"][k],
             req["uplink_bps"][k], req["propagation_s"][k], req["deadline_s"][k],
             req["unit_s"][k]) for k in idx]


class CpuPool:
    """A process pool created once, outside every timed region."""

    def __init__(self, procs: int):
        from multiprocessing import get_context
        # one thread per worker process (no BLAS / OpenMP oversubscription of
        # the host cores the pool already covers)
        for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
            os.environ.setdefault(k, "1")
        self.procs = procs
        self.pool = get_context("fork").Pool(procs) if procs > 1 else None

    def run(self, jobs):
        """(DP cells, seconds) of the jobs on the pool's processes."""
        t0 = time.perf_counter()
        out = self.pool.map(_cpu_one, jobs, chunksize=1) if self.pool else [_cpu_one(j) for j in jobs]
        return sum(c for c, _ in out), time.perf_counter() - t0

    def close(self):
        if self.pool:
            self.pool.close()
            self.pool.join()


def cpu_info() -> dict:
    model = platform.processor() or ""
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "numpy": np.__version__,
            "python": platform.python_version()}


def cpu_baseline(req_np: dict, seconds: float = 12.0) -> dict:
    """The oracle port on every host core (fork pool, harness-level
    parallelism as SURVEY 8(d) prescribes) and on one core, on bounded samples
    of the same requests (about `seconds` of wall time each)."""
    procs = max(1, min(os.cpu_count() or 1, 128))
    pool = CpuPool(procs)
    try:
        _cells, per_req_s = pool.run(_cpu_jobs(req_np, range(procs)))  # one request per process, untimed
        n_all = int(max(procs, min(len(req_np["seq_len"]), procs * max(1.0, seconds / max(per_req_s, 1e-3)))))
        cells, dt = pool.run(_cpu_jobs(req_np, range(n_all)))
    finally:
        pool.close()
    one = CpuPool(1)
    n_one = int(max(2, min(64, (seconds / 2) / max(per_req_s, 1e-3))))
    c1, t1 = one.run(_cpu_jobs(req_np, range(n_one)))
    return {"value": cells / dt, "unit": "DP cells/s", "cores": procs, "kind": "port",
            "sample": f"{n_all} cfg2 requests (profile -> build_problem -> plan_dp, oracle numpy port of the "
                      f"reference, full fp64 tables) on {procs} processes, {dt:.1f} s wall",
            "scenarios_per_s": n_all / dt,
            "one_core": {"value": c1 / t1, "unit": "DP cells/s", "sample": f"{n_one} requests, {t1:.1f} s",
                         "scenarios_per_s": n_one / t1},
            **cpu_info()}


# ---------------------------------------------------------------------------
# clocks


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING a timed region: NVML
    polled every ~2 ms on a thread plus one sample taken as the region closes
    (a cfg2 step takes about a millisecond, too short for nvidia-smi's loop),
    nvidia-smi -lms 100 if NVML is unavailable."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, index: int):
        self.index = index
        self.sm: list[float] = []
        self.mx: list[float] = []
        self.max_mhz = None
        self.reasons: set[str] = set()
        self.stop = threading.Event()
        self.source = "none"
        self._nv = None

    def _nvml_sample(self) -> bool:
        nv, h = self._nv
        try:
            self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.reasons.update(name for name, b in self._bits if b and r & b)
        except Exception:
            return False
        return True

    def _nvml_loop(self):
        while not self.stop.is_set() and self._nvml_sample():
            time.sleep(0.002)

    def sample_now(self):
        """One synchronous sample, taken while the last timed launches still run
        (a short timed region can end between two polls of the thread)."""
        if self._nv is not None:
            self._nvml_sample()

    def _smi_loop(self):
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                  "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                  "clocks_event_reasons.sw_power_cap")
        try:
            p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={fields}",
                                  "--format=csv,noheader,nounits", "-lms", "100"],
                                 stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            return
        names = [n for n, _ in self.REASONS]
        for line in p.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                try:
                    self.sm.append(float(parts[0]))
                    self.mx.append(float(parts[1]))
                except ValueError:
                    pass
                self.reasons.update(n for n, v in zip(names, parts[2:]) if v.lower() == "active")
            if self.stop.is_set():
                break
        p.terminate()

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self._nv = (nv, h)
            self._bits = [(name, getattr(nv, attr, 0)) for name, attr in self.REASONS]
            self.source = "nvml, 2 ms + one sample at the end of the region"
            self.thread = threading.Thread(target=self._nvml_loop, daemon=True)
        except Exception:
            self.source = "nvidia-smi, 100 ms"
            self.thread = threading.Thread(target=self._smi_loop, daemon=True)
        self.thread.start()
        # the sampler is live before the timed region opens; only samples
        # taken inside the region are kept
        t0 = time.perf_counter()
        while not self.sm and time.perf_counter() - t0 < 2.0:
            time.sleep(0.002)
        self.sm.clear()
        self.mx.clear()
        self.reasons.clear()
        return self

    def __exit__(self, *exc):
        self.stop.set()
        self.thread.join(timeout=5)

    def summary(self) -> dict:
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None,
                "sm_max_mhz": max(self.mx) if self.mx else self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": self.source}


# ---------------------------------------------------------------------------
# roofline


def measured_peak_hbm():
    try:
        doc = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(doc["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


VARIANTS = {0: "dp_stage_kernel<smem rows>", 2: "dp_stage_kernel<global rows>",
            4: "dp_stream_kernel<L2 rows, bulk-copy staged windows>",
            5: "dp_grid_kernel<one instance over the GPU>",
            7: "dp_steps_kernel<rows as breakpoint lists>"}
NCU_SUMMARY = {0: "dp_smem_ncu_summary.json", 4: "dp_stream_ncu_summary.json", 7: "dp_steps_ncu_summary.json"}


def latest_summary(name: str):
    for d in sorted((ROOT / "profiles").glob("r*"), reverse=True):
        f = d / name
        if f.exists():
            return json.loads(f.read_text()), str(f.relative_to(ROOT))
    return None, None


class Profile:
    """sp_profile_* around a region: DP-stage kernel time, launches, cells,
    algorithmic bytes, all library launches and the dominant variant."""

    def __init__(self, lib):
        self.lib = lib

    def __enter__(self):
        self.lib.sp_profile_enable(1)
        self.lib.sp_profile_collect(None, None, None, None, None, None)
        return self

    def __exit__(self, *exc):
        ms, n, cells, byts, al, var = (C.c_double(), C.c_int64(), C.c_double(), C.c_double(), C.c_int64(),
                                       C.c_int32())
        self.lib.sp_profile_collect(C.byref(ms), C.byref(n), C.byref(cells), C.byref(byts), C.byref(al),
                                    C.byref(var))
        self.lib.sp_profile_enable(0)
        self.ms, self.n, self.cells, self.bytes = ms.value, n.value, cells.value, byts.value
        self.launches, self.variant = al.value, var.value


def _l2_ceiling():
    """Measured mixed-mode L2 throughput (GB/s) of the newest profiles/rNN/l2_ceiling run."""
    for d in sorted((ROOT / "profiles").glob("r*"), reverse=True):
        f = d / "l2_ceiling" / "l2_bandwidth.jsonl"
        if f.exists():
            vals = [json.loads(l)["total_GBps"] for l in f.read_text().splitlines()
                    if l.strip() and json.loads(l).get("mode") == "mixed"]
            if vals:
                return max(vals), str(f.relative_to(ROOT))
    return None, None


_CLOCK_HINT = [None]


def clock_mhz_hint():
    """The median SM clock the timed region ran at (set once it is sampled)."""
    return _CLOCK_HINT[0]


def roofline(prof: Profile, step_ms_total: float) -> dict:
    peak, peak_kind = measured_peak_hbm()
    n = max(prof.n, 1)
    avg_ms = prof.ms / n
    bytes_per_launch = prof.bytes / n
    cells_per_launch = prof.cells / n
    achieved = bytes_per_launch / (avg_ms / 1e3) / 1e9 if avg_ms > 0 else None
    doc, src = latest_summary(NCU_SUMMARY.get(prof.variant, ""))
    rate = prof.cells / (prof.ms / 1e3) if prof.ms else None
    out = {
        "kernel": VARIANTS.get(prof.variant, str(prof.variant)),
        "bound": "hbm",
        "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
        "frac": (achieved / peak) if achieved else None,
        "traffic": doc["dram_bytes_per_cell"] * cells_per_launch if doc else None,
        "traffic_source": src,
        "algorithmic_bytes_per_launch": bytes_per_launch,
        "cells_per_launch": cells_per_launch,
        "launches": prof.n, "avg_launch_ms": avg_ms,
        "share_of_step": prof.ms / step_ms_total if step_ms_total else None,
        "cells_per_s_in_kernel": rate,
    }
    if doc:
        out["ncu"] = {k: doc.get(k) for k in ("issue_active_pct", "warps_active_pct", "sm_throughput_pct",
                                              "lts_throughput_pct", "dram_bytes_per_cell", "warp_inst_per_cell")}
    if prof.variant == 7:
        out["note"] = ("breakpoint lists: the algorithmic bytes are the stage records read (24 B/stage) and the "
                       "breakpoints stored for the backtrack (8 B each + 8 B per row pair); the kernel is bound by "
                       "instruction issue of its merges, not by HBM (DESIGN.md 4)")
        if doc and doc.get("warp_inst_per_cell") and avg_ms > 0:
            # the binding resource: warp-instruction issue, 4 schedulers x 148
            # SMs x one instruction per clock (the SM clock sampled in the run)
            inst = doc["warp_inst_per_cell"] * cells_per_launch
            clk = (clock_mhz_hint() or 1965.0) * 1e6
            peak_issue = 148 * 4 * clk
            out["issue"] = {"bound": "warp-instruction issue", "achieved": inst / (avg_ms / 1e3),
                            "peak": peak_issue, "unit": "warp-inst/s",
                            "frac": inst / (avg_ms / 1e3) / peak_issue,
                            "warp_inst_per_launch": inst, "source": src}
    if prof.variant == 4 and doc and rate:
        # the rows live in L2: the L2 bytes per cell (ncu) against the L2
        # ceiling measured with the kernel's own data path (tools/l2_bandwidth.cu)
        l2doc, l2src = _l2_ceiling()
        per_cell = doc["l2_read_bytes_per_cell"] + 8.0 + 0.25
        if l2doc:
            out["l2"] = {"bytes_per_cell": per_cell, "achieved_GBps": rate * per_cell / 1e9,
                         "ceiling_GBps": l2doc, "ceiling_source": l2src,
                         "frac": rate * per_cell / 1e9 / l2doc}
    if prof.variant in (4, 5):
        out["note"] = ("dense L2-row kernel: algorithmic HBM bytes = the 2-bit packed back-pointers (0.25 B/cell); "
                       "the rows stay in L2; the survey's 33 B/cell row-streaming design would need "
                       f"{(rate or 0) * 33 / 1e9:.0f} GB/s for this rate")
    return out


# ---------------------------------------------------------------------------
# the other BASELINE configs (single GPU, rank 0 at N = 1)


def _events():
    import torch
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def bench_cfg3(n: int = 1_000_000) -> dict:
    """configs[2]: Llama-2-7B-like, 1M long-sequence requests, W = 1e4: one
    Engine.solve of all of them (CUDA events; a warm-up solve first)."""
    import torch
    from paper_2410_10759_b200 import _native as N
    from paper_2410_10759_b200 import batch as B
    from paper_2410_10759_b200 import workloads as W
    from paper_2410_10759_b200.requests import Engine, RequestBatch
    req, layers = W.cfg3(n)
    eng = Engine(layers)
    dev = RequestBatch.from_numpy(**req).to(N.device())
    total = int(eng.n_layers[req["model"]].sum())
    off = eng.layer_offsets(dev)
    s = eng.solve(dev, total, off)
    w = B.effective_budget(s.instances).cpu().numpy()
    cells = float((np.diff(s.layer_off.cpu().numpy()) * (w + 1)).sum())
    feasible = int(s.policies.feasible.sum().item())
    del s
    torch.cuda.synchronize()
    e0, e1 = _events()
    e0.record()
    eng.solve(dev, total, off)
    e1.record()
    torch.cuda.synchronize()
    sec = e0.elapsed_time(e1) / 1e3
    fb = int(N.library().sp_last_dense_fallbacks())
    return {"requests": n, "dp_cells": cells, "solve_s": sec, "requests_per_s": n / sec,
            "dp_cells_per_s": cells / sec, "feasible": feasible, "dense_fallbacks": fb,
            "timing": "CUDA events around one Engine.solve (K1 + prep + K2 + K3), device-resident"}


def bench_cfg4() -> dict:
    """configs[3]: the 65,536-scenario Monte-Carlo grid end to end
    (montecarlo.run: plan every request, scenario tables, skeletons, replay)."""
    import torch
    from paper_2410_10759_b200 import montecarlo as MC
    MC.run(np.arange(65536))  # warm-up at full size (workspace, allocator, pools)
    torch.cuda.synchronize()
    secs = []
    for _ in range(2):
        t0 = time.perf_counter()
        res = MC.run(np.arange(65536))
        torch.cuda.synchronize()
        secs.append(time.perf_counter() - t0)
    sec = min(secs)
    return {"scenarios": 65536, "requests": res.requests, "dp_cells": res.dp_cells, "wall_s": sec,
            "scenarios_per_s": 65536 / sec, "simulated": int((res.table_size > 0).sum()),
            "timing": "wall clock of montecarlo.run (host generation, tables and skeletons included); best "
                      "of 2 runs after a full-size warm-up", "runs_s": secs}


def bench_cfg5() -> dict:
    """configs[4]: ONE chain of 1e5 stages x 1e7 budget columns (capacity
    partitions over the whole GPU, checkpoint / recompute)."""
    import torch
    from paper_2410_10759_b200 import batch as B
    from paper_2410_10759_b200 import workloads as W
    x = W.cfg5()
    b = B.InstanceBatch.from_arrays(x["layer_off"], x["i"], x["s"], x["u"], x["d"], x["r"], x["budget"], x["sac"])
    B.plan_dp(b)
    torch.cuda.synchronize()
    e0, e1 = _events()
    e0.record()
    p = B.plan_dp(b)
    e1.record()
    torch.cuda.synchronize()
    sec = e0.elapsed_time(e1) / 1e3
    cells = 1e5 * (1e7 + 1)
    return {"L": 100000, "W": 10000000, "problem_cells": cells, "solve_s": sec,
            "problem_cells_per_s": cells / sec, "feasible": bool(p.feasible.item()),
            "timing": "CUDA events around plan_dp (warm)"}


# ---------------------------------------------------------------------------


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--requests", type=int, default=10_000)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="wall time of each CPU baseline sample")
    ap.add_argument("--cpu-sample", type=int, default=0, help="reference arm: requests per step (0: ~1.5 s)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the cfg3 / cfg4 / cfg5 legs")
    ap.add_argument("--no-dense", action="store_true", help="skip the dense-kernel and fp64 legs")
    ap.add_argument("--seed", type=int, default=2)
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    # SPLITPLAN_BENCH_BACKEND=gloo: exercise the N > 1 path with every rank on
    # the devices there are (a one-GPU box); the driver's runs use NCCL
    backend = os.environ.get("SPLITPLAN_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    from paper_2410_10759_b200 import _native as N
    from paper_2410_10759_b200 import batch as B
    from paper_2410_10759_b200 import cost_model as cm
    from paper_2410_10759_b200.requests import Engine, RequestBatch
    from paper_2410_10759_b200.shard import gather_policies

    req_np = cfg2_requests(args.requests, args.seed * 1000 + rank)
    n = args.requests
    layers = cm.build_preset("gpt2-24", 128).layers
    L = len(layers)
    total_layers = n * L
    engine = Engine([layers])
    dev = torch.device("cuda", local)
    host_req = RequestBatch.from_numpy(pin=True, **req_np)
    dev_req = host_req.to(dev)
    off = engine.layer_offsets(dev_req)
    stream = torch.cuda.current_stream()
    lib = N.library()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def step_device():
        s = engine.solve(dev_req, total_layers, off)
        if world > 1:  # the job's one collective: gather every rank's result records
            gather_policies(s.policies, s.layer_off)
        return s

    def step_e2e():
        r = host_req.to(dev, non_blocking=True)
        s = engine.solve(r, total_layers, off)
        pol = gather_policies(s.policies, s.layer_off)[0] if world > 1 else s.policies
        return s, pol.to_host_async()  # one packed device-to-host copy of the placements and records

    # Timed loops pipeline the steps: step k+1 is queued (Engine.solve_async,
    # its own workspace) before step k is collected (PendingSolve.result), so
    # the host's launch work overlaps the device's; every step still solves
    # its whole batch and is collected inside the timed region.
    # two pipeline slots (workspace, cost table, policies), allocated once:
    # no allocation inside the timed loops
    slots = []

    def run_device(steps: int):
        if not slots:
            slots.extend(engine.solve_slot(n, total_layers, N.workspace().numel()) for _ in range(2))
        prev = None
        for k in range(steps + 1):
            cur = engine.solve_async(dev_req, total_layers, off, slot=slots[k & 1]) if k < steps else None
            if prev is not None:
                s = prev.result()
                if world > 1:
                    gather_policies(s.policies, s.layer_off)
            prev = cur

    host_out = [None, None, None]  # pinned result buffers, reused round-robin

    phase_log = [] if os.environ.get("SPLITPLAN_BENCH_TRACE") == "phases" else None

    def run_e2e(steps: int):
        if not slots:
            slots.extend(engine.solve_slot(n, total_layers, N.workspace().numel()) for _ in range(2))
        prev, s, out = None, None, None
        for k in range(steps + 1):
            t = [time.perf_counter()]
            cur = None
            if k < steps:
                # the host request parameters: one host-to-device copy into the
                # slot, on the engine's copy stream (overlaps the previous step)
                cur = engine.solve_async(host_req, total_layers, off, slot=slots[k & 1])
            t.append(time.perf_counter())
            if prev is not None:
                if world > 1:
                    s = prev.result()
                    t.append(time.perf_counter())
                    pol = gather_policies(s.policies, s.layer_off)[0]
                    out = host_out[k % 3] = pol.to_host_async(into=host_out[k % 3])
                else:
                    # one packed device-to-host copy of the placements and records, on
                    # the copy stream (overlaps the next step)
                    s, out, _done = prev.result_to_host(into=host_out[k % 3])
                    host_out[k % 3] = out
                    t.append(time.perf_counter())
            t.append(time.perf_counter())
            if phase_log is not None:
                phase_log.append([round((b - a) * 1e3, 3) for a, b in zip(t, t[1:])])
            prev = cur
        return s, out

    for _ in range(max(args.warmup, 3)):
        step_device()
    barrier()
    sol = step_device()
    w_eff = B.effective_budget(sol.instances).cpu().numpy()
    cells = float(L * (w_eff + 1).sum())
    assert int(sol.status.abs().sum().item()) == 0, "cost-table errors in the workload"
    domains = value_domains(sol.instances.r.cpu().numpy(), sol.layer_off.cpu().numpy())
    del sol

    # ---- device-resident timing (no instrumentation inside) --------------
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    run_device(max(args.warmup, 3))  # the pipelined path and its second workspace, untimed
    barrier()
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        run_device(args.steps)
        ev1.record(stream)
        clocks.sample_now()
        barrier()
    dev_ms = ev0.elapsed_time(ev1)
    clk = clocks.summary()
    _CLOCK_HINT[0] = clk.get("sm_mhz") if isinstance(clk, dict) else None

    # ---- kernel accounting (a separate, instrumented pass) ----------------
    barrier()
    with Profile(lib) as prof:
        for _ in range(args.steps):
            step_device()
        barrier()

    # ---- end-to-end timing (host buffers, copies inside) ------------------
    # warm the host <-> device path (pinned staging, allocator) holding the
    # previous step's results while the next one runs, as the timed loop does
    s, out = run_e2e(max(args.warmup, 3))
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    trace = os.environ.get("SPLITPLAN_BENCH_TRACE")
    tw = []
    e0.record(stream)
    if trace and phase_log is None:
        for _ in range(args.steps):
            tw.append(time.perf_counter())
            s, out = step_e2e()
    else:
        s, out = run_e2e(args.steps)
    stream.wait_stream(engine.copy_stream())  # the last results' copy is inside the timed region
    e1.record(stream)
    if trace and phase_log is None:
        tw.append(time.perf_counter())
        print("e2e step wall ms:", [round((b - a) * 1e3, 3) for a, b in zip(tw, tw[1:])], file=sys.stderr)
    if phase_log is not None:
        print("e2e phases ms (queue, result, copy):", phase_log, file=sys.stderr)
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    d2h = out._buf.numel()
    del s

    t = torch.tensor([dev_ms, e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms, e2e_ms = float(t[0]), float(t[1])
    step_ms = dev_ms / args.steps
    total_cells = cells * world
    value = total_cells / (step_ms / 1e3)

    # ---- the same batch on the dense kernel, and in the fp64 domain -------
    legs = {}
    if not args.no_dense and world == 1:
        legs = dense_and_f64_legs(engine, dev_req, total_layers, off, cells, lib)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "DP cells/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": step_ms,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": dtype_label(domains),
            "data": "synthetic (seeded cfg2 request parameters; no datasets involved)",
            "config": {
                "workload": "cfg2: gpt2-24 (L=98), 10k requests/GPU, W_eff=1e5 units",
                "requests_per_gpu": n, "layers_per_request": L,
                "dp_cells_per_gpu_step": cells,
                "dp_cell": "one cell of the reference's (L+1) x (W_eff+1) DP tables (planner.py:128-143); "
                           "solved as breakpoint lists (bit-identical tables, DESIGN.md 4)",
                "value_domains": domains,
                "seq_len": "U{128..2048}", "links_bps": "log-U[3e7,1e9] sym, 10 ms prop",
                "deadline": "f x all-client time, f~U(0.05,1); unit = deadline/1e5",
                "step": "Engine.solve: K1 cost table + prep + K2 DP + K3 backtrack",
                "pipelining": "step k+1 queued (Engine.solve_async) before step k is collected; two reused slots "
                              "(workspace, cost table, policies); e2e: each step's request upload and result "
                              "download run on the engine's copy stream, overlapping the neighbouring steps' "
                              "kernels",
                "l2": "inputs and outputs larger than L2: each step writes ~%.1f GB of breakpoint stores "
                      "(CUDA-event timing, no flush needed)" % (prof.bytes / max(prof.n, 1) / 1e9),
                "parallelism": f"request-sharded dp{world}",
                "collective": "none in the solve; one all_gather of result records per step when N > 1",
                "scenario": "scenarios_per_s counts solved requests: one (model, seq_len, link, deadline) "
                            "placement problem, a run_sweep cell of the reference (evaluator.py:211-226); the "
                            "Monte-Carlo grid's scenarios/s (configs[3]) is configs.cfg4.scenarios_per_s",
            },
            "scenarios_per_s": n * world / (step_ms / 1e3),
            "e2e": {"value": total_cells / (e2e_ms / args.steps / 1e3), "unit": "DP cells/s",
                    "scenarios_per_s": n * world / (e2e_ms / args.steps / 1e3),
                    "ms_per_step": e2e_ms / args.steps,
                    "h2d_bytes_per_step": host_req._buf.numel(), "d2h_bytes_per_step": d2h},
            "gpu_launches": int(prof.launches),
            # the kernel's share of the device-timed (pipelined) steps: the
            # accounting pass runs the same step count unpipelined, with host
            # gaps between its steps
            "roofline": roofline(prof, dev_ms),
            "clocks": clk,
        }
        line.update(legs)
        if not args.no_configs and world == 1:
            line["configs"] = {"cfg3": bench_cfg3(), "cfg4": bench_cfg4(), "cfg5": bench_cfg5()}
        if not args.no_cpu_baseline and world == 1:  # rank 0 at N=1 only
            line["cpu_baseline"] = cpu_baseline(req_np, args.cpu_seconds)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def dense_and_f64_legs(engine, dev_req, total_layers, off, cells, lib) -> dict:
    """The benchmark batch forced onto the dense L2-streaming kernel (what the
    breakpoint lists replace), and the same instances with every r_k scaled
    by (1 + 2^-20) so the DP runs in the fp64 value domain (the reference's
    general case, planner.py:139-142), on the engine's default path and dense."""
    import torch
    from paper_2410_10759_b200 import batch as B

    def timed(fn, steps, *, variant=None):
        if variant:
            os.environ["SPLITPLAN_DP_VARIANT"] = variant
        try:
            fn()
            torch.cuda.synchronize()
            with Profile(lib) as prof:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(steps):
                    fn()
                e1.record()
                torch.cuda.synchronize()
            return e0.elapsed_time(e1) / steps, prof
        finally:
            os.environ.pop("SPLITPLAN_DP_VARIANT", None)

    out = {}
    ms, prof = timed(lambda: engine.solve(dev_req, total_layers, off), 3, variant="stream")
    out["dense_kernel"] = {"value": cells / (ms / 1e3), "unit": "DP cells/s", "ms_per_step": ms,
                           "what": "the same cfg2 batch forced onto the dense kernels (SPLITPLAN_DP_VARIANT=stream)",
                           "roofline": roofline(prof, ms * 3)}
    sol = engine.solve(dev_req, total_layers, off)
    inst = sol.instances
    f64 = B.InstanceBatch(inst.layer_off, inst.client_units, inst.server_units, inst.up_units, inst.down_units,
                          inst.r * (1.0 + 2.0 ** -20), inst.budget, inst.source_at_client)
    domains = value_domains(f64.r.cpu().numpy(), f64.layer_off.cpu().numpy())
    ms, prof = timed(lambda: B.plan_dp(f64), 5)
    out["f64_domain"] = {"value": cells / (ms / 1e3), "unit": "DP cells/s", "ms_per_step": ms,
                         "value_domains": domains,
                         "what": "cfg2 instances with r x (1 + 2^-20): prep + K2 + K3 (B.plan_dp) in the fp64 domain",
                         "dense_fallbacks": int(lib.sp_last_dense_fallbacks()),
                         "roofline": roofline(prof, ms * 5)}
    ms, prof = timed(lambda: B.plan_dp(f64), 2, variant="stream")
    out["f64_domain"]["dense_kernel"] = {"value": cells / (ms / 1e3), "unit": "DP cells/s", "ms_per_step": ms,
                                         "roofline": roofline(prof, ms * 2)}
    return out


def run_reference(args, rank: int, world: int):
    """The reference arm: the oracle port of the reference path (profile ->
    build_problem -> plan_dp) on every host core, rank 0 only.  The process
    pool is created before the timed steps; each step is a bounded sample of
    about 2.5 s of wall time on all cores (>= 8 requests per worker)."""
    if rank != 0:
        return
    req_np = cfg2_requests(args.requests, args.seed * 1000)
    procs = max(1, min(os.cpu_count() or 1, 128))
    pool = CpuPool(procs)
    try:
        pool.run(_cpu_jobs(req_np, range(procs)))  # fork + first touch, untimed
        # calibration on warm workers: two requests each; a step then gives every
        # worker >= 8 requests (about 2.5 s), so the slowest worker's tail is a
        # small part of the step (with ~5 per worker the arm read half the rate
        # of cpu_baseline on the same box)
        _cells, dt = pool.run(_cpu_jobs(req_np, np.arange(2 * procs) % args.requests))
        per_worker = max(8, int(round(2.5 / max(dt / 2, 1e-3))))
        per = args.cpu_sample or min(procs * per_worker, args.requests)
        times, cells_tot = [], 0.0
        for s in range(args.warmup + args.steps):
            idx = (np.arange(per) + s * per) % args.requests
            cells, dt = pool.run(_cpu_jobs(req_np, idx))
            if s >= args.warmup:
                times.append(dt)
                cells_tot += cells
    finally:
        pool.close()
    wall = sum(times)
    value = cells_tot / wall
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "DP cells/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / max(len(times), 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded cfg2 request parameters)",
        "config": {"workload": "cfg2: gpt2-24 (L=98), W_eff=1e5 units; CPU sample of "
                               f"{per} requests per step",
                   "parallelism": f"{procs} processes (one pool, created before timing)"},
        "scenarios_per_s": per * len(times) / wall,
        "cpu_baseline": {"value": value, "unit": "DP cells/s", "cores": procs, "kind": "port",
                         "sample": f"{per} cfg2 requests per step (profile -> build_problem -> plan_dp, numpy "
                                   "port of the reference)", **cpu_info()},
        "e2e": {"value": value, "unit": "DP cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
