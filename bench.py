"""Benchmark: DP cells/s and solved requests/s of the SplitLLM placement engine.

Workload (BASELINE.json configs[1]): gpt2-24 (L = 98
splittable entries), 10,000 requests per GPU, seq_len ~ U{128..2048}, symmetric
links log-uniform in [3e7, 1e9] bit/s with 10 ms propagation, deadline = f x
all-client time with f ~ U(0.05, 1), unit_s = deadline / 1e5 so every request
has W = W_eff = 100,000 budget columns.  Devices calibrated as the reference
acceptance suite (bert-12 @ 4096 tokens: 7.727 s client, 0.0979 s server).

One step = the hot path over the whole batch: K1 cost table -> prep -> K2 DP
stage -> K3 backtrack (every request gets its optimal placement).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun each rank solves its own 10k requests (weak scaling); the step
time is the max over ranks.  `--impl reference` times the CPU oracle port of
the reference path (profile -> build_problem -> plan_dp) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
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


# ---------------------------------------------------------------------------
# CPU side: the oracle port of the reference path, timed on host cores


def _cpu_one(args):
    from oracle import splitplan_oracle as O
    layers, s, cf, sf, bw, prop, dl, unit = args
    r, cs, ss, tau = O.profile_arrays(layers, int(s), cf, sf)
    inst = O.instance_from_profile(r, cs, ss, tau, bw, bw, prop, dl, unit)
    p = O.plan_dp(inst)
    return len(r) * (O.effective_budget(inst) + 1), p["integer_latency"]


def cpu_run(req: dict, idx, procs: int):
    """Returns (cells, seconds) for the sampled requests on `procs` processes."""
    from multiprocessing import get_context
    from oracle import splitplan_oracle as O
    layers = O.preset_layers("gpt2-24")
    jobs = [(layers, req["seq_len"][k], req["client_fps"][k], req["server_fps"][k],
             req["uplink_bps"][k], req["propagation_s"][k], req["deadline_s"][k],
             req["unit_s"][k]) for k in idx]
    t0 = time.perf_counter()
    if procs <= 1:
        out = [_cpu_one(j) for j in jobs]
    else:
        with get_context("fork").Pool(procs) as pool:
            out = pool.map(_cpu_one, jobs, chunksize=1)
    dt = time.perf_counter() - t0
    return sum(c for c, _ in out), dt


# ---------------------------------------------------------------------------
# clocks


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------


def measured_peak_hbm():
    try:
        doc = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(doc["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


VARIANTS = ["dp_stage_kernel<smem rows>", "dp_cluster_kernel<DSMEM rows>",
            "dp_stage_kernel<global rows>", "dp_coop_kernel<L2 rows>",
            "dp_stream_kernel<L2 rows, bulk-copy staged windows>",
            "dp_grid_kernel<one instance over the GPU>",
            "dp_own_kernel<own block in SMEM, remote windows via L2>",
            "dp_steps_kernel<rows as breakpoint lists>"]
NCU_SUMMARY = {0: "dp_smem_ncu_summary.json", 3: "dp_coop_ncu_summary.json",
               4: "dp_stream_ncu_summary.json"}


def ncu_traffic(variant: int, cells_per_launch: float):
    """DRAM bytes per launch, scaled from the newest committed ncu capture of this
    variant (profiles/rNN/*_ncu_summary.json holds DRAM bytes per DP cell)."""
    name = NCU_SUMMARY.get(variant)
    if not name:
        return None, None
    for d in sorted((ROOT / "profiles").glob("r*"), reverse=True):
        f = d / name
        if f.exists():
            doc = json.loads(f.read_text())
            return doc["dram_bytes_per_cell"] * cells_per_launch, str(f.relative_to(ROOT))
    return None, None


def _latest_summary(name: str):
    for d in sorted((ROOT / "profiles").glob("r*"), reverse=True):
        f = d / name
        if f.exists():
            return json.loads(f.read_text()), str(f.relative_to(ROOT))
    return None, None


def onchip_roofline(variant: int, cells_per_s: float, sm_mhz: float | None) -> dict | None:
    """The resource the DP stage kernel's rows live in (they never reach HBM).

    smem rows: 4 LDS + 2 STS words per cell = 24 B of SMEM traffic (4 B values);
    peak 128 B/clk/SM x 148 SMs.  L2 rows (stream / grid): 16 B of bulk-copy L2
    reads + 8 B of L2 writes per cell; peak = the L2 sector throughput the
    committed ncu capture of the kernel implies (lts__t_sectors per second /
    its pct_of_peak), else 6,300 B/clk (B300_MICROARCH.md LTS cap)."""
    clk = (sm_mhz or 1965.0) * 1e6
    src = "SMEM 128 B/clk/SM"
    if variant == 0:
        per_cell, peak, res = 24.0, 128.0 * 148 * clk, "smem"
    elif variant in (3, 4, 5):
        per_cell, res = 24.0, "l2"
        doc, path = _latest_summary("dp_stream_ncu_summary.json")
        if doc and doc.get("l2_peak_Bps_implied"):
            peak, src = doc["l2_peak_Bps_implied"], f"ncu-implied L2 sector peak ({path})"
        else:
            peak, src = 6300.0 * clk, "6300 B/clk LTS cap (B300_MICROARCH.md)"
    else:
        return None
    ach = cells_per_s * per_cell
    return {"resource": res, "bytes_per_cell": per_cell, "achieved_GBps": ach / 1e9,
            "peak_GBps": peak / 1e9, "peak_source": src, "frac": ach / peak}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--requests", type=int, default=10_000)
    ap.add_argument("--cpu-sample", type=int, default=0, help="requests timed on the CPU")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--seed", type=int, default=2)
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2410_10759_b200 import _native as N
    from paper_2410_10759_b200 import cost_model as cm
    from paper_2410_10759_b200.requests import Engine, RequestBatch

    req_np = cfg2_requests(args.requests, args.seed * 1000 + rank)
    n = args.requests
    L = len(cm.build_preset("gpt2-24", 128).layers)
    total_layers = n * L
    engine = Engine([cm.build_preset("gpt2-24", 128).layers])
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

    from paper_2410_10759_b200.shard import gather_policies

    def step_device():
        s = engine.solve(dev_req, total_layers, off)
        if world > 1:  # the job's one collective: gather every rank's result records
            gather_policies(s.policies, s.layer_off)
        return s

    def step_e2e():
        r = host_req.to(dev, non_blocking=True)
        s = engine.solve(r, total_layers, off)
        pol = gather_policies(s.policies, s.layer_off)[0] if world > 1 else s.policies
        out = (pol.pi.to("cpu", non_blocking=True),
               pol.client_value.to("cpu", non_blocking=True),
               pol.server_load.to("cpu", non_blocking=True),
               pol.integer_latency.to("cpu", non_blocking=True),
               pol.feasible.to("cpu", non_blocking=True))
        return s, out

    for _ in range(max(args.warmup, 0)):
        step_device()
    barrier()
    # cells of one step (W_eff from the device prep, identical every step)
    sol = step_device()
    from paper_2410_10759_b200 import batch as B
    w_eff = B.effective_budget(sol.instances).cpu().numpy()
    cells = float(L * (w_eff + 1).sum())
    assert int(sol.status.abs().sum().item()) == 0, "cost-table errors in the workload"

    # ---- device-resident timing -----------------------------------------
    lib.sp_profile_enable(1)
    lib.sp_profile_collect(None, None, None, None, None, None)
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            step_device()
        ev1.record(stream)
        barrier()
    dev_ms = ev0.elapsed_time(ev1)
    import ctypes as C
    dk_ms, dk_n, dk_cells, dk_bytes, all_l, dk_var = (C.c_double(), C.c_int64(), C.c_double(),
                                                      C.c_double(), C.c_int64(), C.c_int32())
    lib.sp_profile_collect(C.byref(dk_ms), C.byref(dk_n), C.byref(dk_cells), C.byref(dk_bytes),
                           C.byref(all_l), C.byref(dk_var))
    lib.sp_profile_enable(0)

    # ---- end-to-end timing (host buffers, copies inside) ------------------
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        s, out = step_e2e()
    e1.record(stream)
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    d2h = sum(t.numel() * t.element_size() for t in out)

    t = torch.tensor([dev_ms, e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms, e2e_ms = float(t[0]), float(t[1])
    step_ms = dev_ms / args.steps
    total_cells = cells * world
    value = total_cells / (step_ms / 1e3)

    if rank == 0:
        peak, peak_kind = measured_peak_hbm()
        avg_launch_ms = dk_ms.value / max(dk_n.value, 1)
        bytes_per_launch = dk_bytes.value / max(dk_n.value, 1)
        achieved = bytes_per_launch / (avg_launch_ms / 1e3) / 1e9 if avg_launch_ms > 0 else None
        cells_per_launch = dk_cells.value / max(dk_n.value, 1)
        kernel_rate = dk_cells.value / (dk_ms.value / 1e3) if dk_ms.value else None
        traffic, traffic_src = ncu_traffic(dk_var.value, cells_per_launch)
        clk = clocks.summary()
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
            "dtype": "int32",
            "data": "synthetic (seeded cfg2 request parameters; no datasets involved)",
            "config": {
                "workload": "cfg2: gpt2-24 (L=98), 10k requests/GPU, W_eff=1e5 units",
                "requests_per_gpu": n, "layers_per_request": L,
                "dp_cells_per_gpu_step": cells,
                "seq_len": "U{128..2048}", "links_bps": "log-U[3e7,1e9] sym, 10 ms prop",
                "deadline": "f x all-client time, f~U(0.05,1); unit = deadline/1e5",
                "step": "K1 cost table + prep + K2 DP stage + K3 backtrack",
                "l2": "inputs larger than L2: each step writes ~%.1f GB of packed back-pointers"
                      % (cells / 4 / 1e9),
                "parallelism": f"request-sharded dp{world}",
                "collective": "none in the solve; one all_gather of result records per step when N > 1",
            },
            "scenarios_per_s": n * world / (step_ms / 1e3),
            "e2e": {"value": total_cells / (e2e_ms / args.steps / 1e3), "unit": "DP cells/s",
                    "scenarios_per_s": n * world / (e2e_ms / args.steps / 1e3),
                    "h2d_bytes_per_step": host_req.host_bytes(), "d2h_bytes_per_step": d2h},
            "gpu_launches": int(all_l.value),
            "roofline": {
                "kernel": VARIANTS[dk_var.value],
                "bound": "hbm",
                "achieved": achieved,
                "peak": peak,
                "peak_kind": peak_kind,
                "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None,
                "traffic": traffic,
                "traffic_source": traffic_src,
                "bytes_per_cell": bytes_per_launch / max(cells_per_launch, 1),
                "launches": dk_n.value,
                "avg_launch_ms": avg_launch_ms,
                "share_of_step": dk_ms.value / dev_ms if dev_ms else None,
                "cells_per_s_in_kernel": kernel_rate,
                "onchip": onchip_roofline(dk_var.value, kernel_rate, clk.get("sm_mhz")),
                "row_streaming_ceiling_cells_per_s": peak * 1e9 / 33.0,
                # the survey's row-streaming design moves 33 B per cell through
                # HBM: the HBM bandwidth it would need for this kernel's rate
                "row_streaming_equivalent": ({
                    "bytes_per_cell": 33.0,
                    "GBps": kernel_rate * 33.0 / 1e9,
                    "frac_of_hbm_peak": kernel_rate * 33.0 / (peak * 1e9)} if kernel_rate else None),
            },
            "clocks": clk,
        }
        if not args.no_cpu_baseline and world == 1:  # rank 0 at N=1 only
            line["cpu_baseline"] = cpu_baseline(req_np, args.cpu_sample)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def cpu_baseline(req_np: dict, sample: int) -> dict:
    procs = max(1, min(os.cpu_count() or 1, 64))
    # ~0.12 s of single-core numpy per cfg2 request: 128 per process is ~15 s wall
    sample = sample or max(64, 128 * procs)
    idx = np.arange(min(sample, len(req_np["seq_len"])))
    cells, dt = cpu_run(req_np, idx, procs)
    return {"value": cells / dt, "unit": "DP cells/s", "cores": procs, "kind": "port",
            "sample": f"{len(idx)} cfg2 requests (profile -> build_problem -> plan_dp, oracle "
                      f"numpy port) on {procs} processes, {dt:.1f} s wall",
            "scenarios_per_s": len(idx) / dt}


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    from paper_2410_10759_b200 import cost_model as cm  # noqa: F401  (host-only import)
    req_np = cfg2_requests(args.requests, args.seed * 1000)
    procs = max(1, min(os.cpu_count() or 1, 128))
    per = args.cpu_sample or max(8, 4 * procs)  # ~0.5 s of host work per step
    times, cells_tot = [], 0.0
    for s in range(args.warmup + args.steps):
        idx = (np.arange(per) + s * per) % args.requests
        cells, dt = cpu_run(req_np, idx, procs)
        if s >= args.warmup:
            times.append(dt)
            cells_tot += cells
    wall = sum(times)
    value = cells_tot / wall
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "DP cells/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / max(len(times), 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded cfg2 request parameters)",
        "config": {"workload": "cfg2: gpt2-24 (L=98), W_eff=1e5 units; CPU sample of "
                               f"{per} requests per step", "parallelism": f"{procs} processes"},
        "scenarios_per_s": per * len(times) / wall,
        "cpu_baseline": {"value": value, "unit": "DP cells/s", "cores": procs, "kind": "port",
                         "sample": f"{per} cfg2 requests per step (profile -> build_problem -> "
                                   "plan_dp, numpy port of the reference)"},
        "e2e": {"value": value, "unit": "DP cells/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
