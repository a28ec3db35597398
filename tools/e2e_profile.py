"""Where the end-to-end step of bench.py goes (host buffers in, results out).

    python tools/e2e_profile.py [--steps 5]

Runs bench.py's `step_e2e` under torch.profiler (CPU ops + CUDA kernels and
copies) after warm-up and prints, for the last step, a timeline of the host
calls and device activities in microseconds from the step start, plus the
device-busy fraction.  Timings under the profiler are for attribution only.
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--requests", type=int, default=10_000)
    ap.add_argument("--blocks", type=int, default=0, help="N blocks of 20 device / e2e steps, with SM clocks")
    ap.add_argument("--plain", action="store_true", help="no profiler: CUDA-event times of device and e2e steps")
    ap.add_argument("--pipelined", action="store_true", help="e2e steps as bench.py times them (solve_async)")
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile, record_function
    import bench
    from paper_2410_10759_b200 import cost_model as cm
    from paper_2410_10759_b200.requests import Engine, RequestBatch

    req_np = bench.cfg2_requests(args.requests, 2000)
    layers = cm.build_preset("gpt2-24", 128).layers
    eng = Engine([layers])
    dev = torch.device("cuda", 0)
    host_req = RequestBatch.from_numpy(pin=True, **req_np)
    dev_req = host_req.to(dev)
    off = eng.layer_offsets(dev_req)
    total = args.requests * len(layers)

    from paper_2410_10759_b200 import _native as N
    state = {"prev": None, "k": 0, "ws": None, "out": [None, None, None]}

    def step_e2e():
        if not args.pipelined:
            r = host_req.to(dev, non_blocking=True)
            s = eng.solve(r, total, off)
            return s.policies.to_host_async()
        # bench.py's timed loop: queue step k, then collect step k - 1
        if state["ws"] is None:
            eng.solve(dev_req, total, off)  # sizes the cached workspace for the batch
            state["ws"] = [N.workspace(), torch.empty_like(N.workspace())]
        k = state["k"]
        cur = eng.solve_async(host_req.to(dev, non_blocking=True), total, off, ws=state["ws"][k & 1])
        out = None
        if state["prev"] is not None:
            s = state["prev"].result()
            out = state["out"][k % 3] = s.policies.to_host_async(into=state["out"][k % 3])
        state["prev"], state["k"] = cur, k + 1
        return out

    for _ in range(5):
        step_e2e()
    torch.cuda.synchronize()
    if args.blocks:
        import pynvml as nv
        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(0)
        for b in range(args.blocks):
            for name, fn in (("device", lambda: eng.solve(dev_req, total, off)), ("e2e", step_e2e)):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(20):
                    out = fn()
                clk = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                e1.record()
                torch.cuda.synchronize()
                print(json.dumps({"block": b, "kind": name, "ms": e0.elapsed_time(e1) / 20, "sm_mhz": clk,
                                  "reasons": nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)}))
                del out
        return
    if args.plain:
        import time
        res = {}
        for name, fn in (("device", lambda: eng.solve(dev_req, total, off)), ("e2e", step_e2e),
                         ("device2", lambda: eng.solve(dev_req, total, off)), ("e2e2", step_e2e)):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record()
            for _ in range(20):
                out = fn()
            e1.record()
            torch.cuda.synchronize()
            res[name] = {"event_ms": e0.elapsed_time(e1) / 20, "wall_ms": (time.perf_counter() - t0) * 50}
            del out
        print(json.dumps(res))
        return
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for i in range(args.steps):
            with record_function(f"step{i}"):
                step_e2e()
        torch.cuda.synchronize()
    ev = prof.events()
    last = [e for e in ev if e.name == f"step{args.steps - 1}"][0]
    t0 = last.time_range.start
    t1 = last.time_range.end
    rows = []
    for e in ev:
        s = e.time_range.start
        if s < t0 or s > t1 + 5000:
            continue
        dev_kind = e.device_type.name
        rows.append((s - t0, e.time_range.elapsed_us(), dev_kind, e.name[:90]))
    rows.sort()
    busy = sum(r[1] for r in rows if r[2] == "CUDA")
    for r in rows:
        if r[1] >= 3 or r[2] == "CUDA":
            print(f"{r[0]:9.1f} {r[1]:9.1f} {r[2]:5s} {r[3]}")
    print(json.dumps({"step_us": t1 - t0, "device_busy_us": busy}))
    print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=30))


if __name__ == "__main__":
    main()
