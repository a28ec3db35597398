"""Per-step wall and device time of the bench step (host jitter check)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

if __name__ == "__main__":
    import torch
    import bench
    from paper_2410_10759_b200 import cost_model as cm
    from paper_2410_10759_b200.requests import Engine, RequestBatch
    req_np = bench.cfg2_requests(10_000, 2000)
    L = len(cm.build_preset("gpt2-24", 128).layers)
    engine = Engine([cm.build_preset("gpt2-24", 128).layers])
    dev_req = RequestBatch.from_numpy(pin=True, **req_np).to("cuda")
    off = engine.layer_offsets(dev_req)
    out = []
    for s in range(12):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record()
        engine.solve(dev_req, 10_000 * L, off)
        e1.record()
        torch.cuda.synchronize()
        out.append((round((time.perf_counter() - t0) * 1e3, 2), round(e0.elapsed_time(e1), 2)))
    print(json.dumps(out))
