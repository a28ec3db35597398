"""Wall time of the cfg4 Monte-Carlo run (montecarlo.run) at a given scenario count."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

if __name__ == "__main__":
    import os
    import numpy as np
    import torch
    from paper_2410_10759_b200 import montecarlo as MC
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    MC.run(np.arange(256))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = MC.run(np.arange(n))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps({"scenarios": n, "wall_s": dt, "scenarios_per_s": n / dt, "cpus": os.cpu_count(),
                      "skeletons": "device",
                      "requests": r.requests, "dp_cells": r.dp_cells}))
