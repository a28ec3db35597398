"""cProfile of one cfg4 Monte-Carlo run (host phases vs device passes).

    python tools/mc_profile.py [--scenarios 16384]
"""
import argparse
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scenarios", type=int, default=16384)
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2410_10759_b200 import montecarlo as MC
    MC.run(np.arange(256))  # warm-up (library load, kernels)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    MC.run(np.arange(args.scenarios))
    torch.cuda.synchronize()
    pr.disable()
    print("wall_s", time.perf_counter() - t0)
    pstats.Stats(pr).sort_stats("cumulative").print_stats(35)


if __name__ == "__main__":
    main()
