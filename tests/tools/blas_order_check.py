"""Check the summation order the exhaustive kernel replicates for `x @ r`
(planner.py:253) against numpy on this host (test infrastructure, CPU).

numpy passes the (masks x L) @ (L,) product to OpenBLAS dgemv_t; the model
(csrc/sp_planner.cu mask_value): four lane-strided accumulators over the first
4*floor(L/4) layers reduced as (a0 + a2) + (a1 + a3), then the last L mod 4
layers left to right.  Decimal r make the order visible (0.1 + 0.2 != 0.3).

    python tests/tools/blas_order_check.py > profiles/r02/oracle_blas_order.json
"""
import json

import numpy as np


def model(x, r):
    L = len(r)
    m3 = L & 3
    m1 = L - m3
    y = 0.0
    if m1:
        a = [0.0, 0.0, 0.0, 0.0]
        for i in range(m1):
            a[i & 3] = a[i & 3] + x[i] * r[i]
        y = y + ((a[0] + a[2]) + (a[1] + a[3]))
    if m3:
        t = x[m1] * r[m1]
        for i in range(m1 + 1, L):
            t = t + x[i] * r[i]
        y = y + t
    return y


def main():
    rng = np.random.default_rng(1)
    vals = np.array([0.1, 0.2, 0.3, 0.7, 1.1, 0.05, 0.15, 2.2, 1e-3, 3.3])
    total = bad = seq_bad = 0
    for L in range(1, 25):
        for _ in range(40):
            r = rng.choice(vals, L) * rng.choice([1.0, 1.0, 1.37], L)
            n = 64 if L >= 6 else 2 ** L
            ms = rng.integers(0, 2 ** L, n)
            x = np.array([[(m >> (L - 1 - k)) & 1 for k in range(L)] for m in ms], dtype=float)
            v = x @ r
            for q in range(n):
                total += 1
                bad += model(x[q], r) != v[q]
                seq = 0.0
                for k in range(L):
                    seq += x[q, k] * r[k]
                seq_bad += seq != v[q]
    try:
        import threadpoolctl
        blas = [{k: d.get(k) for k in ("internal_api", "version", "architecture")}
                for d in threadpoolctl.threadpool_info() if d.get("user_api") == "blas"]
    except Exception:
        blas = None
    print(json.dumps({"masks_checked": total, "model_mismatches": int(bad),
                      "sequential_sum_mismatches": int(seq_bad), "numpy": np.__version__, "blas": blas},
                     indent=1))


if __name__ == "__main__":
    main()
