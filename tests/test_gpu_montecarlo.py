"""cfg4 Monte-Carlo sweep on the GPU against the live reference's own pipeline
(golden vectors from tests/golden/gen_montecarlo.py): scenario tables,
capacities, and per-variant max / mean FIFO waits, bit for bit."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_json, same_float

pytestmark = pytest.mark.gpu


def test_montecarlo_matches_reference(gpu):
    from paper_2410_10759_b200 import montecarlo as MC
    doc = load_json("montecarlo.json")
    res = MC.run(doc["sids"], beta_per_ms=doc["beta_per_ms"], horizon=doc["horizon"],
                 omega_requests=doc["omega"])
    for s, exp in enumerate(doc["scenarios"]):
        assert res.table_size[s] == exp["table_size"], exp["sid"]
        if not exp["table_size"]:
            assert np.all(res.status[s] == -1)
            continue
        assert same_float(res.capacity[s], exp["capacity"]), exp["sid"]
        if "deadlock" in exp:
            assert np.any(res.status[s] == 5)
            continue
        assert np.all(res.status[s] == 0)
        for v in range(3):
            assert same_float(res.max_wait_ms[s, v], exp["max_wait_ms"][v]), (exp["sid"], v)
            assert same_float(res.mean_wait_ms[s, v], exp["mean_wait_ms"][v]), (exp["sid"], v)


def test_montecarlo_grid_slice_properties(gpu):
    """1,024 scenarios: dp never waits longer than nosplit on average when both
    ran, and every simulated scenario sized its server to 500 nosplit requests."""
    from paper_2410_10759_b200 import montecarlo as MC
    res = MC.run(np.arange(0, 65536, 64))
    sim = res.table_size > 0
    assert sim.mean() > 0.5
    ok = sim & np.all(res.status == 0, axis=1)
    assert np.allclose(res.capacity[ok], 500.0, rtol=1e-12)
    assert np.all(res.mean_wait_ms[ok, 0] <= res.mean_wait_ms[ok, 2] + 1e-9)


def test_device_skeletons_equal_numpy_draws(gpu):
    """sp_sim_skeletons (one thread per run) draws numpy's default_rng(seed)
    stream bit for bit (throughput_sim.py:179-186): 4,096 seeds x 2,000
    requests -- about 3,700 ziggurat tail draws through the device log1p --
    with table ranges from one row (no draw) to 2^31 rows."""
    from paper_2410_10759_b200.throughput_sim import skeletons_device
    horizon, beta = 2000, 0.057
    seeds = np.arange(4096, dtype=np.int64) * 7 + 3
    spans = np.array([1, 2, 3, 64, 1000, 2 ** 31 - 1])[np.arange(4096) % 6]
    lo = np.arange(4096, dtype=np.int64) % 5
    arr, rows, ex = (x.cpu().numpy() for x in skeletons_device(seeds, lo, lo + spans, horizon, beta, 10))
    for r in range(4096):
        g = np.random.default_rng(int(seeds[r]))
        a = np.cumsum(g.exponential(scale=1.0 / beta, size=horizon))
        c = g.integers(0, spans[r], size=horizon) + lo[r]
        e = g.integers(1, 11, size=horizon)
        assert np.array_equal(arr[r].view(np.int64), a.view(np.int64)), r
        assert np.array_equal(rows[r], c), r
        assert np.array_equal(ex[r], e), r


def test_device_skeletons_reject_empty_ranges(gpu):
    from paper_2410_10759_b200.throughput_sim import skeletons_device
    with pytest.raises(ValueError):
        skeletons_device([1, 2], [0, 5], [3, 5], 10, 0.057)
