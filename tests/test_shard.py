"""Multi-rank host logic of the sharded path on CPU (gloo, world_size 2).

The GPU job shards independent requests/scenarios over ranks and gathers the
fixed-size result records once at the end; here the same
code runs over gloo with CPU tensors standing in for each rank's solved
shard, and the gathered job must equal the unsharded concatenation.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_10759_b200.batch import PolicyBatch
from paper_2410_10759_b200.shard import gather_policies, shard_bounds, shard_by_cost


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _fake_shard(seed: int, n: int):
    """A deterministic stand-in for one rank's solved shard."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, 40, n)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    pol = PolicyBatch(torch.from_numpy(rng.integers(0, 2, off[-1]).astype(np.uint8)),
                      torch.from_numpy(rng.random(n) * 1e12),
                      torch.from_numpy(np.where(rng.random(n) < 0.1, -np.inf, rng.random(n))),
                      torch.from_numpy(rng.integers(-5, 10 ** 12, n)),
                      torch.from_numpy(rng.integers(0, 2, n).astype(np.uint8)),
                      torch.from_numpy(rng.integers(0, 5, n).astype(np.int32)))
    return pol, torch.from_numpy(off)




def _worker(rank: int, world: int, port: int, sizes, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pol, off = _fake_shard(100 + rank, sizes[rank])
        got, goff = gather_policies(pol, off)
        parts = [_fake_shard(100 + r, sizes[r]) for r in range(world)]
        exp_pi = torch.cat([p.pi for p, _ in parts])
        ok = torch.equal(got.pi, exp_pi)
        for f in ("client_value", "server_load", "integer_latency", "feasible", "status"):
            e = torch.cat([getattr(p, f) for p, _ in parts])
            g = getattr(got, f)
            ok &= g.dtype == e.dtype and torch.equal(g.view(torch.uint8) if g.is_floating_point() else g,
                                                     e.view(torch.uint8) if e.is_floating_point() else e)
        lens = torch.cat([o[1:] - o[:-1] for _, o in parts])
        ok &= torch.equal(goff[1:] - goff[:-1], lens) and int(goff[0]) == 0
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("sizes", [(37, 64), (0, 5), (12, 12)])
def test_gather_policies_gloo_world2(sizes):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, sizes, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert results == {0: True, 1: True}


def test_shard_bounds():
    for n in (0, 1, 7, 10_000):
        for w in (1, 2, 3, 8):
            off = shard_bounds(n, w)
            assert off[0] == 0 and off[-1] == n and np.all(np.diff(off) >= 0)
            assert np.diff(off).max() - np.diff(off).min() <= 1


def test_shard_by_cost_balances_cells():
    rng = np.random.default_rng(3)
    cost = rng.integers(1, 1000, 5000) * rng.integers(1, 100, 5000)
    for w in (1, 2, 4, 8):
        off = shard_by_cost(cost, w)
        assert off[0] == 0 and off[-1] == cost.size and np.all(np.diff(off) >= 0)
        per = np.array([cost[off[r]:off[r + 1]].sum() for r in range(w)])
        assert per.max() - per.min() <= 2 * cost.max()
    assert list(shard_by_cost([], 4)) == [0, 0, 0, 0, 0]
    assert list(shard_by_cost([0, 0, 0], 2)) in ([0, 1, 3], [0, 2, 3], [0, 3, 3], [0, 0, 3])


def _mc_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2410_10759_b200.montecarlo import MonteCarloResult, _gather
        sids = np.arange(10)
        b = shard_bounds(len(sids), world)

        def fake(lo, hi):
            n = hi - lo
            s = np.arange(lo, hi, dtype=np.float64)
            return MonteCarloResult(sids[lo:hi], np.arange(lo, hi), s * 2.0,
                                    np.stack([s, s + 1, s + 2], 1), np.stack([s / 3, s / 5, s / 7], 1),
                                    np.zeros((n, 3), np.int32), 64 * n, 1e6 * n)
        got = _gather(fake(b[rank], b[rank + 1]), sids, b, None)
        exp = fake(0, 10)
        ok = (np.array_equal(got.table_size, exp.table_size) and np.array_equal(got.capacity, exp.capacity)
              and np.array_equal(got.max_wait_ms, exp.max_wait_ms)
              and np.array_equal(got.mean_wait_ms, exp.mean_wait_ms)
              and got.requests == exp.requests and got.dp_cells == exp.dp_cells)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_montecarlo_gather_gloo_world2():
    """Per-scenario records of a sharded Monte-Carlo sweep reassemble in scenario order."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert results == {0: True, 1: True}
