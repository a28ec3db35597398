"""The one-process-per-GPU capacity-partition protocol.

CPU part (gloo, world 2 and 3): `capacity.solve_partitioned` drives a
table-based stand-in for the device operations -- each rank "owns" a column
range of the oracle's full DP tables and walks only its own columns -- so the
bookkeeping is checked without a GPU: segment agreement across ranks, the
reset / barrier / launch order of every phase, the end state from the owner
of column W_eff, the right-to-left backtrack handoff of (stage, column, side)
inside each checkpoint segment, and the combined placement, which must equal
the oracle's plan_dp (planner.py:146-202).

GPU part: the same protocol through the C ABI (sp_grid_*, CUDA IPC) with two
processes sharing the one GPU of the box.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import splitplan_oracle as O
from paper_2410_10759_b200.capacity import solve_partitioned


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _instance(seed: int, L: int, W: int, sac: bool, r_kind: str = "int"):
    rng = np.random.default_rng(seed)
    r = rng.integers(0, 100, L).astype(float) if r_kind == "int" else rng.random(L) * 50
    return dict(i=rng.integers(0, 9, L), s=rng.integers(0, 9, L), u=rng.integers(0, 9, L),
                d=rng.integers(0, 9, L), r=r, budget=W, sac=sac)


class TableOps:
    """Device operations of one rank, emulated on the oracle's full tables."""

    def __init__(self, inst, rank: int, budget_stages: int):
        self.inst = inst
        self.rank = rank
        self.budget_stages = budget_stages
        self.C, self.S = O.dp_tables(inst)
        self.log: list[str] = []
        self.info = None

    def plan(self, nparts: int, force_segment: int = 0) -> dict:
        L = len(self.inst["r"])
        ncol = O.effective_budget(self.inst) + 1
        wp = -(-ncol // nparts)
        nparts = -(-ncol // wp)
        K = min(force_segment or self.budget_stages, L)
        nseg = -(-L // K)
        self.info = dict(nparts=nparts, nseg=nseg, n_layers=L, seg_stages=K, part_cols=wp,
                         owner_part=(ncol - 1) // wp, ncol=ncol)
        self.log.append(f"plan K={K}")
        return dict(self.info)

    def plan_info(self) -> dict:
        return dict(self.info)

    def seg_begin(self, sg: int) -> int:
        L, K, nseg = self.info["n_layers"], self.info["seg_stages"], self.info["nseg"]
        return 0 if sg == 0 else L - (nseg - sg) * K

    def alloc(self):
        self.log.append("alloc")

    def export(self):
        return (f"handle{self.rank}".encode(), self.rank)

    def map_peers(self, handles):
        assert [h[1] for h in handles] == list(range(len(handles)))
        self.log.append(f"map {len(handles)}")

    def prepare(self):
        self.log.append("prepare")

    def reset(self):
        self.log.append("reset")

    def sync(self):
        pass

    def forward(self, seg, write_ckpt, keep_bp):
        assert self.log[-1] == "reset", self.log[-3:]
        self.log.append(f"fwd {seg} {int(write_ckpt)} {int(keep_bp)}")

    def close(self):
        self.log.append("close")

    def end(self, must):
        assert self.rank == self.info["owner_part"]
        ec, es = self.C[-1, -1], self.S[-1, -1]
        if must == 1:
            es = O.NEG
        elif must == 0:
            ec = O.NEG
        flag = 1 if max(ec, es) == O.NEG else 0
        return np.array([self.info["ncol"] - 1, int(ec >= es), flag, self.info["n_layers"] - 1], dtype=np.int64)

    def backtrack(self, seg, state, pi):
        """planner.py:146-179 over this rank's columns and this segment's stages."""
        j, client, flag, k = (int(x) for x in state)
        pi = pi.copy()
        if flag:
            return state, pi
        k0 = self.seg_begin(seg)
        p0 = self.rank * self.info["part_cols"]
        # a partition right of the column was never skipped while stages of this segment remain
        assert k < k0 or j < p0 + self.info["part_cols"], (j, p0, k, k0)
        x = self.inst
        while k >= k0 and j >= p0:
            ik, sk, uk, dk, rk = int(x["i"][k]), int(x["s"][k]), int(x["u"][k]), int(x["d"][k]), x["r"][k]
            if client:
                pi[k] = 1
                if j >= ik and self.C[k, j - ik] + rk == self.C[k + 1, j]:
                    j -= ik
                elif j >= ik + dk and self.S[k, j - ik - dk] + rk == self.C[k + 1, j]:
                    j, client = j - ik - dk, 0
                else:
                    return np.array([j, client, 2, k], dtype=np.int64), pi
            else:
                pi[k] = 0
                if j >= sk and self.S[k, j - sk] == self.S[k + 1, j]:
                    j -= sk
                elif j >= sk + uk and self.C[k, j - sk - uk] == self.S[k + 1, j]:
                    j, client = j - sk - uk, 1
                else:
                    return np.array([j, client, 2, k], dtype=np.int64), pi
            k -= 1
        self.log.append(f"bt {seg} handoff k={k}")
        return np.array([j, client, 0, k], dtype=np.int64), pi


def _worker(rank, world, port, cases, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for seed, L, W, sac, must, stages in cases:
            inst = _instance(seed, L, W, sac)
            # every rank proposes a different segment length: the protocol takes the shortest
            ops = TableOps(inst, rank, stages + 3 * rank)
            res = solve_partitioned(ops, None, {None: -1, "server": 0, "client": 1}[must])
            exp = O.plan_dp(inst, must)
            assert tuple(int(v) for v in res.pi) == exp["pi"], (seed, res.pi, exp["pi"])
            assert ops.info["seg_stages"] == min(stages, L)
            assert res.nseg == -(-L // min(stages, L))
            fwd = [e for e in ops.log if e.startswith("fwd")]
            if rank < res.nparts:
                # forward segments in order, then recomputes from the second-last down
                n = res.nseg
                assert fwd[:n] == [f"fwd {s} 1 {int(s == n - 1)}" for s in range(n)]
                assert fwd[n:] == [f"fwd {s} 0 1" for s in range(n - 2, -1, -1)]
            else:
                assert fwd == []
        q.put((rank, "ok"))
    except Exception as exc:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partition_protocol_handoff_matches_oracle(world):
    # (seed, L, W, source_at_client, must_end_at, segment stages)
    cases = [(1, 40, 60, True, None, 7), (2, 25, 90, False, None, 100), (3, 60, 45, True, "server", 13),
             (4, 30, 200, False, "client", 1), (5, 50, 3, True, None, 9), (6, 35, 0, True, None, 4),
             (7, 20, 150, True, None, 6)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res


# ---------------------------------------------------------------------------
# GPU: the C-ABI partition operations, two processes on the one GPU

def _gpu_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        torch.cuda.set_device(0)
        from paper_2410_10759_b200 import batch as B
        from paper_2410_10759_b200.capacity import plan_dp_partitioned
        rng = np.random.default_rng(11)
        for t, (L, W) in enumerate(((48, 40_000), (32, 9_000), (24, 60_000))):
            inst = dict(i=rng.integers(0, 400, L), s=rng.integers(0, 400, L), u=rng.integers(0, 400, L),
                        d=rng.integers(0, 400, L),
                        r=(rng.integers(0, 1000, L).astype(float) if t != 1 else rng.random(L) * 100),
                        budget=W, sac=bool(t % 2 == 0))
            b = B.InstanceBatch.from_arrays([0, L], inst["i"], inst["s"], inst["u"], inst["d"], inst["r"],
                                            [W], [int(inst["sac"])])
            # two CTAs per partition (both processes time-share the GPU), a
            # workspace small enough to force checkpoint segments
            pol = plan_dp_partitioned(b, ctas_per_part=2, part_ws_bytes=(6 << 20) if t == 0 else None)
            got = pol.to_host()
            exp = O.plan_dp(inst)
            assert tuple(int(v) for v in got["pi"]) == exp["pi"], t
            assert got["client_value"][0] == exp["client_value"] and got["server_load"][0] == exp["server_load"]
            assert got["integer_latency"][0] == exp["integer_latency"] and bool(got["feasible"][0]) == exp["feasible"]
        q.put((rank, "ok"))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_partitioned_processes_on_one_gpu(gpu):
    """Two ranks, one partition each, mapped into each other through CUDA IPC
    (both on the box's one GPU): bit-exact placements vs the oracle."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res
