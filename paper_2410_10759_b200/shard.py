"""Multi-GPU sharding of independent placement units (one process per GPU).

Every request and every sweep scenario is an independent placement problem
(`evaluator.py:214-226` solves them in a plain loop), so the
data path needs no collective at all: rank r solves a contiguous shard of the
units on its own GPU.  The only communication is ONE gather of fixed-size
result records at the end (`gather_policies`), over NCCL between GPUs (or
gloo in the CPU tests).

    shard_bounds(n, world)            contiguous equal-count shards
    shard_by_cost(cost, world)        contiguous shards of ~equal DP cells
    gather_policies(pol, off, group)  all ranks' PolicyBatch -> the job's results
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .batch import PolicyBatch


def shard_bounds(n: int, world: int) -> np.ndarray:
    """Offsets [world+1] of contiguous shards whose sizes differ by at most one."""
    if world < 1:
        raise ValueError("world must be >= 1")
    base, extra = divmod(int(n), world)
    sizes = np.full(world, base, dtype=np.int64)
    sizes[:extra] += 1
    off = np.zeros(world + 1, dtype=np.int64)
    np.cumsum(sizes, out=off[1:])
    return off


def shard_by_cost(cost, world: int) -> np.ndarray:
    """Offsets [world+1] of contiguous shards of roughly equal total cost.

    `cost[k]` is the work of unit k (DP cells: L_k x (W_eff_k + 1)).  Shard r
    ends at the first unit whose inclusive prefix cost reaches (r+1)/world of
    the total, so the order of units (and thus of the gathered results) is
    preserved."""
    if world < 1:
        raise ValueError("world must be >= 1")
    c = np.asarray(cost, dtype=np.float64)
    n = c.size
    off = np.zeros(world + 1, dtype=np.int64)
    off[world] = n
    if n == 0:
        return off
    pre = np.cumsum(c)
    total = pre[-1]
    for r in range(1, world):
        off[r] = np.searchsorted(pre, total * r / world, side="left") + 1 if total > 0 else n * r // world
        off[r] = min(max(off[r], off[r - 1]), n)
    return off


def _pack_records(pol: PolicyBatch) -> torch.Tensor:
    """Fixed-size per-unit records as int64 [n, 4]: value bits, load bits,
    integer latency, feasible | status << 8."""
    n = pol.client_value.numel()
    rec = torch.empty((n, 4), dtype=torch.int64, device=pol.client_value.device)
    rec[:, 0] = pol.client_value.view(torch.int64)
    rec[:, 1] = pol.server_load.view(torch.int64)
    rec[:, 2] = pol.integer_latency
    rec[:, 3] = pol.feasible.to(torch.int64) | (pol.status.to(torch.int64) << 8)
    return rec


def _all_gather_padded(t: torch.Tensor, rows: list[int], group) -> list[torch.Tensor]:
    """all_gather of tensors whose first dimension differs per rank."""
    width = max(rows)
    pad = torch.zeros((width,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    bufs = [torch.empty_like(pad) for _ in rows]
    dist.all_gather(bufs, pad, group=group)
    return [b[:r] for b, r in zip(bufs, rows)]


def gather_policies(pol: PolicyBatch, layer_off: torch.Tensor, group=None) -> tuple[PolicyBatch, torch.Tensor]:
    """Assemble every rank's results, in rank order, on every rank.

    `pol` and `layer_off` ([n+1], local CSR over layers) describe this rank's
    shard.  Returns the concatenated PolicyBatch and the global layer
    offsets.  Three collectives: the shard sizes, the per-unit records, and
    the placement bytes."""
    world = dist.get_world_size(group)
    dev = pol.client_value.device
    n_local = pol.client_value.numel()
    t_local = pol.pi.numel()
    sizes = torch.tensor([n_local, t_local], dtype=torch.int64, device=dev)
    all_sizes = [torch.empty_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=group)
    ns = [int(s[0]) for s in all_sizes]
    ts = [int(s[1]) for s in all_sizes]

    recs = _all_gather_padded(_pack_records(pol), ns, group)
    lens = (layer_off[1:] - layer_off[:-1]).to(torch.int64)
    lens_all = _all_gather_padded(lens, ns, group)
    pis = _all_gather_padded(pol.pi, ts, group)

    rec = torch.cat(recs)
    out = PolicyBatch(torch.cat(pis), rec[:, 0].contiguous().view(torch.float64),
                      rec[:, 1].contiguous().view(torch.float64), rec[:, 2].contiguous(),
                      (rec[:, 3] & 0xFF).to(torch.uint8), (rec[:, 3] >> 8).to(torch.int32))
    off = torch.zeros(sum(ns) + 1, dtype=torch.int64, device=dev)
    torch.cumsum(torch.cat(lens_all), 0, out=off[1:])
    return out, off
