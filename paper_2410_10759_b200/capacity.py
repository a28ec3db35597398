"""One huge instance, capacity axis split over ranks: one process per GPU.

SURVEY.md 8(e), cfg5: a single placement chain too wide for one GPU
(L = 1e5 stages x W = 1e7 budget columns) has its budget axis cut into one
contiguous column range per rank.  Because every DP shift goes right
(planner.py:110-117), partition p reads only its own columns and the last
`halo` columns of partition p-1, so:

* each rank keeps its partition's rows, checkpoint rows and back-pointers in
  ONE workspace on its own GPU (sp_grid_plan.part_bytes);
* every rank maps every other rank's workspace through CUDA IPC
  (`sp_ipc_export` / `sp_ipc_import`, handles exchanged over the process
  group), so the DP kernel stores its last columns straight into the right
  neighbour's halo (NVLink peer stores) and polls its neighbours' progress
  counters (system-scope acquire / release) -- no NCCL on the data path;
* the backtrack (planner.py:146-179) runs rank by rank from the right, each
  rank walking its own back-pointers while the column stays in its range and
  handing (stage, column, side) to its left neighbour;
* the placement is combined with one all-reduce (every stage is written by
  exactly one rank) and evaluated (`_finish`, planner.py:88-101).

`solve_partitioned(ops, group)` is the protocol; `NativePartition` the
device operations through the C ABI.  The protocol only talks to `ops`, so
the CPU tests drive it with a table-based stand-in under gloo.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N
from . import batch as B

STATE_OK, STATE_INFEASIBLE, STATE_BACKTRACE_ERROR = 0, 1, 2


@dataclass
class PartitionedResult:
    pi: np.ndarray          # uint8 [L]
    state: np.ndarray       # int64 [4]: final {column, side, flag, next stage}
    nparts: int
    nseg: int


def _comm_device(group) -> torch.device:
    backend = dist.get_backend(group)
    return torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")


def _broadcast_state(state: np.ndarray, src: int, group) -> np.ndarray:
    t = torch.as_tensor(np.asarray(state, dtype=np.int64)).to(_comm_device(group))
    dist.broadcast(t, src=dist.get_global_rank(group, src) if group is not None else src, group=group)
    return t.cpu().numpy()


def _barrier(ops, group) -> None:
    ops.sync()
    dist.barrier(group=group)


def agree_segment(ops, world: int, group) -> None:
    """Every rank plans for its own workspace budget; all take the shortest
    segment (the one the tightest rank can hold) so the phases line up."""
    plan = ops.plan(world)
    t = torch.tensor([plan["seg_stages"]], dtype=torch.int64, device=_comm_device(group))
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    k = int(t.item())
    if k != plan["seg_stages"]:
        ops.plan(world, force_segment=k)


def solve_partitioned(ops, group=None, must_end_at: int = -1) -> PartitionedResult:
    """Run the partitioned DP + backtrack on every rank of `group` (collective).

    Ranks beyond the plan's partition count (a chain with fewer columns than
    ranks, or one whose stage shifts span a whole partition) stay idle but
    take part in every collective."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    ops.rank = rank  # partition index = rank in the group
    agree_segment(ops, world, group)
    plan = ops.plan_info()
    nparts, nseg, L = plan["nparts"], plan["nseg"], plan["n_layers"]
    mine = rank < nparts
    # map every partition workspace into every participating process
    ops.alloc()
    handles = [None] * world
    dist.all_gather_object(handles, ops.export() if mine else None, group=group)
    ops.map_peers(handles[:nparts])
    if mine:
        ops.prepare()

    def phase(seg: int, write_ckpt: bool, keep_bp: bool) -> None:
        if mine:
            ops.reset()
        _barrier(ops, group)  # every partition's counters are zero before any partition starts
        if mine:
            ops.forward(seg, write_ckpt, keep_bp)
        _barrier(ops, group)  # the phase is complete everywhere

    for seg in range(nseg):  # forward pass: checkpoints, last segment's back-pointers
        phase(seg, True, seg == nseg - 1)
    owner = plan["owner_part"]
    state = ops.end(must_end_at) if rank == owner else np.zeros(4, dtype=np.int64)
    state = _broadcast_state(state, owner, group)
    pi = np.zeros(L, dtype=np.uint8)
    for seg in range(nseg - 1, -1, -1):
        if seg < nseg - 1:  # recompute this segment's back-pointers from its checkpoint
            phase(seg, False, True)
        for p in range(nparts - 1, -1, -1):  # right to left: the column never grows
            if rank == p:
                state, pi = ops.backtrack(seg, state, pi)
            state = _broadcast_state(state, p, group)
    # every stage was decided by exactly one rank
    t = torch.as_tensor(pi.astype(np.int32)).to(_comm_device(group))
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    pi = t.cpu().numpy().astype(np.uint8)
    if state[2] == STATE_INFEASIBLE:
        pi[:] = 0
    ops.close()
    return PartitionedResult(pi=pi, state=state, nparts=nparts, nseg=nseg)


class NativePartition:
    """Device side of one rank: the partition workspace on this rank's GPU and
    the peers' workspaces mapped through CUDA IPC (sp_grid_* in the C ABI)."""

    def __init__(self, batch: B.InstanceBatch, part_ws_bytes: int | None = None, ctas_per_part: int = 0):
        if batch.n != 1:
            raise ValueError("one instance per partitioned solve")
        self.batch = batch
        self.ctas = int(ctas_per_part)
        self.budget = part_ws_bytes
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self._plan = None
        self._peers: list[int] = []
        self._bases: list[int] = []
        self.ws = None
        self.lib = N.library()

    # -- planning -----------------------------------------------------------
    def plan(self, nparts: int, force_segment: int = 0) -> dict:
        if self.budget is None:
            self.budget = int(N.free_bytes(N.device()) * 0.8)
        p = N.SpGridPlan()
        s = self.batch.struct()
        rc = N.with_workspace(lambda ws, nb: self.lib.sp_grid_plan_make(
            s, int(nparts), self.ctas, C.c_size_t(int(self.budget)), int(force_segment), C.byref(p), ws, nb,
            N.stream_ptr()))
        N.check(rc, "sp_grid_plan_make")
        self._plan = p
        return self.plan_info()

    def plan_info(self) -> dict:
        return {f: int(getattr(self._plan, f)) for f, _ in N.SpGridPlan._fields_}

    # -- workspaces -----------------------------------------------------------
    def alloc(self) -> None:
        self.ws = torch.empty(int(self._plan.part_bytes), dtype=torch.uint8, device=N.device())

    def export(self):
        handle = (C.c_ubyte * 64)()
        off = C.c_size_t(0)
        N.check(self.lib.sp_ipc_export(N.ptr(self.ws), C.cast(handle, C.c_void_p), C.byref(off)), "sp_ipc_export")
        return bytes(handle), int(off.value)

    def map_peers(self, handles) -> None:
        me = self.rank
        self._peers = []
        for r, h in enumerate(handles):
            if r == me:
                self._peers.append(self.ws.data_ptr())
                continue
            buf = (C.c_ubyte * 64).from_buffer_copy(h[0])
            dptr, base = C.c_void_p(0), C.c_void_p(0)
            N.check(self.lib.sp_ipc_import(C.cast(buf, C.c_void_p), C.c_size_t(h[1]), C.byref(dptr), C.byref(base)),
                    "sp_ipc_import")
            self._peers.append(int(dptr.value))
            self._bases.append(int(base.value))

    def close(self) -> None:
        torch.cuda.synchronize()
        for b in self._bases:
            self.lib.sp_ipc_close(C.c_void_p(b))
        self._bases = []

    # -- phases ---------------------------------------------------------------
    def sync(self) -> None:
        torch.cuda.synchronize()

    def prepare(self) -> None:
        N.check(self.lib.sp_grid_part_prepare(C.byref(self._plan), self.batch.struct(), N.ptr(self.ws),
                                              N.stream_ptr()), "sp_grid_part_prepare")

    def reset(self) -> None:
        N.check(self.lib.sp_grid_part_reset(C.byref(self._plan), N.ptr(self.ws), N.stream_ptr()),
                "sp_grid_part_reset")

    def forward(self, seg: int, write_ckpt: bool, keep_bp: bool) -> None:
        arr = (C.c_void_p * len(self._peers))(*self._peers)
        N.check(self.lib.sp_grid_part_forward(C.byref(self._plan), self.rank, C.cast(arr, C.c_void_p), seg,
                                              int(write_ckpt), int(keep_bp), N.stream_ptr()),
                "sp_grid_part_forward")

    def end(self, must_end_at: int) -> np.ndarray:
        st = torch.zeros(4, dtype=torch.int64, device=N.device())
        N.check(self.lib.sp_grid_part_end(C.byref(self._plan), N.ptr(self.ws), int(must_end_at), N.ptr(st),
                                          N.stream_ptr()), "sp_grid_part_end")
        return st.cpu().numpy()

    def backtrack(self, seg: int, state: np.ndarray, pi: np.ndarray):
        st = torch.as_tensor(np.asarray(state, dtype=np.int64)).to(N.device())
        p = torch.as_tensor(pi).to(N.device())
        N.check(self.lib.sp_grid_part_backtrack(C.byref(self._plan), self.rank, N.ptr(self.ws), seg, N.ptr(st),
                                                N.ptr(p), N.stream_ptr()), "sp_grid_part_backtrack")
        return st.cpu().numpy(), p.cpu().numpy()


def plan_dp_partitioned(batch: B.InstanceBatch, group=None, must_end_at: str | None = None,
                        part_ws_bytes: int | None = None, ctas_per_part: int = 0) -> B.PolicyBatch:
    """planner.plan_dp of ONE instance with its capacity axis split over the
    ranks of `group` (collective; every rank passes the same instance and
    gets the same PolicyBatch on its own device)."""
    must = {None: -1, "server": 0, "client": 1}[must_end_at]
    ops = NativePartition(batch, part_ws_bytes, ctas_per_part)
    res = solve_partitioned(ops, group, must)
    out = B.PolicyBatch.empty(1, batch.total_layers, batch.r.device)
    if res.state[2] == STATE_BACKTRACE_ERROR:
        out.status.fill_(N.SP_ERR_BACKTRACE)
        return out
    pi = torch.as_tensor(res.pi).to(batch.r.device)
    ws = N.workspace(4 * batch.total_layers)
    N.check(N.library().sp_evaluate_policy(batch.struct(), N.ptr(pi), out.struct(), N.ptr(ws), ws.numel(),
                                           N.stream_ptr()), "sp_evaluate_policy")
    out.pi.copy_(pi)
    if res.state[2] == STATE_INFEASIBLE:
        out.feasible.zero_()
    return out
