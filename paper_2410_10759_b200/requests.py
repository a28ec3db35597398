"""Request-level pipeline: (model, seq_len, devices, link, SLA) per request ->
cost table (K1) -> optimal placement (prep + K2 + K3).

This is the batched path BASELINE.json's configs exercise: every request is
one independent SplitLLM placement problem (cost_model.profile ->
problem.build_problem -> planner.plan_dp in the reference).  `RequestBatch`
holds the per-request parameters in device memory; `solve()` runs the whole
chain on one stream and leaves every result on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import batch as B
from .cost_model import encode_models

_REQ_FIELDS = ("model", "seq_len", "client_fps", "server_fps", "uplink_bps", "downlink_bps",
               "propagation_s", "deadline_s", "unit_s", "flags")
_REQ_DTYPES = dict(model=np.int32, seq_len=np.int64, flags=np.uint8)
_REQ_TORCH = {np.int32: torch.int32, np.int64: torch.int64, np.uint8: torch.uint8, np.float64: torch.float64}


def _req_layout(n: int):
    return [(f, n, _REQ_TORCH[_REQ_DTYPES.get(f, np.float64)]) for f in _REQ_FIELDS]


@dataclass
class RequestBatch:
    """Per-request scenario parameters (sp_requests), host or device tensors."""

    model: torch.Tensor
    seq_len: torch.Tensor
    client_fps: torch.Tensor
    server_fps: torch.Tensor
    uplink_bps: torch.Tensor
    downlink_bps: torch.Tensor
    propagation_s: torch.Tensor
    deadline_s: torch.Tensor
    unit_s: torch.Tensor
    flags: torch.Tensor

    @property
    def n(self) -> int:
        return int(self.model.numel())

    @classmethod
    def from_numpy(cls, pin: bool = False, **arrays) -> "RequestBatch":
        """Host batch; every field in ONE (optionally pinned) buffer, so that
        `to(device)` is a single host-to-device copy."""
        n = len(arrays["model"])
        buf, v = N.packed(_req_layout(n), "cpu", pin=pin)
        for f in _REQ_FIELDS:
            v[f].copy_(torch.from_numpy(np.ascontiguousarray(arrays[f], dtype=_REQ_DTYPES.get(f, np.float64))))
        out = cls(**v)
        out._buf = buf
        return out

    def to(self, device, non_blocking: bool = False) -> "RequestBatch":
        buf = getattr(self, "_buf", None)
        if buf is None:
            return RequestBatch(**{f: getattr(self, f).to(device, non_blocking=non_blocking)
                                   for f in _REQ_FIELDS})
        dbuf, v = N.packed(_req_layout(self.n), device)
        dbuf.copy_(buf, non_blocking=non_blocking)
        out = RequestBatch(**v)
        out._buf = dbuf
        return out

    def host_bytes(self) -> int:
        return sum(getattr(self, f).numel() * getattr(self, f).element_size() for f in _REQ_FIELDS)

    def struct(self) -> N.SpRequests:
        return N.SpRequests(self.n, *[N.ptr(getattr(self, f)).value for f in _REQ_FIELDS])


@dataclass
class Solved:
    """Device results of one `solve` call."""

    layer_off: torch.Tensor
    instances: B.InstanceBatch
    policies: B.PolicyBatch
    status: torch.Tensor       # K1 status word per request (0 ok; else the placement is not valid)
    client_s: torch.Tensor
    server_s: torch.Tensor
    up_s: torch.Tensor
    down_s: torch.Tensor


class Engine:
    """Holds the encoded model table on the device and solves request batches."""

    def __init__(self, layer_lists, device=None):
        self.device = device or N.device()
        self.models, self._keep = encode_models(layer_lists, self.device)
        self.n_layers = np.array([len(x) for x in layer_lists], dtype=np.int64)

    def layer_offsets(self, req: RequestBatch) -> torch.Tensor:
        off = torch.empty(req.n + 1, dtype=torch.int64, device=self.device)
        N.check(N.library().sp_request_layer_offsets(self.models, req.struct(), N.ptr(off),
                                                     N.stream_ptr()), "sp_request_layer_offsets")
        return off

    def cost_buffers(self, n: int, total_layers: int) -> dict:
        """The cost table's outputs for n requests / total_layers entries in
        ONE device allocation (views by name); reusable across calls."""
        T = int(total_layers)
        spec = [(k, T, torch.float64) for k in ("r", "cs", "ss", "up", "dn")]
        spec += [(k, T, torch.int64) for k in ("i", "s", "u", "d")]
        spec += [("budget", n, torch.int64), ("sac", n, torch.uint8), ("status", n, torch.int32)]
        return N.packed(spec, self.device)[1]

    def cost_table(self, req: RequestBatch, total_layers: int, off: torch.Tensor | None = None,
                   bufs: dict | None = None):
        off = self.layer_offsets(req) if off is None else off
        T = int(total_layers)
        v = bufs if bufs is not None else self.cost_buffers(req.n, T)
        f = {k: v[k] for k in ("r", "cs", "ss", "up", "dn")}
        i = {k: v[k] for k in ("i", "s", "u", "d")}
        budget, sac, status = v["budget"], v["sac"], v["status"]
        tab = N.SpCostTable(N.ptr(off).value, T, N.ptr(f["r"]).value, N.ptr(f["cs"]).value, None,
                            None, N.ptr(f["ss"]).value, N.ptr(f["up"]).value, N.ptr(f["dn"]).value,
                            N.ptr(i["i"]).value, N.ptr(i["s"]).value, N.ptr(i["u"]).value,
                            N.ptr(i["d"]).value, N.ptr(budget).value, N.ptr(sac).value,
                            N.ptr(status).value)
        N.check(N.library().sp_build_cost_table(self.models, req.struct(), 1, tab, N.stream_ptr()),
                "sp_build_cost_table")
        inst = B.InstanceBatch(off, i["i"], i["s"], i["u"], i["d"], f["r"], budget, sac)
        return inst, status, f

    def solve_slot(self, n: int, total_layers: int, ws_bytes: int) -> dict:
        """Everything one solve_async call writes -- workspace, cost table,
        policies, the device copy of host request parameters -- allocated
        once, for a pipelined caller to reuse (no allocation inside its loop)."""
        buf, v = N.packed(_req_layout(n), self.device)
        req = RequestBatch(**v)
        req._buf = buf
        return dict(ws=torch.empty(ws_bytes, dtype=torch.uint8, device=self.device),
                    cost=self.cost_buffers(n, total_layers),
                    pol=B.PolicyBatch.empty(n, int(total_layers), self.device), req=req,
                    k1_done=None, d2h_done=None)

    def copy_stream(self) -> torch.cuda.Stream:
        """The engine's stream for host <-> device copies of pipelined calls:
        a step's request upload and its results' download overlap the
        neighbouring steps' kernels."""
        if getattr(self, "_copies", None) is None:
            self._copies = torch.cuda.Stream(self.device)
        return self._copies

    def _upload(self, host_req: RequestBatch, slot: dict) -> RequestBatch:
        """Host (pinned, packed) request parameters into the slot's device
        buffer on the copy stream, once the slot's previous cost table has
        read it; the compute stream waits for the copy."""
        cs, cur = self.copy_stream(), torch.cuda.current_stream(self.device)
        dreq = slot["req"]
        if getattr(host_req, "_buf", None) is None:  # not packed: pack it (one copy still)
            host_req = RequestBatch.from_numpy(**{f: getattr(host_req, f).numpy() for f in _REQ_FIELDS})
        if slot["k1_done"] is not None:
            cs.wait_event(slot["k1_done"])
        with torch.cuda.stream(cs):
            dreq._buf.copy_(host_req._buf, non_blocking=True)
        cur.wait_stream(cs)
        return dreq

    def solve_async(self, req: RequestBatch, total_layers: int | None = None, off: torch.Tensor | None = None,
                    ws: torch.Tensor | None = None, slot: dict | None = None) -> "PendingSolve":
        """`solve` without a stream synchronisation (sp_plan_dp_async): the
        whole chain is queued and the call returns; PendingSolve.result()
        completes it.  A caller pipelines batches by queueing the next one
        before collecting this one, each in flight with its own workspace --
        or its own `slot` (solve_slot: workspace and every output reused; the
        results of a slot are valid until the slot is queued again)."""
        if total_layers is None:
            total_layers = int(self.n_layers[req.model.cpu().numpy()].sum())
        if req.model.device.type == "cpu":  # host parameters
            if slot is not None:  # uploaded on the copy stream into the slot
                req = self._upload(req, slot)
            else:
                req = req.to(self.device, non_blocking=True)
        inst, status, f = self.cost_table(req, total_layers, off, bufs=slot["cost"] if slot else None)
        if slot is not None:
            cur = torch.cuda.current_stream(self.device)
            slot["k1_done"] = torch.cuda.Event()
            slot["k1_done"].record(cur)
            if slot["d2h_done"] is not None:  # the slot's previous results have been copied out
                cur.wait_event(slot["d2h_done"])
        pend = B.plan_dp_async(inst, out=slot["pol"] if slot else None, ws=slot["ws"] if slot else ws)
        ps = PendingSolve(pend, inst, status, f, self, slot)
        if slot is not None:
            # the feasibility mask and the results' ready event are queued now,
            # right behind this batch's kernels -- not behind the next batch's,
            # which a pipelined caller queues before collecting this one
            torch.mul(pend.out.feasible, status == 0, out=pend.out.feasible)
            ps.ready = torch.cuda.Event()
            ps.ready.record(torch.cuda.current_stream(self.device))
        return ps

    def solve(self, req: RequestBatch, total_layers: int | None = None,
              off: torch.Tensor | None = None) -> Solved:
        """K1 cost table + DP placement for every request (one stream)."""
        if req.model.device.type == "cpu":  # host parameters: one copy to the device
            req = req.to(self.device)
        if total_layers is None:
            total_layers = int(self.n_layers[req.model.cpu().numpy()].sum())
        inst, status, f = self.cost_table(req, total_layers, off)
        pol = B.plan_dp(inst)
        # a request whose cost table failed (NaN / inf / negative / overflowing
        # times: the reference raises and records an error cell) is never a
        # feasible placement; its status word says why
        torch.mul(pol.feasible, status == 0, out=pol.feasible)
        return Solved(inst.layer_off, inst, pol, status, f["cs"], f["ss"], f["up"], f["dn"])


class PendingSolve:
    """An Engine.solve_async call in flight."""

    def __init__(self, pending: B.PendingPlan, inst: B.InstanceBatch, status: torch.Tensor, f: dict,
                 engine: "Engine | None" = None, slot: dict | None = None):
        self.pending, self.inst, self.status, self.f = pending, inst, status, f
        self.engine, self.slot = engine, slot
        self.ready = None  # recorded behind the batch's kernels (slot calls)

    def result(self) -> Solved:
        pol = self.pending.finish()
        if self.ready is None or self.pending.launched_more:
            # (again after the kernels finish() queued: the mask is idempotent)
            torch.mul(pol.feasible, self.status == 0, out=pol.feasible)
            if self.ready is not None:
                self.ready.record(torch.cuda.current_stream(self.engine.device))
        f = self.f
        return Solved(self.inst.layer_off, self.inst, pol, self.status, f["cs"], f["ss"], f["up"], f["dn"])

    def result_to_host(self, into: B.PolicyBatch | None = None):
        """result(), then the policies copied to pinned host memory on the
        engine's copy stream (overlapping the next step's kernels).  Returns
        (Solved, host PolicyBatch, event): read the host batch after the event."""
        s = self.result()
        eng = self.engine
        cs, cur = eng.copy_stream(), torch.cuda.current_stream(eng.device)
        ready = self.ready
        if ready is None:
            ready = torch.cuda.Event()
            ready.record(cur)
        cs.wait_event(ready)
        with torch.cuda.stream(cs):
            host = s.policies.to_host_async(into=into)
        done = torch.cuda.Event()
        done.record(cs)
        if self.slot is not None:
            self.slot["d2h_done"] = done
        return s, host, done
