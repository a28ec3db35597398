"""Batched device API: many independent placement instances per call.

`InstanceBatch` is the CSR form of a list of `PlanProblem`s (the C ABI's
`sp_instances`) held in CUDA tensors; `PolicyBatch` the matching
`sp_policies`.  The reference-compatible functions in `planner.py` wrap these
with n == 1; sweeps and benches call them directly with thousands of
instances.
"""

from __future__ import annotations

from dataclasses import dataclass

import ctypes as C

import numpy as np
import torch

from . import _native as N


@dataclass
class InstanceBatch:
    layer_off: torch.Tensor      # int64 [n+1]
    client_units: torch.Tensor   # int64 [T]
    server_units: torch.Tensor
    up_units: torch.Tensor
    down_units: torch.Tensor
    r: torch.Tensor              # float64 [T]
    budget: torch.Tensor         # int64 [n]
    source_at_client: torch.Tensor  # uint8 [n]
    must_end_at: torch.Tensor | None = None  # int8 [n]
    n_layers_host: np.ndarray | None = None  # int64 [n] (host copy of lengths, optional)

    @property
    def n(self) -> int:
        return int(self.budget.numel())

    @property
    def total_layers(self) -> int:
        return int(self.r.numel())

    def struct(self) -> N.SpInstances:
        return N.SpInstances(self.n, self.total_layers, N.ptr(self.layer_off).value,
                             N.ptr(self.client_units).value, N.ptr(self.server_units).value,
                             N.ptr(self.up_units).value, N.ptr(self.down_units).value,
                             N.ptr(self.r).value, N.ptr(self.budget).value,
                             N.ptr(self.source_at_client).value,
                             N.ptr(self.must_end_at).value if self.must_end_at is not None else None)

    @classmethod
    def from_arrays(cls, layer_off, i, s, u, d, r, budget, sac, must=None) -> "InstanceBatch":
        """Host arrays -> one device allocation, one host-to-device copy."""
        dev = N.device()
        lo = np.asarray(layer_off, dtype=np.int64)
        n, T = lo.size - 1, int(lo[-1]) if lo.size else 0
        spec = [("layer_off", n + 1, torch.int64)] + [(k, T, torch.int64) for k in ("i", "s", "u", "d")]
        spec += [("r", T, torch.float64), ("budget", n, torch.int64), ("sac", n, torch.uint8)]
        arrays = dict(layer_off=lo, i=np.asarray(i, np.int64), s=np.asarray(s, np.int64),
                      u=np.asarray(u, np.int64), d=np.asarray(d, np.int64), r=np.asarray(r, np.float64),
                      budget=np.asarray(budget, np.int64), sac=np.asarray(sac, np.uint8))
        if must is not None:
            spec.append(("must", n, torch.int8))
            arrays["must"] = np.asarray(must, np.int8)
        for name, numel, _dt in spec:
            if np.size(arrays[name]) != numel:
                raise ValueError(f"{name}: {np.size(arrays[name])} values, expected {numel}")
        v = N.packed_upload(spec, arrays, dev)
        out = cls(v["layer_off"], v["i"], v["s"], v["u"], v["d"], v["r"], v["budget"], v["sac"],
                  v.get("must"), np.diff(lo))
        out._buf = v["_buf"]
        return out

    @classmethod
    def from_problems(cls, problems, must_end_at=None) -> "InstanceBatch":
        lens = np.array([p.n_layers for p in problems], dtype=np.int64)
        off = np.zeros(len(problems) + 1, dtype=np.int64)
        np.cumsum(lens, out=off[1:])
        cat = lambda name, dt: (np.concatenate([np.asarray(getattr(p, name), dtype=dt) for p in problems])
                                if problems else np.zeros(0, dt))
        must = None
        if must_end_at is not None:
            must = np.array([-1 if m is None else (1 if m == "client" else 0) for m in must_end_at],
                            dtype=np.int8)
        return cls.from_arrays(off, cat("client_units", np.int64), cat("server_units", np.int64),
                               cat("up_units", np.int64), cat("down_units", np.int64),
                               cat("r", np.float64),
                               np.array([p.budget for p in problems], dtype=np.int64),
                               np.array([p.source_at_client for p in problems], dtype=np.uint8),
                               must)


def _POLICY_LAYOUT(n: int, total: int):
    # pi and status first: the two arrays zeroed up front
    return [("pi", total, torch.uint8), ("status", n, torch.int32), ("client_value", n, torch.float64),
            ("server_load", n, torch.float64), ("integer_latency", n, torch.int64), ("feasible", n, torch.uint8)]


@dataclass
class PolicyBatch:
    pi: torch.Tensor               # uint8 [T]
    client_value: torch.Tensor     # float64 [n]
    server_load: torch.Tensor      # float64 [n]
    integer_latency: torch.Tensor  # int64 [n]
    feasible: torch.Tensor         # uint8 [n]
    status: torch.Tensor           # int32 [n]

    @classmethod
    def empty(cls, n: int, total: int, dev=None) -> "PolicyBatch":
        """One device allocation, zeroed with one fill (pi and status must
        start at zero; the alignment gaps are zeroed too, so the one-copy
        to_host reads no uninitialised bytes)."""
        dev = dev or N.device()
        buf, v = N.packed(_POLICY_LAYOUT(n, total), dev, zero_prefix=len(_POLICY_LAYOUT(0, 0)))
        out = cls(v["pi"], v["client_value"], v["server_load"], v["integer_latency"], v["feasible"],
                  v["status"])
        out._buf = buf
        return out

    def to_host_async(self, into: "PolicyBatch | None" = None) -> "PolicyBatch":
        """The results in pinned host memory: ONE device-to-host copy when the
        batch owns a packed buffer (PolicyBatch.empty), stream-ordered; read
        them after the stream (or the copy) has completed.  `into`: a host
        batch of the same shape from an earlier call, reused (a caller
        streaming many batches keeps a few and avoids pinned allocations)."""
        buf = getattr(self, "_buf", None)
        n, total = self.client_value.numel(), self.pi.numel()
        if into is not None and getattr(into, "_buf", None) is not None and into.pi.numel() == total \
                and into.client_value.numel() == n:
            hbuf = into._buf
            v = {k: getattr(into, k) for k in ("pi", "client_value", "server_load", "integer_latency",
                                               "feasible", "status")}
        else:
            hbuf, v = N.packed(_POLICY_LAYOUT(n, total), "cpu", pin=True)
        if buf is not None and buf.numel() == hbuf.numel():
            hbuf.copy_(buf, non_blocking=True)
        else:
            for k in v:
                v[k].copy_(getattr(self, k), non_blocking=True)
        out = PolicyBatch(v["pi"], v["client_value"], v["server_load"], v["integer_latency"], v["feasible"],
                          v["status"])
        out._buf = hbuf
        return out

    def nbytes(self) -> int:
        return sum(getattr(self, k).numel() * getattr(self, k).element_size()
                   for k in ("pi", "client_value", "server_load", "integer_latency", "feasible", "status"))

    def struct(self) -> N.SpPolicies:
        return N.SpPolicies(N.ptr(self.pi).value, N.ptr(self.client_value).value,
                            N.ptr(self.server_load).value, N.ptr(self.integer_latency).value,
                            N.ptr(self.feasible).value, N.ptr(self.status).value)

    def to_host(self) -> dict:
        buf = getattr(self, "_buf", None)
        if buf is not None and buf.device.type != "cpu":  # one device-to-host copy
            hbuf = buf.cpu()
            base = buf.data_ptr()
            view = lambda t: hbuf[t.data_ptr() - base: t.data_ptr() - base + t.numel() * t.element_size()] \
                .view(t.dtype).numpy()
            return dict(pi=view(self.pi), client_value=view(self.client_value), server_load=view(self.server_load),
                        integer_latency=view(self.integer_latency), feasible=view(self.feasible).astype(bool),
                        status=view(self.status))
        return dict(pi=self.pi.cpu().numpy(), client_value=self.client_value.cpu().numpy(),
                    server_load=self.server_load.cpu().numpy(),
                    integer_latency=self.integer_latency.cpu().numpy(),
                    feasible=self.feasible.cpu().numpy().astype(bool),
                    status=self.status.cpu().numpy())


# ---------------------------------------------------------------------------
# planners


def effective_budget(batch: InstanceBatch) -> torch.Tensor:
    out = torch.empty(batch.n, dtype=torch.int64, device=batch.r.device)
    s = batch.struct()
    N.check(N.library().sp_effective_budget(s, N.ptr(out), N.stream_ptr()), "sp_effective_budget")
    return out


def plan_dp(batch: InstanceBatch, out: PolicyBatch | None = None, devices=None) -> PolicyBatch:
    """K1-prep + K2 DP stage + K3 backtrack over the whole batch (sp_plan_dp).

    `devices` (a list of CUDA device indices, the current one first) splits
    the capacity axis of huge instances over those devices
    (sp_plan_dp_devices), one partition workspace per listed device."""
    out = out or PolicyBatch.empty(batch.n, batch.total_layers, batch.r.device)
    s, o = batch.struct(), out.struct()
    lib = N.library()
    if devices:
        parts = partition_workspaces(batch, devices)
        arr = (C.c_int32 * len(devices))(*[int(d) for d in devices])
        wptr = (C.c_void_p * len(devices))(*[t.data_ptr() for t in parts])
        wlen = (C.c_size_t * len(devices))(*[t.numel() for t in parts])
        rc = N.with_workspace(lambda ws, nb: lib.sp_plan_dp_devices(
            s, o, C.cast(arr, C.c_void_p), len(devices), ws, nb, C.cast(wptr, C.c_void_p),
            C.cast(wlen, C.c_void_p), N.stream_ptr()))
        N.check(rc, "sp_plan_dp_devices")
        return out
    # grow the cached workspace ahead of the call to what runs the
    # device-planned tier in one wave (host arithmetic; within the cap and the
    # free memory), instead of many small waves in a first call
    N.grow_workspace_hint(int(lib.sp_plan_dp_onewave_bytes(batch.n, batch.total_layers)))
    ws = N.workspace()
    rc = lib.sp_plan_dp(s, o, N.ptr(ws), ws.numel(), N.stream_ptr())
    if rc == N.SP_ERR_WORKSPACE:
        # size it from the query (prep only, no DP): the useful size at once,
        # instead of running the batch in waves of a minimal workspace
        del ws
        mn, full = dp_workspace_bytes(batch)
        N.workspace(N.useful_size(mn, full))
        rc = N.with_workspace(lambda w, nb: lib.sp_plan_dp(s, o, w, nb, N.stream_ptr()))
    else:
        del ws
    N.check(rc, "sp_plan_dp")
    N.grow_workspace_hint(int(lib.sp_last_full_workspace()))
    return out


class PendingPlan:
    """An sp_plan_dp_async call in flight: `finish()` waits for its
    device-planned tier (not for the whole stream), runs the host-planned
    tiers for what it left and returns the policies.  The workspace must not
    be reused before finish()."""

    def __init__(self, batch, out, ws, pend, s, o, done: bool):
        self.batch, self.out, self.ws, self.pend, self.s, self.o = batch, out, ws, pend, s, o
        self.done = done
        self.launched_more = False  # finish() queued kernels (instances the device-planned tier left)

    def finish(self) -> PolicyBatch:
        if not self.done:
            rc = N.library().sp_plan_dp_finish(self.s, self.o, N.ptr(self.ws), self.ws.numel(), N.stream_ptr(),
                                               N.ptr(self.pend))
            self.done = True
            # the record's first word: instances the device-planned tier solved
            self.launched_more = int(self.pend[:8].view(torch.int64)[0]) < self.batch.n
            _PEND_FREE.append(self.pend)  # its record is consumed: reusable
            N.check(rc, "sp_plan_dp_finish")
        return self.out


# pinned pending records of sp_plan_dp_async, reused: a pinned allocation
# inside a pipelined loop can stall the host for milliseconds (page pinning)
_PEND_FREE: list = []


def _pending_record() -> torch.Tensor:
    return _PEND_FREE.pop() if _PEND_FREE else torch.empty(N.SP_PENDING_BYTES, dtype=torch.uint8, pin_memory=True)


def _host_packed(specs, arrays: dict | None = None):
    """One host (numpy) buffer holding typed arrays at 256-B aligned offsets:
    (buffer, {name: numpy view}); `arrays` fills them."""
    offs, o = [], 0
    for _name, numel, dt in specs:
        o = (o + 255) & ~255
        offs.append(o)
        o += int(numel) * dt.itemsize
    h = np.zeros(max(o, 1), dtype=np.uint8)
    views = {name: h[off:off + int(numel) * dt.itemsize].view(N._NP_OF[dt])
             for (name, numel, dt), off in zip(specs, offs)}
    if arrays:
        for name, v in views.items():
            v[:] = arrays[name]
    return h, views


def plan_dp_host(layer_off, i, s, u, d, r, budget, sac, must=None, prefix: int | None = None) -> dict:
    """plan_dp (or, with `prefix` = SP_GREEDY / SP_ALL_SERVER / SP_ALL_CLIENT,
    plan_prefix) of a few host instances in one library call
    (sp_plan_dp_host / sp_plan_prefix_host): the instances packed into one
    host buffer go in with one copy, the policies come back with one copy --
    the scalar drop-in's path.  Returns the host results (to_host's dict)."""
    lo = np.asarray(layer_off, dtype=np.int64)
    n, T = lo.size - 1, int(lo[-1]) if lo.size else 0
    spec = [("layer_off", n + 1, torch.int64)] + [(k, T, torch.int64) for k in ("i", "s", "u", "d")]
    spec += [("r", T, torch.float64), ("budget", n, torch.int64), ("sac", n, torch.uint8)]
    arrays = dict(layer_off=lo, i=i, s=s, u=u, d=d, r=r, budget=budget, sac=sac)
    if must is not None:
        spec.append(("must", n, torch.int8))
        arrays["must"] = must
    hin, v = _host_packed(spec, arrays)
    hout, o = _host_packed(_POLICY_LAYOUT(n, T))
    addr = lambda a: a.ctypes.data
    ins = N.SpInstances(n, T, *[addr(v[k]) for k in ("layer_off", "i", "s", "u", "d", "r", "budget", "sac")],
                        addr(v["must"]) if must is not None else None)
    outs = N.SpPolicies(addr(o["pi"]), addr(o["client_value"]), addr(o["server_load"]),
                        addr(o["integer_latency"]), addr(o["feasible"]), addr(o["status"]))
    lib = N.library()
    if prefix is None:
        rc = N.with_workspace(lambda ws, nb: lib.sp_plan_dp_host(ins, outs, ws, nb, N.stream_ptr()))
    else:
        rc = N.with_workspace(lambda ws, nb: lib.sp_plan_prefix_host(ins, prefix, outs, ws, nb, N.stream_ptr()))
    N.check(rc, "sp_plan_dp_host" if prefix is None else "sp_plan_prefix_host")
    return dict(pi=o["pi"], client_value=o["client_value"], server_load=o["server_load"],
                integer_latency=o["integer_latency"], feasible=o["feasible"].astype(bool), status=o["status"])


def plan_dp_async(batch: InstanceBatch, out: PolicyBatch | None = None,
                  ws: torch.Tensor | None = None) -> PendingPlan:
    """plan_dp without a stream synchronisation: the batch's device-planned
    tier is queued and the call returns (sp_plan_dp_async); PendingPlan.finish()
    completes it.  `ws`: this call's workspace (distinct per call in flight),
    else the shared cached one.  Falls back to plan_dp when the tier cannot
    take the batch in `ws`."""
    out = out or PolicyBatch.empty(batch.n, batch.total_layers, batch.r.device)
    ws = N.workspace() if ws is None else ws
    pend = _pending_record()
    s, o = batch.struct(), out.struct()
    rc = N.library().sp_plan_dp_async(s, o, N.ptr(ws), ws.numel(), N.stream_ptr(), N.ptr(pend))
    if rc == N.SP_ERR_WORKSPACE:
        _PEND_FREE.append(pend)
        plan_dp(batch, out)
        return PendingPlan(batch, out, ws, _pending_record(), s, o, True)
    N.check(rc, "sp_plan_dp_async")
    return PendingPlan(batch, out, ws, pend, s, o, False)


def partition_workspaces(batch: InstanceBatch, devices) -> list[torch.Tensor]:
    """One workspace per capacity partition, each on its device: the size that
    keeps every back-pointer stage if it fits the device, else the minimum
    (checkpoint / recompute) -- sp_plan_dp_devices_workspace_bytes."""
    s = batch.struct()
    arr = (C.c_int32 * len(devices))(*[int(d) for d in devices])
    ws_min, pmin, pfull = C.c_size_t(0), C.c_size_t(0), C.c_size_t(0)
    rc = N.with_workspace(lambda ws, nb: N.library().sp_plan_dp_devices_workspace_bytes(
        s, C.cast(arr, C.c_void_p), len(devices), C.byref(ws_min), C.byref(pmin), C.byref(pfull), ws, nb,
        N.stream_ptr()))
    N.check(rc, "sp_plan_dp_devices_workspace_bytes")
    N.workspace(int(ws_min.value))
    # the partitions of one device share 80 % of its free memory; each takes
    # what keeps every back-pointer stage if that fits its share, else its
    # share (the library checkpoints within it), never below the minimum
    share = {}
    for d in set(int(x) for x in devices):
        dev = torch.device("cuda", d)
        share[d] = min(int(N.free_bytes(dev) * 0.8), N.workspace_cap(dev)) // sum(int(x) == d for x in devices)
    out = []
    for d in devices:
        want = max(int(pmin.value), min(int(pfull.value), share[int(d)]))
        out.append(torch.empty(max(want, 256), dtype=torch.uint8, device=torch.device("cuda", int(d))))
    return out


def dp_workspace_bytes(batch: InstanceBatch) -> tuple[int, int]:
    """(min, full) workspace bytes of plan_dp on this batch (sp_plan_dp_workspace_bytes)."""
    s = batch.struct()
    mn, full = C.c_size_t(0), C.c_size_t(0)
    rc = N.with_workspace(lambda ws, nb: N.library().sp_plan_dp_workspace_bytes(
        s, C.byref(mn), C.byref(full), ws, nb, N.stream_ptr()))
    N.check(rc, "sp_plan_dp_workspace_bytes")
    return int(mn.value), int(full.value)


def plan_prefix(batch: InstanceBatch, which: int, out: PolicyBatch | None = None) -> PolicyBatch:
    out = out or PolicyBatch.empty(batch.n, batch.total_layers, batch.r.device)
    s, o = batch.struct(), out.struct()
    N.check(N.library().sp_plan_prefix(s, which, o, N.stream_ptr()), "sp_plan_prefix")
    return out


def plan_exhaustive(batch: InstanceBatch, out: PolicyBatch | None = None) -> PolicyBatch:
    out = out or PolicyBatch.empty(batch.n, batch.total_layers, batch.r.device)
    s, o = batch.struct(), out.struct()
    N.check(N.library().sp_plan_exhaustive(s, o, N.stream_ptr()), "sp_plan_exhaustive")
    return out


def build_dp_tables(batch: InstanceBatch) -> tuple[torch.Tensor, torch.Tensor]:
    if batch.n != 1:
        raise ValueError("build_dp_tables takes exactly one instance")
    w = int(effective_budget(batch).item())
    L = batch.total_layers
    C = torch.empty((L + 1, w + 1), dtype=torch.float64, device=batch.r.device)
    S = torch.empty_like(C)
    s = batch.struct()
    rc = N.with_workspace(lambda ws, nb: N.library().sp_build_dp_tables(
        s, w, N.ptr(C), N.ptr(S), ws, nb, N.stream_ptr()))
    N.check(rc, "sp_build_dp_tables")
    return C, S


def latency_eq1(batch: InstanceBatch, client_s, server_s, up_s, down_s, pi) -> torch.Tensor:
    out = torch.empty(batch.n, dtype=torch.float64, device=batch.r.device)
    s = batch.struct()
    N.check(N.library().sp_latency_eq1(s, N.ptr(client_s), N.ptr(server_s), N.ptr(up_s),
                                       N.ptr(down_s), N.ptr(pi), N.ptr(out), N.stream_ptr()),
            "sp_latency_eq1")
    return out
