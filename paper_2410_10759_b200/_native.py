"""ctypes binding of the C ABI declared in include/splitplan_b200.h.

This is the only place Python talks to the CUDA library.  Device memory and
streams come from PyTorch (plumbing only); every computation on the hot path
is one of the `sp_*` entry points.  There is no CPU fallback: if the library
or a CUDA device is missing, calls raise.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np
import torch

from ._build import LIB

SP_OK = 0
SP_ERR_INVALID = 1
SP_ERR_CUDA = 2
SP_ERR_WORKSPACE = 3
SP_ERR_BACKTRACE = 4
SP_ERR_DEADLOCK = 5
SP_ERR_UNSUPPORTED = 6

SP_GREEDY, SP_ALL_SERVER, SP_ALL_CLIENT = 0, 1, 2

SP_REQ_PAPER_ROUNDING = 1
SP_REQ_SOURCE_CLIENT = 2
SP_REQ_ZERO_SERVER = 4
SP_REQ_METRIC_MEMORY = 8

KIND_CODE = {"embedding": 0, "attention": 1, "feed_forward": 2,
             "layer_norm": 3, "classifier": 4, "custom": 5}

P = C.c_void_p


class SpInstances(C.Structure):
    _fields_ = [("n", C.c_int64), ("total_layers", C.c_int64), ("layer_off", P),
                ("client_units", P), ("server_units", P), ("up_units", P), ("down_units", P),
                ("r", P), ("budget", P), ("source_at_client", P), ("must_end_at", P)]


class SpPolicies(C.Structure):
    _fields_ = [("pi", P), ("client_value", P), ("server_load", P),
                ("integer_latency", P), ("feasible", P), ("status", P)]


class SpModels(C.Structure):
    _fields_ = [("n_models", C.c_int64), ("layer_off", P), ("kind", P), ("hidden_dim", P),
                ("heads", P), ("ffn_dim", P), ("out_dim", P), ("seq_divisor", P),
                ("flop_coeffs", P), ("mem_coeffs", P), ("has_mem_coeffs", P),
                ("out_bytes_per_token", P), ("has_out_bytes", P)]


class SpRequests(C.Structure):
    _fields_ = [("n", C.c_int64), ("model", P), ("seq_len", P), ("client_fps", P),
                ("server_fps", P), ("uplink_bps", P), ("downlink_bps", P),
                ("propagation_s", P), ("deadline_s", P), ("unit_s", P), ("flags", P)]


class SpProfiles(C.Structure):
    _fields_ = [("r", P), ("client_time_s", P), ("server_time_s", P), ("tau_bytes", P)]


class SpCostTable(C.Structure):
    _fields_ = [("layer_off", P), ("total_layers", C.c_int64), ("r", P), ("client_time_s", P),
                ("server_time_s", P), ("tau_bytes", P), ("server_s", P), ("up_s", P),
                ("down_s", P), ("client_units", P), ("server_units", P), ("up_units", P),
                ("down_units", P), ("budget", P), ("source_at_client", P), ("status", P)]


class SpSimBatch(C.Structure):
    _fields_ = [("n_runs", C.c_int64), ("total_requests", C.c_int64), ("run_off", P),
                ("arrival_ms", P), ("demand", P), ("duration_ms", P), ("capacity", P)]


class SpGridPlan(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("mode", "n_layers", "ctas", "chunks_per_cta", "nparts", "seg_stages",
                                         "nseg", "nckpt", "sac", "owner_part")] + \
               [(n, C.c_int64) for n in ("ncol", "part_cols", "halo", "span", "row_words")] + \
               [(n, C.c_uint64) for n in ("rec_off", "prog_off", "state_off", "rows_off", "ckpt_off", "bp_off",
                                          "ckpt_bytes", "bp_stage", "part_bytes")]


class SpSimOut(C.Structure):
    _fields_ = [("admit_ms", P), ("wait_ms", P), ("cum_wait_ms", P), ("max_wait_ms", P),
                ("mean_wait_ms", P), ("status", P), ("deadlock_req", P)]


SP_PENDING_BYTES = 64  # include/splitplan_b200.h

# name -> (restype, argtypes); the full list the header declares
SIGNATURES = {
    "sp_abi_version": (C.c_int, []),
    "sp_last_error": (C.c_char_p, []),
    "sp_last_required_workspace": (C.c_size_t, []),
    "sp_last_full_workspace": (C.c_size_t, []),
    "sp_last_dense_fallbacks": (C.c_int64, []),
    "sp_profile_enable": (None, [C.c_int]),
    "sp_profile_collect": (C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                     C.POINTER(C.c_double), C.POINTER(C.c_double),
                                     C.POINTER(C.c_int64), C.POINTER(C.c_int32)]),
    "sp_effective_budget": (C.c_int, [C.POINTER(SpInstances), P, P]),
    "sp_plan_dp": (C.c_int, [C.POINTER(SpInstances), C.POINTER(SpPolicies), P, C.c_size_t, P]),
    "sp_plan_dp_async": (C.c_int, [C.POINTER(SpInstances), C.POINTER(SpPolicies), P, C.c_size_t, P, P]),
    "sp_plan_dp_finish": (C.c_int, [C.POINTER(SpInstances), C.POINTER(SpPolicies), P, C.c_size_t, P, P]),
    "sp_plan_dp_devices": (C.c_int, [C.POINTER(SpInstances), C.POINTER(SpPolicies), P, C.c_int32, P,
                                     C.c_size_t, P, P, P]),
    "sp_plan_dp_devices_workspace_bytes": (C.c_int, [C.POINTER(SpInstances), P, C.c_int32,
                                                     C.POINTER(C.c_size_t), C.POINTER(C.c_size_t),
                                                     C.POINTER(C.c_size_t), P, C.c_size_t, P]),
    "sp_grid_plan_make": (C.c_int, [C.POINTER(SpInstances), C.c_int32, C.c_int32, C.c_size_t, C.c_int32,
                                    C.POINTER(SpGridPlan), P, C.c_size_t, P]),
    "sp_grid_part_prepare": (C.c_int, [C.POINTER(SpGridPlan), C.POINTER(SpInstances), P, P]),
    "sp_grid_part_reset": (C.c_int, [C.POINTER(SpGridPlan), P, P]),
    "sp_grid_part_forward": (C.c_int, [C.POINTER(SpGridPlan), C.c_int32, P, C.c_int32, C.c_int32, C.c_int32,
                                       P]),
    "sp_grid_part_end": (C.c_int, [C.POINTER(SpGridPlan), P, C.c_int8, P, P]),
    "sp_grid_part_backtrack": (C.c_int, [C.POINTER(SpGridPlan), C.c_int32, P, C.c_int32, P, P, P]),
    "sp_ipc_export": (C.c_int, [P, P, C.POINTER(C.c_size_t)]),
    "sp_ipc_import": (C.c_int, [P, C.c_size_t, C.POINTER(P), C.POINTER(P)]),
    "sp_ipc_close": (C.c_int, [P]),
    "sp_plan_dp_workspace_bytes": (C.c_int, [C.POINTER(SpInstances), C.POINTER(C.c_size_t),
                                             C.POINTER(C.c_size_t), P, C.c_size_t, P]),
    "sp_build_dp_tables": (C.c_int, [C.POINTER(SpInstances), C.c_int64, P, P, P, C.c_size_t, P]),
    "sp_plan_prefix": (C.c_int, [C.POINTER(SpInstances), C.c_int32, C.POINTER(SpPolicies), P]),
    "sp_plan_exhaustive": (C.c_int, [C.POINTER(SpInstances), C.POINTER(SpPolicies), P]),
    "sp_latency_eq1": (C.c_int, [C.POINTER(SpInstances), P, P, P, P, P, P, P]),
    "sp_request_layer_offsets": (C.c_int, [C.POINTER(SpModels), C.POINTER(SpRequests), P, P]),
    "sp_build_cost_table": (C.c_int, [C.POINTER(SpModels), C.POINTER(SpRequests), C.c_int32,
                                      C.POINTER(SpCostTable), P]),
    "sp_integerize_profiles": (C.c_int, [C.POINTER(SpProfiles), C.POINTER(SpRequests),
                                         C.POINTER(SpCostTable), P]),
    "sp_evaluate_policy": (C.c_int, [C.POINTER(SpInstances), P, C.POINTER(SpPolicies), P,
                                     C.c_size_t, P]),
    "sp_to_units": (C.c_int, [P, C.c_int64, C.c_double, C.c_int32, P, P, P]),
    "sp_segment_sum": (C.c_int, [P, P, C.c_int64, P, P]),
    "sp_sim_workspace_bytes": (C.c_size_t, [C.POINTER(SpSimBatch)]),
    "sp_sim_replay": (C.c_int, [C.POINTER(SpSimBatch), C.POINTER(SpSimOut), P, C.c_size_t, P]),
    "sp_sim_skeletons": (C.c_int, [P, P, P, C.c_int64, C.c_int64, C.c_double, C.c_int64, P, P, P, P, P]),
    "sp_plan_dp_onewave_bytes": (C.c_size_t, [C.c_int64, C.c_int64]),
    "sp_plan_dp_host": (C.c_int, [C.POINTER(SpInstances), C.POINTER(SpPolicies), P, C.c_size_t, P]),
    "sp_plan_prefix_host": (C.c_int, [C.POINTER(SpInstances), C.c_int32, C.POINTER(SpPolicies), P, C.c_size_t,
                                      P]),
}

_lib = None
_lock = threading.Lock()


def library() -> C.CDLL:
    """Load (never silently rebuild on the GPU box) the in-tree library."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not Path(LIB).exists():
                raise RuntimeError(f"splitplan-b200 CUDA library missing at {LIB}; "
                                   "run __graft_entry__.build() first")
            # SPLITPLAN_LIB: an alternative build of the same library (A/B
            # measurements of compile-time variants; tools only)
            lib = C.CDLL(os.environ.get("SPLITPLAN_LIB") or str(LIB))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name, None)
                if fn is None:
                    continue
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    lib = library()
    return [n for n in SIGNATURES if hasattr(lib, n)]


class NativeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def check(rc: int, what: str = "") -> None:
    if rc == SP_OK:
        return
    msg = library().sp_last_error().decode(errors="replace")
    if rc == SP_ERR_INVALID:
        raise ValueError(f"{what}: {msg}")
    raise NativeError(rc, f"{what}: {msg}")


# ---------------------------------------------------------------------------
# device plumbing


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("splitplan-b200 requires a CUDA device (B200, sm_100a); none is visible")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> P:
    return P(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> P:
    if t is None:
        return P(0)
    return P(t.data_ptr())


def to_dev(a, dtype, dev=None) -> torch.Tensor:
    dev = dev or device()
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=dtype).contiguous()
    arr = np.ascontiguousarray(a)
    t = torch.from_numpy(arr)
    if t.dtype != dtype:
        t = t.to(dtype)
    return t.to(dev, non_blocking=False)


def packed(specs, device=None, pin: bool = False, zero_prefix: int = 0):
    """One allocation holding several typed arrays: `specs` is a list of
    (name, numel, torch dtype); each array starts 256-B aligned.  Returns
    (buffer, {name: view}).  The first `zero_prefix` arrays are zeroed with
    one fill.  One copy per direction moves the whole set (the arrays stay
    independent tensors for every consumer)."""
    offs, o = [], 0
    for _name, numel, dt in specs:
        o = (o + 255) & ~255
        offs.append(o)
        o += int(numel) * dt.itemsize
    if device is None or (isinstance(device, str) and device == "cpu"):
        buf = torch.empty(max(o, 1), dtype=torch.uint8, pin_memory=pin)
    else:
        buf = torch.empty(max(o, 1), dtype=torch.uint8, device=device)
    views = {name: buf[off:off + int(numel) * dt.itemsize].view(dt)
             for (name, numel, dt), off in zip(specs, offs)}
    if zero_prefix:
        _name, numel, dt = specs[zero_prefix - 1]
        buf[:offs[zero_prefix - 1] + int(numel) * dt.itemsize].zero_()
    return buf, views


def packed_upload(specs, arrays: dict, device) -> dict:
    """Host arrays -> device views of ONE allocation, with ONE host-to-device
    copy (a call with a handful of small arrays costs one copy instead of one
    per array).  `specs` as for `packed`; `arrays[name]` array-likes."""
    offs, o = [], 0
    for _name, numel, dt in specs:
        o = (o + 255) & ~255
        offs.append(o)
        o += int(numel) * dt.itemsize
    h = np.empty(max(o, 1), dtype=np.uint8)  # staged with numpy: a few us per array
    for (name, numel, dt), off in zip(specs, offs):
        src = arrays[name]
        if isinstance(src, torch.Tensor):
            src = src.cpu().numpy()
        h[off:off + int(numel) * dt.itemsize].view(_NP_OF[dt])[:] = src
    dbuf = torch.from_numpy(h).to(device)
    out = {name: dbuf[off:off + int(numel) * dt.itemsize].view(dt) for (name, numel, dt), off in zip(specs, offs)}
    out["_buf"] = dbuf
    return out


_NP_OF = {torch.int64: np.int64, torch.int32: np.int32, torch.float64: np.float64, torch.uint8: np.uint8,
          torch.int8: np.int8}


_ws: dict[int, torch.Tensor] = {}
_total_mem: dict[int, int] = {}
_WS_MIN = 64 << 20
_WS_ROUND = 64 << 20


def _round_ws(n: int) -> int:
    return max(_WS_MIN, (int(n) + _WS_ROUND - 1) // _WS_ROUND * _WS_ROUND)


def workspace_cap(dev=None) -> int:
    """Largest scratch buffer grown opportunistically: SPLITPLAN_WS_GB, else
    75 % of the device's memory.  Growth beyond what a call requires happens
    only when the call reports it would use the room (sp_last_full_workspace:
    one wave instead of several, fewer checkpoint segments)."""
    env = os.environ.get("SPLITPLAN_WS_GB")
    if env:
        return int(float(env) * (1 << 30))
    d = dev or device()
    key = d.index if d.index is not None else torch.cuda.current_device()
    if key not in _total_mem:
        _total_mem[key] = int(torch.cuda.get_device_properties(key).total_memory)
    return int(_total_mem[key] * 0.75)


def free_bytes(dev) -> int:
    """Free device memory including what PyTorch's caching allocator holds unused."""
    free, _total = torch.cuda.mem_get_info(dev)
    return int(free) + int(torch.cuda.memory_reserved(dev) - torch.cuda.memory_allocated(dev))


def workspace(min_bytes: int = 0) -> torch.Tensor:
    """Per-device cached scratch buffer: 64 MB at first, then grown to what a
    call reports it needs (at least doubling); never grabbed speculatively."""
    dev = device()
    cur = _ws.get(dev.index)
    if cur is None or cur.numel() < min_bytes:
        want = _round_ws(max(min_bytes, 2 * cur.numel() if cur is not None else 0))
        if cur is not None and want > max(workspace_cap(), min_bytes):
            want = _round_ws(min_bytes)
        if cur is not None:
            del _ws[dev.index]
            cur = None
            torch.cuda.empty_cache()
        _ws[dev.index] = torch.empty(want, dtype=torch.uint8, device=dev)
    return _ws[dev.index]


def grow_workspace_hint(full_bytes: int) -> None:
    """After a call that ran in waves: grow the cached workspace to what one
    wave needs (sp_last_full_workspace), within the cap and free memory."""
    dev = device()
    cur = _ws.get(dev.index)
    have = cur.numel() if cur is not None else 0
    del cur  # no reference may keep the old buffer alive while it is replaced
    if full_bytes <= have + (have >> 2):  # the common case: nothing to do, no driver query
        return
    target = min(int(full_bytes), workspace_cap(dev), have + int(free_bytes(dev) * 0.9))
    if target <= have + (have >> 2):  # not worth a reallocation
        return
    workspace(target)


def release_workspace() -> None:
    """Drop the cached scratch buffer of the current device."""
    _ws.pop(device().index, None)
    torch.cuda.empty_cache()


def _useful_size(need: int, full: int, have: int, dev) -> int:
    """What to grow to: at least `need`; up to `full` (one wave, no recompute)
    within the cap and the free memory."""
    room = have + int(free_bytes(dev) * 0.9)
    return max(int(need), min(int(full), workspace_cap(dev), room))


def useful_size(need: int, full: int) -> int:
    """The workspace to allocate for a call that needs `need` bytes and would
    use `full` (one wave, no recompute) on the current device."""
    dev = device()
    cur = _ws.get(dev.index)
    have = cur.numel() if cur is not None else 0
    del cur
    return _useful_size(need, full, have, dev)


def with_workspace(fn, *args):
    """Call fn(*args, ws_ptr, ws_bytes), growing the workspace on SP_ERR_WORKSPACE
    (to what the call reports as useful, not just its minimum)."""
    ws = workspace()
    rc = fn(*args, ptr(ws), C.c_size_t(ws.numel()))
    for _ in range(8):  # each retry covers the largest instance seen failing so far
        if rc != SP_ERR_WORKSPACE:
            break
        lib = library()
        need = int(lib.sp_last_required_workspace())
        if need <= ws.numel():
            break
        have = ws.numel()
        target = _useful_size(need + (1 << 20), int(lib.sp_last_full_workspace()), have, ws.device)
        del ws  # released before the larger buffer is allocated
        ws = workspace(target)
        rc = fn(*args, ptr(ws), C.c_size_t(ws.numel()))
    return rc
