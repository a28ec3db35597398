"""CPU oracle for the SplitLLM placement hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package `splitplan`
(`/root/reference/pkg/src/splitplan`).  It exists so that the CUDA engine in
`paper_2410_10759_b200` can be checked bit-for-bit on the GPU box, where the
reference itself is not available.  Only `tests/`, `__graft_entry__.smoke()`
and the `cpu_baseline` / `--impl reference` legs of `bench.py` may import it;
the product never routes through it.

Parity pinning: every function here is checked against golden vectors that
`tests/golden/gen_golden.py` produced by running the live reference in the
build container (see `tests/test_oracle_golden.py`).

Each function cites the reference file:line it restates.  Arrays replace the
reference's dataclasses: an *instance* is a dict with keys
`i, s, u, d` (int64[L]), `r` (float64[L]), `budget` (int), `sac` (bool).
"""

from __future__ import annotations

import heapq
import math

import numpy as np

NEG = -np.inf
BYTES_PER_ELEMENT = 4
SNAP_REL_TOL = 1e-9
ORACLE_MAX_LAYERS = 24

# layer-kind codes shared with the CUDA cost-table kernel
KIND_CODES = {"embedding": 0, "attention": 1, "feed_forward": 2,
              "layer_norm": 3, "classifier": 4, "custom": 5}


# ---------------------------------------------------------------------------
# cost model  (cost_model.py:137-192, 305-329)


def eff_seq(layer: dict, seq_len: int) -> int:
    """cost_model.py:137-138"""
    return max(1, seq_len // layer.get("seq_divisor", 1))


def _quad(c, s):
    # cost_model.py:141-143 -- evaluated left to right, no fused multiply-add
    q, l, k = c
    return q * s * s + l * s + k


def layer_flops(layer: dict, seq_len: int):
    """cost_model.py:146-165 (exact Python ints for derived kinds)."""
    s = eff_seq(layer, seq_len)
    d = layer["hidden_dim"]
    kind = layer["kind"]
    if kind == "attention":
        return 8 * s * d * d + 4 * s * s * d + 5 * s * s * layer.get("heads", 1)
    if kind == "feed_forward":
        return 4 * s * d * layer["ffn_dim"]
    if kind == "layer_norm":
        return 5 * s * d
    if kind == "embedding":
        return 2 * s * d
    if kind == "classifier":
        return 2 * s * d * layer["out_dim"]
    return _quad(layer["flop_coeffs"], s)


def layer_memory(layer: dict, seq_len: int):
    """cost_model.py:168-177"""
    s = eff_seq(layer, seq_len)
    if layer["kind"] == "custom":
        c = layer.get("mem_coeffs") or (0.0, BYTES_PER_ELEMENT * layer["hidden_dim"], 0.0)
        return _quad(c, s)
    m = s * layer["hidden_dim"] * BYTES_PER_ELEMENT
    if layer["kind"] == "attention":
        m += s * s * layer.get("heads", 1) * BYTES_PER_ELEMENT
    return m


def layer_out_bytes(layer: dict, seq_len: int):
    """cost_model.py:180-187"""
    s = eff_seq(layer, seq_len)
    if layer["kind"] == "classifier":
        return layer["out_dim"] * BYTES_PER_ELEMENT
    if layer["kind"] == "custom" and layer.get("out_bytes_per_token") is not None:
        return layer["out_bytes_per_token"] * s
    return s * layer["hidden_dim"] * BYTES_PER_ELEMENT


def total_flops(layers, seq_len):
    """cost_model.py:195-197"""
    return sum(layer_flops(l, seq_len) for l in layers)


def calibrate_rate(layers, seq_len, target_s):
    """cost_model.py:294-302: flops_per_s so the model takes target_s."""
    return total_flops(layers, seq_len) / target_s


def profile_arrays(layers, seq_len, client_fps, server_fps, metric="flop"):
    """cost_model.py:305-329 -> (r, client_s, server_s, tau) float64 arrays."""
    n = len(layers)
    r = np.empty(n)
    cs = np.empty(n)
    ss = np.empty(n)
    tau = np.empty(n)
    prev_out = seq_len * BYTES_PER_ELEMENT  # raw_input_bytes, cost_model.py:190-192
    for k, layer in enumerate(layers):
        f = layer_flops(layer, seq_len)
        r[k] = float(f if metric == "flop" else layer_memory(layer, seq_len))
        cs[k] = f / client_fps
        ss[k] = f / server_fps
        tau[k] = float(prev_out)
        prev_out = layer_out_bytes(layer, seq_len)
    return r, cs, ss, tau


# -- presets (cost_model.py:204-287), expressed as layer dicts


def _enc(d, h, f, div=1):
    return [dict(kind="attention", hidden_dim=d, heads=h, seq_divisor=div),
            dict(kind="layer_norm", hidden_dim=d, seq_divisor=div),
            dict(kind="feed_forward", hidden_dim=d, ffn_dim=f, seq_divisor=div),
            dict(kind="layer_norm", hidden_dim=d, seq_divisor=div)]


def _dec(d, h, f):
    return [dict(kind="attention", hidden_dim=d, heads=h),
            dict(kind="layer_norm", hidden_dim=d),
            dict(kind="attention", hidden_dim=d, heads=h),
            dict(kind="layer_norm", hidden_dim=d),
            dict(kind="feed_forward", hidden_dim=d, ffn_dim=f),
            dict(kind="layer_norm", hidden_dim=d)]


def preset_layers(name: str):
    if name == "bert-12":
        d, h, f, v, nb = 768, 12, 3072, 30522, 12
    elif name == "gpt2-24":
        d, h, f, v, nb = 1024, 16, 4096, 50257, 24
    elif name == "vanilla-6x6":
        d, h, f, v = 512, 8, 2048, 32000
        out = [dict(kind="embedding", hidden_dim=d, out_dim=v)]
        for _ in range(6):
            out += _enc(d, h, f)
        for _ in range(6):
            out += _dec(d, h, f)
        return out + [dict(kind="classifier", hidden_dim=d, out_dim=v)]
    elif name == "cmt-like":
        out = [dict(kind="embedding", hidden_dim=64)]
        for st, (d, h) in enumerate(zip((64, 128, 256, 512), (1, 2, 4, 8))):
            div = 4 ** st
            if st:
                out.append(dict(kind="embedding", hidden_dim=d, seq_divisor=div))
            for _ in range(2):
                out += _enc(d, h, 4 * d, div)
        return out + [dict(kind="classifier", hidden_dim=512, out_dim=1000, seq_divisor=64)]
    else:
        raise ValueError(name)
    out = [dict(kind="embedding", hidden_dim=d, out_dim=v)]
    for _ in range(nb):
        out += _enc(d, h, f)
    return out + [dict(kind="classifier", hidden_dim=d, out_dim=v)]


# ---------------------------------------------------------------------------
# integerization  (problem.py:58-115, 188-222)


def link_times(tau, up_bps, down_bps, prop_s):
    """problem.py:58-65 -- ((8*tau)/bps) + prop, elementwise."""
    tau = np.asarray(tau, dtype=float)
    return 8.0 * tau / up_bps + prop_s, 8.0 * tau / down_bps + prop_s


def _snapped(q: float) -> float:
    # problem.py:68-72 (Python round = half-to-even)
    n = round(q)
    return float(n) if abs(q - n) <= SNAP_REL_TOL * max(1.0, abs(n)) else q


def units_of(times, unit_s, mode="conservative"):
    """problem.py:79-92"""
    out = []
    for t in np.atleast_1d(np.asarray(times, dtype=float)):
        q = _snapped(t / unit_s)
        out.append(int(math.floor(q + 0.5)) if mode == "paper" else int(math.ceil(q)))
    return np.array(out, dtype=np.int64)


def budget_of(deadline_s, unit_s, mode="conservative"):
    """problem.py:95-104"""
    q = _snapped(deadline_s / unit_s)
    return int(math.floor(q + 0.5)) if mode == "paper" else int(math.floor(q))


def instance_from_profile(r, cs, ss, tau, up_bps, down_bps, prop_s, deadline_s,
                          unit_s=1e-3, sac=True, mode="conservative",
                          zero_server_time=False):
    """problem.py:188-222 -> instance dict (+ real-valued times)."""
    ss = np.zeros(len(r)) if zero_server_time else np.asarray(ss, dtype=float)
    up_s, down_s = link_times(tau, up_bps, down_bps, prop_s)
    cs = np.asarray(cs, dtype=float)
    return dict(i=units_of(cs, unit_s, mode), s=units_of(ss, unit_s, mode),
                u=units_of(up_s, unit_s, mode), d=units_of(down_s, unit_s, mode),
                r=np.asarray(r, dtype=float), budget=budget_of(deadline_s, unit_s, mode),
                sac=bool(sac), client_s=cs, server_s=ss, up_s=up_s, down_s=down_s,
                deadline_s=deadline_s)


# ---------------------------------------------------------------------------
# planners  (planner.py)


def effective_budget(inst) -> int:
    """planner.py:120-125"""
    worst = int(np.sum(np.maximum(inst["i"] + inst["d"], inst["s"] + inst["u"])))
    return min(int(inst["budget"]), worst)


def _shifted(row, k):
    # planner.py:110-117: move right by k columns, vacated cells unreachable
    if k == 0:
        return row
    out = np.full_like(row, NEG)
    if k < row.size:
        out[k:] = row[: row.size - k]
    return out


def dp_tables(inst):
    """planner.py:128-143 -> (C, S) float64 [(L+1), (W_eff+1)]."""
    L = len(inst["r"])
    W = effective_budget(inst)
    C = np.full((L + 1, W + 1), NEG)
    S = np.full((L + 1, W + 1), NEG)
    (C if inst["sac"] else S)[0, :] = 0.0
    with np.errstate(invalid="ignore"):
        for k in range(L):
            ik, sk = int(inst["i"][k]), int(inst["s"][k])
            uk, dk = int(inst["u"][k]), int(inst["d"][k])
            C[k + 1] = np.maximum(_shifted(C[k], ik), _shifted(S[k], ik + dk)) + inst["r"][k]
            S[k + 1] = np.maximum(_shifted(S[k], sk), _shifted(C[k], sk + uk))
    return C, S


class BacktraceError(AssertionError):
    pass


def backtrace(C, S, inst, side_client: bool):
    """planner.py:146-179 -- value-re-deriving walk from (L, W_eff)."""
    L = len(inst["r"])
    j = C.shape[1] - 1
    pi = np.zeros(L, dtype=np.int64)
    on_client = side_client
    for k in range(L, 0, -1):
        ik, sk = int(inst["i"][k - 1]), int(inst["s"][k - 1])
        uk, dk = int(inst["u"][k - 1]), int(inst["d"][k - 1])
        rk = inst["r"][k - 1]
        if on_client:
            pi[k - 1] = 1
            v = C[k, j]
            if j >= ik and C[k - 1, j - ik] + rk == v:
                j -= ik
            elif j >= ik + dk and S[k - 1, j - ik - dk] + rk == v:
                j -= ik + dk
                on_client = False
            else:
                raise BacktraceError("no predecessor reproduces the stored value")
        else:
            v = S[k, j]
            if j >= sk and S[k - 1, j - sk] == v:
                j -= sk
            elif j >= sk + uk and C[k - 1, j - sk - uk] == v:
                j -= sk + uk
                on_client = True
            else:
                raise BacktraceError("no predecessor reproduces the stored value")
    return pi


def latency_units(pi, inst) -> int:
    """planner.py:69-85 (exact integer sum)."""
    prev = 1 if inst["sac"] else 0
    tot = 0
    for k, x in enumerate(pi):
        x = int(x)
        if x:
            tot += int(inst["i"][k]) + (int(inst["d"][k]) if prev == 0 else 0)
        else:
            tot += int(inst["s"][k]) + (int(inst["u"][k]) if prev == 1 else 0)
        prev = x
    return tot


def finish(pi, inst, planner, feasible=None):
    """planner.py:88-101 -> policy dict; sums use numpy's pairwise np.sum."""
    x = np.asarray(pi, dtype=np.int64)
    lat = latency_units(x, inst)
    return dict(planner=planner, pi=tuple(int(v) for v in x),
                client_value=float(np.sum(inst["r"][x == 1])),
                server_load=float(np.sum(inst["r"][x == 0])),
                integer_latency=lat,
                feasible=bool(lat <= inst["budget"] if feasible is None else feasible))


def infeasible(inst, planner):
    """planner.py:104-107"""
    return finish(np.zeros(len(inst["r"]), dtype=np.int64), inst, planner, feasible=False)


def plan_dp(inst, must_end_at=None):
    """planner.py:182-202"""
    C, S = dp_tables(inst)
    ec, es = C[-1, -1], S[-1, -1]
    if must_end_at == "client":
        es = NEG
    elif must_end_at == "server":
        ec = NEG
    elif must_end_at is not None:
        raise ValueError(f"must_end_at must be 'client' or 'server', got {must_end_at!r}")
    if max(ec, es) == NEG:  # Python max: keeps the first operand unless the second is larger
        return infeasible(inst, "dp")
    return finish(backtrace(C, S, inst, bool(ec >= es)), inst, "dp")


def prefix_latency(inst, m: int) -> int:
    """Closed form of planner.py:69-85 for pi = 1^m 0^(L-m)."""
    L = len(inst["r"])
    i, s, u, d = inst["i"], inst["s"], inst["u"], inst["d"]
    lat = int(np.sum(i[:m])) + int(np.sum(s[m:]))
    if m < L and (m >= 1 or inst["sac"]):
        lat += int(u[m])
    if m >= 1 and not inst["sac"]:
        lat += int(d[0])
    return lat


def plan_greedy(inst):
    """planner.py:205-214"""
    L = len(inst["r"])
    for m in range(L, -1, -1):
        if prefix_latency(inst, m) <= inst["budget"]:
            return finish(np.r_[np.ones(m, np.int64), np.zeros(L - m, np.int64)], inst, "greedy")
    return infeasible(inst, "greedy")


def plan_trivial(inst, side):
    """planner.py:217-225"""
    L = len(inst["r"])
    if side == "all_server":
        return finish(np.zeros(L, np.int64), inst, side)
    if side == "all_client":
        return finish(np.ones(L, np.int64), inst, side)
    raise ValueError(f"side must be 'all_server' or 'all_client', got {side!r}")


def plan_exhaustive(inst, chunk=1 << 16):
    """planner.py:228-268 -- every mask in chunks of 65,536: latency as a float
    sum, value = x @ r (numpy's BLAS dgemv: its summation order decides ties
    under non-dyadic r), np.argmax inside a chunk (first max; a NaN value
    wins), across chunks only a strictly greater value replaces the best."""
    L = len(inst["r"])
    if L > ORACLE_MAX_LAYERS:
        raise ValueError(f"oracle limited to {ORACLE_MAX_LAYERS} layers, got {L}")
    i, s = inst["i"].astype(float), inst["s"].astype(float)
    u, d = inst["u"].astype(float), inst["d"].astype(float)
    r = np.asarray(inst["r"], dtype=float)
    x0 = 1.0 if inst["sac"] else 0.0
    shifts = np.arange(L - 1, -1, -1, dtype=np.uint32)
    best_value, best_mask = None, None
    with np.errstate(invalid="ignore"):
        for start in range(0, 1 << L, chunk):
            masks = np.arange(start, min(start + chunk, 1 << L), dtype=np.uint32)
            x = ((masks[:, None] >> shifts[None, :]) & 1).astype(float)
            xprev = np.empty_like(x)
            xprev[:, 0] = x0
            xprev[:, 1:] = x[:, :-1]
            lat = np.sum(x * (i + (1 - xprev) * d) + (1 - x) * (s + xprev * u), axis=1)
            value = x @ r
            ok = lat <= inst["budget"]
            if not np.any(ok):
                continue
            value_ok = np.where(ok, value, NEG)
            idx = int(np.argmax(value_ok))
            if best_value is None or value_ok[idx] > best_value:
                best_value, best_mask = float(value_ok[idx]), int(masks[idx])
    if best_value is None:
        return infeasible(inst, "oracle")
    pi = np.array([(best_mask >> int(sh)) & 1 for sh in shifts], np.int64)
    return finish(pi, inst, "oracle")


# ---------------------------------------------------------------------------
# evaluator  (evaluator.py:64-113)


def eq1_latency(pi, cs, ss, up, down, sac) -> float:
    """evaluator.py:64-69 (elementwise terms, then pairwise np.sum)."""
    x = np.asarray(pi, dtype=float)
    xp = np.empty_like(x)
    xp[0] = 1.0 if sac else 0.0
    xp[1:] = x[:-1]
    terms = x * (cs + (1.0 - xp) * down) + (1.0 - x) * (ss + xp * up)
    return float(np.sum(terms))


# ---------------------------------------------------------------------------
# throughput simulator  (throughput_sim.py:179-256)


class Deadlock(RuntimeError):
    pass


def skeleton(seed, n, beta_per_ms, n_scen, exec_max=10):
    """throughput_sim.py:179-186"""
    g = np.random.default_rng(seed)
    arr = np.cumsum(g.exponential(scale=1.0 / beta_per_ms, size=n))
    idx = g.integers(0, n_scen, size=n)
    ex = g.integers(1, exec_max + 1, size=n)
    return arr, idx, ex


def fifo_replay(arrival, demand, duration, capacity):
    """throughput_sim.py:207-256 -> admit times (float64[n])."""
    n = len(arrival)
    admit = np.zeros(n)
    eps = 1e-9 * capacity
    free = capacity
    busy = []  # (finish, seq, req)
    head = 0
    seq = 0
    nxt = 0
    waiting = []
    while nxt < n or busy:
        t_arr = arrival[nxt] if nxt < n else np.inf
        if busy and busy[0][0] <= t_arr:
            now, _, done = heapq.heappop(busy)
            free += demand[done]
        else:
            waiting.append(nxt)
            now = t_arr
            nxt += 1
        while head < len(waiting):
            q = waiting[head]
            if demand[q] <= free + eps:
                admit[q] = now
                free -= demand[q]
                heapq.heappush(busy, (now + duration[q], seq, q))
                seq += 1
                head += 1
            else:
                if demand[q] > capacity + eps:
                    raise Deadlock(q)
                break
    return admit
