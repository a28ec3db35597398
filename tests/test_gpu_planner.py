"""CUDA planners vs the reference's golden vectors and the pinned oracle.

Bit-exact: placements, integer latencies and feasibility must be equal, and
client_value / server_load equal as float64 bit patterns."""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import GOLDEN, Battery, assert_policy, load_npz
from oracle import splitplan_oracle as O

pytestmark = pytest.mark.gpu

BATTERIES = ["battery_acceptance", "battery_special", "battery_float", "battery_oracle_ties",
             "battery_wide"]


def _batch(bat: Battery, with_must=True):
    from paper_2410_10759_b200 import batch as B
    z = bat.z
    return B.InstanceBatch.from_arrays(z["off"], z["i"], z["s"], z["u"], z["d"], z["r"],
                                       z["budget"], z["sac"], z["must"] if with_must else None)


def _compare(bat: Battery, planner: str, host: dict, *, backtrace_ok=False):
    from paper_2410_10759_b200 import _native as N
    off = bat.off
    for k in range(bat.n):
        exp = bat.expected(planner, k)
        if exp is None:
            assert host["status"][k] == N.SP_ERR_BACKTRACE, f"{bat.name}[{k}] expected assertion"
            continue
        assert host["status"][k] == 0, f"{bat.name}[{k}] status {host['status'][k]}"
        got = dict(pi=host["pi"][off[k]:off[k + 1]], client_value=host["client_value"][k],
                   server_load=host["server_load"][k], integer_latency=host["integer_latency"][k],
                   feasible=host["feasible"][k])
        assert_policy(got, exp, f"{bat.name}[{k}] {planner}")


@pytest.mark.parametrize("name", BATTERIES)
def test_dp_batch_matches_reference(gpu, name):
    from paper_2410_10759_b200 import batch as B
    bat = Battery(name)
    b = _batch(bat)
    w = B.effective_budget(b).cpu().numpy()
    np.testing.assert_array_equal(w, bat.z["w_eff"])
    _compare(bat, "dp", B.plan_dp(b).to_host())


@pytest.mark.parametrize("name", BATTERIES)
def test_prefix_planners_match_reference(gpu, name):
    from paper_2410_10759_b200 import _native as N, batch as B
    bat = Battery(name)
    if not bat.has("greedy"):
        pytest.skip("battery has no greedy outputs")
    b = _batch(bat, with_must=False)
    for planner, code in (("greedy", N.SP_GREEDY), ("all_server", N.SP_ALL_SERVER),
                          ("all_client", N.SP_ALL_CLIENT)):
        _compare(bat, planner, B.plan_prefix(b, code).to_host())


@pytest.mark.parametrize("name", ["battery_acceptance", "battery_oracle_ties", "battery_oracle_float"])
def test_exhaustive_matches_reference(gpu, name):
    from paper_2410_10759_b200 import batch as B
    bat = Battery(name)
    _compare(bat, "oracle", B.plan_exhaustive(_batch(bat, with_must=False)).to_host())


def test_dp_tables_match_reference(gpu):
    from paper_2410_10759_b200 import planner as P
    from paper_2410_10759_b200.problem import PlanProblem
    z = load_npz("dp_tables")
    off, pos = z["off"], 0
    for k in range(len(off) - 1):
        a, b = off[k], off[k + 1]
        prob = PlanProblem.from_costs(z["i"][a:b], z["s"][a:b], z["u"][a:b], z["d"][a:b],
                                      z["r"][a:b], int(z["budget"][k]),
                                      source_at_client=bool(z["sac"][k]))
        t = P.build_dp_tables(prob)
        cnt = t.client.size
        np.testing.assert_array_equal(t.client.ravel(), z["C"][pos:pos + cnt])
        np.testing.assert_array_equal(t.server.ravel(), z["S"][pos:pos + cnt])
        pos += cnt


@pytest.mark.parametrize("variant", ["global", "smem", "stream"])
def test_dp_tables_every_variant(gpu, variant, monkeypatch):
    """Full tables from each K2 variant equal the reference's build_dp_tables."""
    from paper_2410_10759_b200 import planner as P
    from paper_2410_10759_b200.problem import PlanProblem
    monkeypatch.setenv("SPLITPLAN_DP_VARIANT", variant)
    z = load_npz("dp_tables")
    off, pos = z["off"], 0
    for k in range(len(off) - 1):
        a, b = off[k], off[k + 1]
        prob = PlanProblem.from_costs(z["i"][a:b], z["s"][a:b], z["u"][a:b], z["d"][a:b],
                                      z["r"][a:b], int(z["budget"][k]),
                                      source_at_client=bool(z["sac"][k]))
        t = P.build_dp_tables(prob)
        cnt = t.client.size
        np.testing.assert_array_equal(t.client.ravel(), z["C"][pos:pos + cnt], err_msg=f"C {k}")
        np.testing.assert_array_equal(t.server.ravel(), z["S"][pos:pos + cnt], err_msg=f"S {k}")
        pos += cnt


def test_dropin_fixtures(gpu):
    """The reference's own frozen fixtures (tests/test_planner.py:26-108)."""
    from paper_2410_10759_b200.planner import plan_dp, plan_greedy, plan_oracle, plan_trivial, run_planner
    from paper_2410_10759_b200.problem import PlanProblem
    a = PlanProblem.from_costs([4, 4, 4], [0, 0, 0], [1, 1, 1], [1, 1, 1], [5.0, 1.0, 5.0], 9)
    b = PlanProblem.from_costs([4, 4, 4], [0, 0, 0], [1, 1, 1], [1, 1, 1], [1.0, 1.0, 10.0], 9)
    p = plan_dp(a)
    assert p.pi == (1, 1, 0) and p.server_load == 5.0 and p.client_value == 6.0
    assert p.integer_latency == 9 and p.feasible
    p = plan_dp(b)
    assert p.pi == (0, 0, 1) and p.server_load == 2.0 and p.integer_latency == 6
    g = plan_greedy(b)
    assert g.pi == (1, 1, 0) and g.server_load == 10.0 and g.feasible
    assert plan_trivial(a, "all_server").integer_latency == 1
    assert plan_oracle(b).pi == (0, 0, 1)
    assert plan_dp(b, must_end_at="server").pi[-1] == 0
    with pytest.raises(ValueError):
        plan_dp(b, must_end_at="edge")
    with pytest.raises(ValueError):
        run_planner("simulated-annealing", b)
    assert run_planner("all-server", b).pi == (0, 0, 0)
    nan = PlanProblem.from_costs([1, 1, 1], [1, 1, 1], [1, 1, 1], [1, 1, 1], [math.nan, 1.0, 2.0], 5)
    with pytest.raises(AssertionError, match="no predecessor"):
        plan_dp(nan)


def _random_instances(seed, n, L_range, W_choices, r_kind):
    rng = np.random.default_rng(seed)
    out = []
    for t in range(n):
        L = int(rng.integers(*L_range))
        W = int(rng.choice(W_choices))
        hi = max(2, W // max(4, L // 3))
        i, s = rng.integers(0, hi, L), rng.integers(0, max(2, hi // 6), L)
        u, d = rng.integers(0, hi, L), rng.integers(0, hi, L)
        if r_kind == "int":
            r = rng.integers(0, 1000, L).astype(float)
        elif r_kind == "bigint":
            r = rng.integers(0, 2 ** 40, L).astype(float)
        elif r_kind == "float":
            r = rng.random(L) * 10.0 ** rng.integers(-2, 12, L)
        else:
            r = rng.integers(0, 10, L).astype(float)
            r[rng.integers(0, L)] = math.inf
        out.append(dict(i=i, s=s, u=u, d=d, r=r, budget=W, sac=bool(t % 2)))
    return out


@pytest.mark.parametrize("r_kind", ["int", "bigint", "float", "inf"])
def test_dp_vs_oracle_smem_and_global_rows(gpu, r_kind):
    """Seeded instances spanning SMEM-resident rows and global rows, in every
    value domain (int32 exact, fp64 finite, fp64 NaN-propagating)."""
    from paper_2410_10759_b200 import batch as B
    seed = {"int": 1, "bigint": 2, "float": 3, "inf": 4}[r_kind]
    insts = _random_instances(seed, 10, (3, 40), [50, 900, 9000, 20000, 40000], r_kind)
    off = np.zeros(len(insts) + 1, np.int64)
    np.cumsum([len(x["r"]) for x in insts], out=off[1:])
    cat = lambda k: np.concatenate([x[k] for x in insts])
    b = B.InstanceBatch.from_arrays(off, cat("i"), cat("s"), cat("u"), cat("d"), cat("r"),
                                    [x["budget"] for x in insts], [x["sac"] for x in insts])
    host = B.plan_dp(b).to_host()
    for k, inst in enumerate(insts):
        try:
            exp = O.plan_dp(inst)
        except AssertionError:
            assert host["status"][k] != 0
            continue
        got = dict(pi=host["pi"][off[k]:off[k + 1]], client_value=host["client_value"][k],
                   server_load=host["server_load"][k], integer_latency=host["integer_latency"][k],
                   feasible=host["feasible"][k])
        assert_policy(got, dict(exp, pi=tuple(exp["pi"])), f"{r_kind}[{k}]")


@pytest.mark.parametrize("variant", ["global", "smem", "stream", "grid"])
@pytest.mark.parametrize("name", ["battery_wide", "battery_float", "battery_large_model"])
def test_dp_kernel_variants_agree(gpu, variant, name, monkeypatch):
    """Every K2 variant (rows in one CTA's SMEM, in L2-resident global rows,
    in global memory, over the whole GPU) is bit-exact on the same instances
    (the host falls back where a variant cannot hold a row)."""
    if not (GOLDEN / f"{name}.npz").exists():
        pytest.skip("battery not generated")
    from paper_2410_10759_b200 import batch as B
    monkeypatch.setenv("SPLITPLAN_DP_VARIANT", variant)
    bat = Battery(name)
    _compare(bat, "dp", B.plan_dp(_batch(bat)).to_host())


@pytest.mark.parametrize("threads", ["64", "128", "256", "512"])
def test_single_cta_thread_configs(gpu, threads, monkeypatch):
    """Every T x E instantiation of the single-CTA kernel (SMEM and global rows)."""
    from paper_2410_10759_b200 import batch as B
    monkeypatch.setenv("SPLITPLAN_DP_THREADS", threads)
    monkeypatch.setenv("SPLITPLAN_DP_SINGLE_E", "4")
    for variant in ("smem", "global"):
        monkeypatch.setenv("SPLITPLAN_DP_VARIANT", variant)
        bat = Battery("battery_float")
        _compare(bat, "dp", B.plan_dp(_batch(bat)).to_host())


@pytest.mark.parametrize("threads", ["128", "256", ""])
def test_single_cta_eight_columns_per_thread(gpu, threads, monkeypatch):
    """The int32 single-CTA kernel with 8 columns per thread per chunk."""
    from paper_2410_10759_b200 import batch as B
    monkeypatch.setenv("SPLITPLAN_DP_SINGLE_E", "8")
    monkeypatch.setenv("SPLITPLAN_DP_THREADS", threads)
    monkeypatch.setenv("SPLITPLAN_DP_VARIANT", "smem")
    for name in ("battery_acceptance", "battery_wide", "battery_special"):
        bat = Battery(name)
        _compare(bat, "dp", B.plan_dp(_batch(bat)).to_host())


@pytest.mark.parametrize("cluster", ["1", "3", "16"])
def test_stream_cluster_sizes(gpu, cluster, monkeypatch):
    """The streaming kernel at forced cluster sizes (1 CTA, odd, the non-portable 16)."""
    from paper_2410_10759_b200 import batch as B
    monkeypatch.setenv("SPLITPLAN_DP_VARIANT", "stream")
    monkeypatch.setenv("SPLITPLAN_DP_CLUSTER", cluster)
    for name in ("battery_wide", "battery_large_model"):
        bat = Battery(name)
        _compare(bat, "dp", B.plan_dp(_batch(bat)).to_host())


@pytest.mark.parametrize("segment", ["0", "7", "1"])
def test_grid_checkpoint_recompute(gpu, segment, monkeypatch):
    """The whole-GPU path for one huge instance, with the back-pointers kept
    whole (segment 0) or recomputed from checkpoint rows every 7 / 1 stages."""
    from paper_2410_10759_b200 import batch as B
    monkeypatch.setenv("SPLITPLAN_DP_VARIANT", "grid")
    monkeypatch.setenv("SPLITPLAN_GRID_SEGMENT", segment)
    for name in ("battery_wide", "battery_special"):
        bat = Battery(name)
        _compare(bat, "dp", B.plan_dp(_batch(bat)).to_host())
    for r_kind in ("int", "float", "inf"):
        insts = _random_instances(7, 6, (3, 30), [900, 20000], r_kind)
        off = np.zeros(len(insts) + 1, np.int64)
        np.cumsum([len(x["r"]) for x in insts], out=off[1:])
        cat = lambda k: np.concatenate([x[k] for x in insts])
        b = B.InstanceBatch.from_arrays(off, cat("i"), cat("s"), cat("u"), cat("d"), cat("r"),
                                        [x["budget"] for x in insts], [x["sac"] for x in insts])
        host = B.plan_dp(b).to_host()
        for k, inst in enumerate(insts):
            try:
                exp = O.plan_dp(inst)
            except AssertionError:
                assert host["status"][k] != 0
                continue
            got = dict(pi=host["pi"][off[k]:off[k + 1]], client_value=host["client_value"][k],
                       server_load=host["server_load"][k], integer_latency=host["integer_latency"][k],
                       feasible=host["feasible"][k])
            assert_policy(got, dict(exp, pi=tuple(exp["pi"])), f"grid {r_kind}[{k}]")


@pytest.mark.parametrize("parts,segment,mode", [("2", "0", ""), ("3", "13", ""), ("8", "0", ""),
                                                ("2", "0", "separate"), ("4", "13", "separate"),
                                                ("3", "0", "separate+sys")])
def test_grid_capacity_partitions(gpu, parts, segment, mode, monkeypatch):
    """The capacity axis split into partitions (one per device in a multi-GPU
    run, emulated here on one GPU) with the left neighbour's columns mirrored
    in a halo: bit-exact against the live reference's cfg5-reduced chains."""
    from paper_2410_10759_b200 import batch as B
    monkeypatch.setenv("SPLITPLAN_DP_VARIANT", "grid")
    monkeypatch.setenv("SPLITPLAN_GRID_PARTS", parts)
    monkeypatch.setenv("SPLITPLAN_GRID_SEGMENT", segment)
    # "separate": one launch per partition, all in flight together (the
    # multi-device protocol with every partition on this GPU); "+sys":
    # system-scope progress counters as across devices
    monkeypatch.setenv("SPLITPLAN_GRID_SEPARATE", "1" if "separate" in mode else "0")
    monkeypatch.setenv("SPLITPLAN_GRID_SYS", "1" if "sys" in mode else "0")
    for name, must in (("battery_large_chain", False), ("battery_wide", True)):
        bat = Battery(name)
        _compare(bat, "dp", B.plan_dp(_batch(bat, with_must=must)).to_host())


@pytest.mark.parametrize("name", ["battery_large_model", "battery_large_chain"])
def test_full_size_batteries(gpu, name):
    """W_eff = 1e5 model-derived instances (BASELINE cfg2 shape) and the
    cfg5-reduced chains (L=1e5 x W=1e3, L=1e3 x W=1e5)."""
    if not (GOLDEN / f"{name}.npz").exists():
        pytest.skip("large battery not generated")
    from paper_2410_10759_b200 import _native as N, batch as B
    bat = Battery(name)
    b = _batch(bat, with_must=False)
    _compare(bat, "dp", B.plan_dp(b).to_host())
    if bat.has("greedy"):
        _compare(bat, "greedy", B.plan_prefix(b, N.SP_GREEDY).to_host())


@pytest.mark.parametrize("devices,segment", [([0, 0], "0"), ([0, 0, 0, 0], "0"), ([0] * 8, "0"),
                                             ([0, 0], "13"), ([0, 0, 0], "1"), ([0] * 8, "29")])
def test_plan_dp_devices_partitions(gpu, devices, segment, monkeypatch):
    """sp_plan_dp_devices: the capacity axis of whole-GPU instances split over
    a device list (here the one GPU listed several times: one launch per
    partition, system-scope counters, the multi-device code path).  Every
    partition keeps its rows, checkpoints and back-pointers in its OWN
    workspace allocation, and the backtrack hands (stage, column, side) from
    partition to partition; with and without checkpoint / recompute."""
    from paper_2410_10759_b200 import batch as B
    monkeypatch.setenv("SPLITPLAN_DP_VARIANT", "grid")
    monkeypatch.setenv("SPLITPLAN_GRID_SEGMENT", segment)
    for name, must in (("battery_large_chain", False), ("battery_wide", True)):
        bat = Battery(name)
        _compare(bat, "dp", B.plan_dp(_batch(bat, with_must=must), devices=devices).to_host())


def test_plan_dp_devices_minimum_partition_workspaces(gpu, monkeypatch):
    """Partition workspaces of exactly the queried minimum (checkpoint /
    recompute chosen by the library) give the same placements; one byte less
    than what a partition needs is a clean SP_ERR_WORKSPACE."""
    import ctypes as C
    import torch
    from paper_2410_10759_b200 import _native as N, batch as B
    monkeypatch.setenv("SPLITPLAN_DP_VARIANT", "grid")
    bat = Battery("battery_large_chain")
    b = _batch(bat, with_must=False)
    devices = [0, 0, 0]
    arr = (C.c_int32 * 3)(*devices)
    ws_min, pmin, pfull = C.c_size_t(0), C.c_size_t(0), C.c_size_t(0)
    lib = N.library()
    rc = N.with_workspace(lambda ws, nb: lib.sp_plan_dp_devices_workspace_bytes(
        b.struct(), C.cast(arr, C.c_void_p), 3, C.byref(ws_min), C.byref(pmin), C.byref(pfull), ws, nb,
        N.stream_ptr()))
    assert rc == 0, lib.sp_last_error()
    assert 0 < pmin.value <= pfull.value
    for size, ok in ((pmin.value, True), (pfull.value, True), (pmin.value - 4096, False)):
        parts = [torch.empty(size, dtype=torch.uint8, device="cuda") for _ in devices]
        wptr = (C.c_void_p * 3)(*[t.data_ptr() for t in parts])
        wlen = (C.c_size_t * 3)(*[size] * 3)
        out = B.PolicyBatch.empty(b.n, b.total_layers, b.r.device)
        ws = N.workspace(ws_min.value)
        rc = lib.sp_plan_dp_devices(b.struct(), out.struct(), C.cast(arr, C.c_void_p), 3, N.ptr(ws), ws.numel(),
                                    C.cast(wptr, C.c_void_p), C.cast(wlen, C.c_void_p), N.stream_ptr())
        torch.cuda.synchronize()
        if ok:
            assert rc == 0, lib.sp_last_error()
            _compare(bat, "dp", out.to_host())
        else:
            assert rc == N.SP_ERR_WORKSPACE, lib.sp_last_error()


def test_exhaustive_rejects_long_instances(gpu):
    """sp_plan_exhaustive checks L <= 24 itself (no 2^L overflow / index
    overrun), whatever the Python wrapper knows about the lengths."""
    from paper_2410_10759_b200 import _native as N, batch as B
    L = 30
    b = B.InstanceBatch.from_arrays([0, L], np.ones(L), np.ones(L), np.ones(L), np.ones(L), np.ones(L), [10], [1])
    out = B.PolicyBatch.empty(1, L, b.r.device)
    rc = N.library().sp_plan_exhaustive(b.struct(), out.struct(), N.stream_ptr())
    assert rc == N.SP_ERR_UNSUPPORTED
    b.n_layers_host = None  # the batched planner derives the lengths from the device offsets
    from paper_2410_10759_b200.planner import plan_batch
    with pytest.raises(ValueError, match="oracle limited to 24 layers"):
        plan_batch("oracle", b)


def test_build_dp_tables_checks_w_eff(gpu):
    """sp_build_dp_tables refuses tables sized for another W_eff before writing."""
    import torch
    from paper_2410_10759_b200 import _native as N, batch as B
    b = B.InstanceBatch.from_arrays([0, 3], [2, 2, 2], [1, 1, 1], [1, 1, 1], [1, 1, 1], [1.0, 2.0, 3.0], [5], [1])
    C = torch.empty((4, 3), dtype=torch.float64, device="cuda")
    S = torch.empty_like(C)
    rc = N.with_workspace(lambda ws, nb: N.library().sp_build_dp_tables(b.struct(), 2, N.ptr(C), N.ptr(S), ws, nb,
                                                                        N.stream_ptr()))
    assert rc == N.SP_ERR_INVALID and b"does not match" in N.library().sp_last_error()


def test_plan_dp_devices_rejects_bad_lists(gpu):
    from paper_2410_10759_b200 import _native as N, batch as B
    import torch
    bat = Battery("battery_wide")
    b = _batch(bat)
    for bad in ([1 + torch.cuda.device_count()], [torch.cuda.device_count() + 3, 0]):
        with pytest.raises(Exception):
            B.plan_dp(b, devices=bad)


@pytest.mark.parametrize("variant", ["stream", "grid"])
@pytest.mark.parametrize("no_reach", ["0", "1"])
def test_reachable_frontier_skips(gpu, variant, no_reach, monkeypatch):
    """Window copies below the reachable frontier skipped and dead chunks left
    uncomputed (default) or everything computed (SPLITPLAN_NO_REACH=1): the
    same placements either way."""
    from paper_2410_10759_b200 import batch as B
    monkeypatch.setenv("SPLITPLAN_DP_VARIANT", variant)
    monkeypatch.setenv("SPLITPLAN_NO_REACH", no_reach)
    for name, must in (("battery_large_chain", False), ("battery_wide", True), ("battery_large_model", True)):
        bat = Battery(name)
        _compare(bat, "dp", B.plan_dp(_batch(bat, with_must=must)).to_host())


@pytest.mark.parametrize("variant", ["stream", ""])
def test_dp_workspace_query(gpu, variant, monkeypatch):
    """sp_plan_dp_workspace_bytes: plan_dp runs in exactly the reported minimum
    workspace (bit-exact).  The minimum covers the dense kernels every
    instance may fall back to; with the dense kernels forced, one page less
    fails cleanly (by default the breakpoint lists may still fit: then the
    result must be bit-exact)."""
    import torch
    from paper_2410_10759_b200 import _native as N, batch as B
    if variant:
        monkeypatch.setenv("SPLITPLAN_DP_VARIANT", variant)
    bat = Battery("battery_large_model")
    b = _batch(bat)
    mn, full = B.dp_workspace_bytes(b)
    assert 0 < mn <= full
    lib = N.library()
    for size, ok in ((mn, True), (full, True), (mn - 4096, False)):
        ws = torch.empty(size, dtype=torch.uint8, device=N.device())
        out = B.PolicyBatch.empty(b.n, b.total_layers, b.r.device)
        rc = lib.sp_plan_dp(b.struct(), out.struct(), N.ptr(ws), size, N.stream_ptr())
        torch.cuda.synchronize()
        if ok or (rc == 0 and not variant):
            assert rc == 0, N.library().sp_last_error()
            _compare(bat, "dp", out.to_host())
        else:
            assert rc == N.SP_ERR_WORKSPACE


# ---------------------------------------------------------------------------
# breakpoint lists (dp_steps.cuh): rows as step functions, stay_from back-pointers


@pytest.mark.parametrize("name", BATTERIES + ["battery_large_model", "battery_large_chain"])
def test_breakpoint_lists_match_reference(gpu, name, monkeypatch):
    """The breakpoint-list tiers alone (instances they cannot hold fall back to
    the dense kernels): bit-exact on every reference battery, including the
    survey's fp-absorption vector and must_end_at."""
    from paper_2410_10759_b200 import batch as B
    monkeypatch.setenv("SPLITPLAN_DP_VARIANT", "steps")
    bat = Battery(name)
    _compare(bat, "dp", B.plan_dp(_batch(bat, with_must=name != "battery_large_chain")).to_host())


def _dense_rows_instances(seed, n):
    """Every third instance has random float r and shifts of 0..60 over 600
    stages and 30,001 columns: rows of ~1,250 breakpoints, more than both
    breakpoint tiers hold (dense fallback); the others have small integer r
    (a few breakpoints, tier 1)."""
    rng = np.random.default_rng(seed)
    out = []
    for t in range(n):
        hard = t % 3 == 0
        L, W, hi = (600, 30000, 60) if hard else (160, 3000, 400)
        out.append(dict(i=rng.integers(0, hi, L), s=rng.integers(0, hi, L), u=rng.integers(0, hi, L),
                        d=rng.integers(0, hi, L),
                        r=(rng.random(L) * 50 if hard else rng.integers(0, 5, L).astype(float)),
                        budget=int(W), sac=bool(t % 2)))
    return out


@pytest.mark.parametrize("ws_kind", ["large", "small"])
def test_breakpoint_tiers_and_fallback(gpu, ws_kind, monkeypatch):
    """Instances whose rows outgrow the tier-1 lists move to the wide tier and
    then to the dense kernels (sp_last_dense_fallbacks counts the latter);
    with a workspace too small for the device-planned tier everything runs in
    host-planned waves.  Every result is bit-exact against the oracle."""
    import torch
    from paper_2410_10759_b200 import _native as N, batch as B
    insts = _dense_rows_instances(17, 6)
    off = np.zeros(len(insts) + 1, np.int64)
    np.cumsum([len(x["r"]) for x in insts], out=off[1:])
    cat = lambda k: np.concatenate([x[k] for x in insts])
    b = B.InstanceBatch.from_arrays(off, cat("i"), cat("s"), cat("u"), cat("d"), cat("r"),
                                    [x["budget"] for x in insts], [x["sac"] for x in insts])
    lib = N.library()
    if ws_kind == "large":
        host = B.plan_dp(b).to_host()
        assert lib.sp_last_dense_fallbacks() > 0, "expected some instances to outgrow the lists"
    else:
        mn, _full = B.dp_workspace_bytes(b)
        ws = torch.empty(mn, dtype=torch.uint8, device=N.device())
        out = B.PolicyBatch.empty(b.n, b.total_layers, b.r.device)
        rc = lib.sp_plan_dp(b.struct(), out.struct(), N.ptr(ws), mn, N.stream_ptr())
        assert rc == 0, lib.sp_last_error()
        host = out.to_host()
    for k, inst in enumerate(insts):
        exp = O.plan_dp(inst)
        got = dict(pi=host["pi"][off[k]:off[k + 1]], client_value=host["client_value"][k],
                   server_load=host["server_load"][k], integer_latency=host["integer_latency"][k],
                   feasible=host["feasible"][k])
        assert_policy(got, dict(exp, pi=tuple(exp["pi"])), f"{ws_kind}[{k}]")


# ---------------------------------------------------------------------------
# sp_plan_dp_async / sp_plan_dp_finish


@pytest.mark.parametrize("name", BATTERIES + ["battery_large_model"])
def test_plan_dp_async_matches_reference(gpu, name):
    """The two-half call gives the reference's results on every battery (the
    batteries mix instances tier 1 solves with ones the host-planned tiers
    take in finish())."""
    from paper_2410_10759_b200 import batch as B
    bat = Battery(name)
    pend = B.plan_dp_async(_batch(bat))
    _compare(bat, "dp", pend.finish().to_host())


def test_plan_dp_async_fallbacks_and_two_in_flight(gpu):
    """Two batches in flight on one stream with their own workspaces, the
    second queued before the first is finished; the batches need the wide
    tier and the dense kernels (run by finish()).  Bit-exact vs the oracle."""
    import torch
    from paper_2410_10759_b200 import _native as N, batch as B
    sets = [_dense_rows_instances(17, 6), _dense_rows_instances(23, 5)]
    batches, offs = [], []
    for insts in sets:
        off = np.zeros(len(insts) + 1, np.int64)
        np.cumsum([len(x["r"]) for x in insts], out=off[1:])
        cat = lambda k: np.concatenate([x[k] for x in insts])
        batches.append(B.InstanceBatch.from_arrays(off, cat("i"), cat("s"), cat("u"), cat("d"), cat("r"),
                                                   [x["budget"] for x in insts], [x["sac"] for x in insts]))
        offs.append(off)
    _mn, full = B.dp_workspace_bytes(batches[0])
    big = max(full, B.dp_workspace_bytes(batches[1])[1])
    ws = [torch.empty(big, dtype=torch.uint8, device=N.device()) for _ in range(2)]
    p0 = B.plan_dp_async(batches[0], ws=ws[0])
    p1 = B.plan_dp_async(batches[1], ws=ws[1])
    hosts = [p0.finish().to_host(), p1.finish().to_host()]
    for insts, off, host in zip(sets, offs, hosts):
        for k, inst in enumerate(insts):
            exp = O.plan_dp(inst)
            got = dict(pi=host["pi"][off[k]:off[k + 1]], client_value=host["client_value"][k],
                       server_load=host["server_load"][k], integer_latency=host["integer_latency"][k],
                       feasible=host["feasible"][k])
            assert_policy(got, dict(exp, pi=tuple(exp["pi"])), f"async[{k}]")


def test_engine_solve_async_pipelined(gpu):
    """Engine.solve_async with two batches in flight gives exactly Engine.solve's results."""
    import torch
    from paper_2410_10759_b200 import _native as N, cost_model as cm, workloads as W
    from paper_2410_10759_b200.requests import Engine, RequestBatch
    eng = Engine([cm.build_preset("gpt2-24", 128).layers])
    reqs = [RequestBatch.from_numpy(**W.cfg2(300, seed)[0]).to(N.device()) for seed in (5, 6, 7)]
    ref = [eng.solve(r).policies.to_host() for r in reqs]
    ws = [torch.empty(512 << 20, dtype=torch.uint8, device=N.device()) for _ in range(2)]
    prev, got = None, []
    for k, r in enumerate(reqs + [None]):
        cur = eng.solve_async(r, ws=ws[k & 1]) if r is not None else None
        if prev is not None:
            got.append(prev.result().policies.to_host_async())
        prev = cur
    torch.cuda.synchronize()
    for a, b in zip(ref, got):
        for key in ("pi", "client_value", "server_load", "integer_latency", "feasible", "status"):
            np.testing.assert_array_equal(a[key], getattr(b, key).numpy(), err_msg=key)


# ---------------------------------------------------------------------------
# tier 0: the SMEM kernel's instances planned on the device


def _tier0_instances(seed, n):
    """Narrow instances over the tier-0 classes: integral r (int32 domain) at
    widths in all three int32 configurations, float r (fp64 domain) at the
    four fp64 widths (the NaN domain's narrow instances are in the inf-r
    batteries)."""
    rng = np.random.default_rng(seed)
    w_int, w_f64 = [300, 1500, 3000, 6000, 14000], [300, 700, 1500, 2500, 6000, 11000]
    out = []
    for t in range(n):
        kind = t % 5
        widths = w_int if kind < 3 else w_f64
        W = widths[(t // 5) % len(widths)] + int(rng.integers(0, 200))
        L = int(rng.integers(4, 24))
        hi = max(2, W // 6)
        r = rng.integers(0, 9, L).astype(float) if kind < 3 else rng.random(L) * 7
        out.append(dict(i=rng.integers(0, hi, L), s=rng.integers(0, hi, L), u=rng.integers(0, hi, L),
                        d=rng.integers(0, hi, L), r=r, budget=int(W), sac=bool(t % 2)))
    return out


@pytest.mark.parametrize("case", ["tier0_one", "tier0_several", "tier1_several"])
def test_device_planned_tiers_in_waves(gpu, case, capfd, monkeypatch):
    """1,300 narrow instances (six counting blocks) over every tier-0 class:
    the device-planned SMEM tier (breakpoint lists held back) in one wave and
    in several waves of a workspace holding about a third of their
    back-pointer tables; and the default -- tier 1 (breakpoint lists) in waves
    of consecutive instances.  Every
    placement bit-exact against the oracle, nothing left to host planning."""
    import torch
    from paper_2410_10759_b200 import _native as N, batch as B
    insts = _tier0_instances(29, 1300)
    off = np.zeros(len(insts) + 1, np.int64)
    np.cumsum([len(x["r"]) for x in insts], out=off[1:])
    cat = lambda k: np.concatenate([x[k] for x in insts])
    b = B.InstanceBatch.from_arrays(off, cat("i"), cat("s"), cat("u"), cat("d"), cat("r"),
                                    [x["budget"] for x in insts], [x["sac"] for x in insts])
    lib = N.library()
    if case.startswith("tier0"):  # breakpoint lists held back
        monkeypatch.setenv("SPLITPLAN_STEPS_MIN_COLS", str(1 << 30))
        monkeypatch.setenv("SPLITPLAN_NO_TIER1_WAVES", "1")
    mn, full = B.dp_workspace_bytes(b)
    size = full + (1 << 20) if case == "tier0_one" else mn + (full - mn) // 3
    ws = torch.empty(size, dtype=torch.uint8, device=N.device())
    out = B.PolicyBatch.empty(b.n, b.total_layers, b.r.device)
    monkeypatch.setenv("SPLITPLAN_TRACE", "1")
    rc = lib.sp_plan_dp(b.struct(), out.struct(), N.ptr(ws), size, N.stream_ptr())
    assert rc == 0, lib.sp_last_error()
    host = out.to_host()
    err = capfd.readouterr().err
    t0, t1 = err.count("tier-0 wave"), err.count("tier-1 wave")
    if case == "tier0_one":
        assert t0 == 1 and t1 == 0, err[-2000:]
    elif case == "tier0_several":
        assert t0 >= 2 and t1 == 0, err[-2000:]
    else:  # (every row of these is tier 1's by default)
        assert t1 >= 2, err[-2000:]
    assert "items planned" not in err  # nothing left for the host-planned tiers
    for k, inst in enumerate(insts):
        exp = O.plan_dp(inst)
        got = dict(pi=host["pi"][off[k]:off[k + 1]], client_value=host["client_value"][k],
                   server_load=host["server_load"][k], integer_latency=host["integer_latency"][k],
                   feasible=host["feasible"][k])
        assert_policy(got, dict(exp, pi=tuple(exp["pi"])), f"{case}[{k}]")


def test_engine_pipelined_host_requests_and_results(gpu):
    """The pipelined public path bench.py's e2e leg times: host request
    parameters uploaded into reused slots on the engine's copy stream,
    results copied out there (result_to_host), three batches through two
    slots -- exactly Engine.solve's results."""
    import torch
    from paper_2410_10759_b200 import _native as N, cost_model as cm, workloads as W
    from paper_2410_10759_b200.requests import Engine, RequestBatch
    eng = Engine([cm.build_preset("gpt2-24", 128).layers])
    hosts = [RequestBatch.from_numpy(pin=True, **W.cfg2(400, seed)[0]) for seed in (11, 12, 13, 14)]
    ref = [eng.solve(h.to(N.device())).policies.to_host() for h in hosts]
    total = 400 * 98
    slots = [eng.solve_slot(400, total, 512 << 20) for _ in range(2)]
    prev, got = None, []
    for k, h in enumerate(hosts + [None]):
        cur = eng.solve_async(h, total, slot=slots[k & 1]) if h is not None else None
        if prev is not None:
            _s, host, done = prev.result_to_host()
            got.append((host, done))
        prev = cur
    for (host, done), r in zip(got, ref):
        done.synchronize()
        for key in ("pi", "client_value", "server_load", "integer_latency", "feasible", "status"):
            np.testing.assert_array_equal(r[key], getattr(host, key).numpy().astype(r[key].dtype), err_msg=key)


def test_tier1_waves_skip_an_instance_too_large_for_a_wave(gpu, capfd, monkeypatch):
    """With the minimum workspace, a 1,500-stage instance's breakpoint store
    (1,501 x 3 KB) exceeds what a wave may use: tier 1 runs the small ones in
    waves and leaves it, flagged, to the dense kernels (tier 0).  All
    placements bit-exact against the oracle."""
    import torch
    from paper_2410_10759_b200 import _native as N, batch as B
    rng = np.random.default_rng(41)
    insts = []
    for t in range(40):
        L, W = (1500, 600) if t == 17 else (12, 900)
        insts.append(dict(i=rng.integers(0, 60, L), s=rng.integers(0, 60, L), u=rng.integers(0, 60, L),
                          d=rng.integers(0, 60, L), r=rng.integers(0, 9, L).astype(float), budget=W,
                          sac=bool(t % 2)))
    off = np.zeros(len(insts) + 1, np.int64)
    np.cumsum([len(x["r"]) for x in insts], out=off[1:])
    cat = lambda k: np.concatenate([x[k] for x in insts])
    b = B.InstanceBatch.from_arrays(off, cat("i"), cat("s"), cat("u"), cat("d"), cat("r"),
                                    [x["budget"] for x in insts], [x["sac"] for x in insts])
    mn, _full = B.dp_workspace_bytes(b)
    lib = N.library()
    ws = torch.empty(mn, dtype=torch.uint8, device=N.device())
    out = B.PolicyBatch.empty(b.n, b.total_layers, b.r.device)
    monkeypatch.setenv("SPLITPLAN_TRACE", "1")
    rc = lib.sp_plan_dp(b.struct(), out.struct(), N.ptr(ws), mn, N.stream_ptr())
    assert rc == 0, lib.sp_last_error()
    err = capfd.readouterr().err
    assert "tier-1 wave" in err and ("tier-0 wave 1" in err or "items planned" in err), err[-1500:]
    host = out.to_host()
    for k, inst in enumerate(insts):
        exp = O.plan_dp(inst)
        got = dict(pi=host["pi"][off[k]:off[k + 1]], client_value=host["client_value"][k],
                   server_load=host["server_load"][k], integer_latency=host["integer_latency"][k],
                   feasible=host["feasible"][k])
        assert_policy(got, dict(exp, pi=tuple(exp["pi"])), f"big[{k}]")
