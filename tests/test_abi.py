"""The C-ABI library builds for sm_100a, loads without a GPU, and exports
every entry point include/splitplan_b200.h declares (no compute calls)."""

from __future__ import annotations

import ctypes
import re
import subprocess

from conftest import ROOT

HEADER = ROOT / "include" / "splitplan_b200.h"


def declared_functions() -> list[str]:
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|void|size_t|const char\s*\*)\s*(sp_\w+)\s*\(",
                                 text, flags=re.M)))


def test_header_declares_the_hot_path():
    fns = declared_functions()
    for name in ("sp_plan_dp", "sp_build_dp_tables", "sp_plan_prefix", "sp_plan_exhaustive",
                 "sp_effective_budget", "sp_build_cost_table", "sp_integerize_profiles",
                 "sp_latency_eq1", "sp_sim_replay", "sp_to_units", "sp_segment_sum",
                 "sp_evaluate_policy", "sp_last_error"):
        assert name in fns


def test_library_exports_every_declared_symbol():
    from paper_2410_10759_b200 import _native
    lib = _native.library()
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing
    # and the Python binding knows every signature
    assert set(declared_functions()) <= set(_native.SIGNATURES)


def test_library_is_sm100a_and_abi_version():
    from paper_2410_10759_b200 import _native
    from paper_2410_10759_b200._build import LIB
    assert _native.library().sp_abi_version() == 4
    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout, out.stdout


def test_error_state_without_gpu_calls():
    from paper_2410_10759_b200 import _native
    lib = _native.library()
    # argument validation happens before any CUDA call
    rc = lib.sp_plan_prefix(None, 0, None, None)
    assert rc == _native.SP_ERR_INVALID
    assert b"null instance batch" in lib.sp_last_error()
    rc = lib.sp_to_units(None, 1, ctypes.c_double(1e-3), 0, None, None, None)
    assert rc == _native.SP_ERR_INVALID


def test_onewave_bytes_is_host_arithmetic():
    """sp_plan_dp_onewave_bytes needs no device: the fixed part plus one
    breakpoint store (2 rows x (8 + 8 x 192) bytes) per stage and instance."""
    from paper_2410_10759_b200 import _native
    lib = _native.library()
    assert lib.sp_plan_dp_onewave_bytes(0, 0) == 0
    a = lib.sp_plan_dp_onewave_bytes(10_000, 980_000)
    b = lib.sp_plan_dp_onewave_bytes(20_000, 1_960_000)
    assert a >= (980_000 + 10_000) * 2 * (8 + 8 * 192)
    assert a % 256 == 0 and b > 1.9 * a


def test_skeleton_arguments_validated_without_gpu():
    from paper_2410_10759_b200 import _native
    lib = _native.library()
    rc = lib.sp_sim_skeletons(None, None, None, 4, 10, ctypes.c_double(1.0), 10, None, None, None, None, None)
    assert rc == _native.SP_ERR_INVALID
    rc = lib.sp_sim_skeletons(None, None, None, 0, 10, ctypes.c_double(1.0), 0, None, None, None, None, None)
    assert rc == _native.SP_ERR_INVALID  # exec_max < 1
    assert lib.sp_sim_skeletons(None, None, None, 0, 10, ctypes.c_double(1.0), 10, None, None, None, None,
                                None) == 0
