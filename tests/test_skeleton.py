"""The device skeleton generator's restatement of numpy's default_rng stream
(csrc/np_random.cuh), built for the host with g++ and checked against numpy
itself -- the generator the reference's simulator draws with
(throughput_sim.py:179-186) -- on CPU: SeedSequence + PCG64 seeding,
glibc's log1p (the ziggurat tail), and whole skeletons (exponential gaps,
np.cumsum, Lemire-bounded integers).  The GPU suite runs the same header on
the device (tests/test_gpu_montecarlo.py)."""

from __future__ import annotations

import ctypes as C
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

SRC = ROOT / "tests" / "tools" / "np_random_host.cpp"


@pytest.fixture(scope="module")
def nr(tmp_path_factory):
    so = tmp_path_factory.mktemp("nr") / "np_random_host.so"
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-shared", "-fPIC", "-o", str(so), str(SRC)], check=True)
    lib = C.CDLL(str(so))
    lib.nr_seed_state.argtypes = [C.c_uint64, C.c_void_p]
    lib.nr_pcg_state.argtypes = [C.c_uint64, C.c_void_p]
    lib.nr_log1p_many.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
    lib.nr_skeleton.argtypes = [C.c_uint64, C.c_int64, C.c_double, C.c_int64, C.c_int64, C.c_int64,
                                C.c_void_p, C.c_void_p, C.c_void_p]
    return lib


SEEDS = [0, 1, 2, 7, 255, 65535, 12345, 2 ** 31, 2 ** 32 - 1, 2 ** 32, 2 ** 40 + 7, 2 ** 63 - 1]


def test_ziggurat_tables_are_the_installed_numpys():
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "gen_np_ziggurat.py"), "--check"])
    assert r.returncode == 0, "np_ziggurat.inc differs from the installed numpy's tables: regenerate it"


@pytest.mark.parametrize("seed", SEEDS)
def test_seed_sequence_and_pcg64_seeding(nr, seed):
    out = np.zeros(4, dtype=np.uint64)
    nr.nr_seed_state(seed, out.ctypes.data)
    assert np.array_equal(out, np.random.SeedSequence(seed).generate_state(4, np.uint64))
    nr.nr_pcg_state(seed, out.ctypes.data)
    st = np.random.PCG64(seed).state["state"]
    assert (int(out[0]) << 64 | int(out[1])) == st["state"]
    assert (int(out[2]) << 64 | int(out[3])) == st["inc"]


def test_log1p_restatement_is_the_host_libm(nr):
    """The tail draw is r - log1p(-u) with u = next_double; numpy's
    distributions call the host libm's log1p there (log1p@GLIBC_2.2.5), so the
    restatement must equal it for every u (and small magnitudes)."""
    nr.nr_libm_log1p_many.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
    rng = np.random.default_rng(3)
    u = rng.integers(0, 2 ** 53, 2_000_000, dtype=np.int64).astype(np.float64) * 2.0 ** -53
    x = np.concatenate([-u, -np.ldexp(u[:500_000], -rng.integers(0, 60, 500_000)), u[:200_000] * 5,
                        [0.0, -0.0, -0.5, -2.0 ** -29, -2.0 ** -54, -0.2928932188134524, -1 + 2 ** -53]])
    y = np.empty_like(x)
    ref = np.empty_like(x)
    nr.nr_log1p_many(x.ctypes.data, y.ctypes.data, len(x))
    nr.nr_libm_log1p_many(x.ctypes.data, ref.ctypes.data, len(x))
    assert np.array_equal(y.view(np.int64), ref.view(np.int64))


def _numpy_skeleton(seed, horizon, beta, lo, hi, exec_max):
    g = np.random.default_rng(seed)
    arr = np.cumsum(g.exponential(scale=1.0 / beta, size=horizon))
    ch = g.integers(0, hi - lo, size=horizon) + lo
    ex = g.integers(1, exec_max + 1, size=horizon)
    return arr, ch, ex


def test_skeletons_equal_numpy_draws(nr):
    """1,500 seeds x 2,000 requests (about 1,300 ziggurat tail draws), table
    ranges from 1 row (no draw) to 2^32 (raw 32-bit draws)."""
    horizon, beta = 2000, 0.057
    spans = [1, 2, 3, 64, 1000, 2 ** 31 + 11, 2 ** 32]
    for seed in range(1500):
        span = spans[seed % len(spans)]
        lo = seed % 5
        arr = np.empty(horizon)
        ch = np.empty(horizon, np.int64)
        ex = np.empty(horizon, np.int64)
        nr.nr_skeleton(seed, horizon, 1.0 / beta, lo, lo + span, 10, arr.ctypes.data, ch.ctypes.data,
                       ex.ctypes.data)
        ra, rc, re_ = _numpy_skeleton(seed, horizon, beta, lo, lo + span, 10)
        assert np.array_equal(arr.view(np.int64), ra.view(np.int64)), seed
        assert np.array_equal(ch, rc), seed
        assert np.array_equal(ex, re_), seed
