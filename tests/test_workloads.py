"""Host-side checks of the seeded config generators (no GPU): determinism,
shapes, and the budget widths SURVEY.md 8(d) specifies, via the oracle."""

from __future__ import annotations

import numpy as np

from oracle import splitplan_oracle as O
from paper_2410_10759_b200 import workloads as W


def _inst(req, layers, k):
    lay = [dict(kind=l.kind.value, hidden_dim=l.hidden_dim, heads=l.heads, ffn_dim=l.ffn_dim,
                out_dim=l.out_dim, seq_divisor=l.seq_divisor) for l in layers[int(req["model"][k])]]
    r, cs, ss, tau = O.profile_arrays(lay, int(req["seq_len"][k]), req["client_fps"][k],
                                      req["server_fps"][k])
    return O.instance_from_profile(r, cs, ss, tau, req["uplink_bps"][k], req["downlink_bps"][k],
                                   req["propagation_s"][k], req["deadline_s"][k], req["unit_s"][k])


def test_generators_are_deterministic():
    a, _ = W.cfg2(64, seed=7)
    b, _ = W.cfg2(64, seed=7)
    for k in a:
        assert np.array_equal(a[k], b[k])
    c, _, off = W.cfg4([3, 3])
    assert np.array_equal(c["seq_len"][:64], c["seq_len"][64:]) and list(off) == [0, 64, 128]


def test_cfg1_shape():
    req, layers = W.cfg1()
    assert len(req["seq_len"]) == 1200 and len(layers[0]) == 50
    assert req["seq_len"].min() >= 128 and req["seq_len"].max() <= 2048


def test_cfg2_budget_is_1e5_columns():
    req, layers = W.cfg2(40)
    assert len(layers[0]) == 98
    for k in range(0, 40, 7):
        inst = _inst(req, layers, k)
        assert inst["budget"] == 100_000 and O.effective_budget(inst) == 100_000


def test_cfg3_llama_shape_and_budget():
    req, layers = W.cfg3(200)
    assert len(layers[0]) == 130
    assert req["seq_len"].max() <= 32768 and req["seq_len"].min() >= 512
    for k in range(0, 200, 40):
        assert _inst(req, layers, k)["budget"] <= 10_000


def test_cfg4_grid():
    assert W.cfg4_scenario(0) == (0, 0, 0) and W.cfg4_scenario(65535) == (15, 15, 255)
    req, layers, off = W.cfg4([0, 1, 300])
    assert len(layers) == 3 and off[-1] == 3 * 64
    assert set(np.unique(req["model"])) <= {0, 1, 2}


def test_lexsort_device_equals_numpy():
    """The Monte-Carlo table sort (successive stable sorts, here on the CPU
    device) is np.lexsort's permutation, ties and float keys included."""
    import torch
    from paper_2410_10759_b200 import montecarlo as MC
    rng = np.random.default_rng(5)
    n = 50_000
    keys = (rng.choice([3e7, 1e8, 1e9], n), rng.choice([3e7, 2e8], n), rng.random(n).round(2),
            rng.integers(128, 4096, n), rng.integers(0, 3, n), np.repeat(np.arange(n // 64 + 1), 64)[:n])
    assert np.array_equal(np.lexsort(keys), MC.lexsort_device(keys, device=torch.device("cpu")))


def test_cfg4_device_expansion_is_bitwise_cfg4():
    """The Monte-Carlo grid expanded on a device (here the CPU device) equals
    the host generator field by field, bit for bit."""
    import torch  # noqa: F401
    sids = np.arange(0, 65536, 97)
    req, _l, off = W.cfg4(sids)
    rb, _l2, off2 = W.cfg4_device(sids, "cpu")
    assert np.array_equal(off, off2)
    for k, v in req.items():
        a, b = np.asarray(v), getattr(rb, k).numpy()
        assert a.dtype == b.dtype, k
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), k
