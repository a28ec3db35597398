"""Seeded synthetic workloads of BASELINE.json's configs.

Each generator returns host numpy arrays in the `sp_requests` layout
(`RequestBatch.from_numpy(**arrays)`) plus the model table they index, so the
same inputs feed the CUDA engine (`requests.Engine`), the CPU oracle in the
tests, and `bench.py`.  Nothing here touches the GPU.

    cfg1  bert-12, 100 mixed-length requests x 4 SLAs x 3 links      (configs[0])
    cfg2  gpt2-24, 10k requests, W_eff = 1e5 budget columns           (configs[1])
    cfg3  Llama-2-7B-like (L = 130), long sequences, W = 1e4          (configs[2])
    cfg4  Monte-Carlo scenario grid: 16 SLA scales x 16 bandwidths x
          256 workload-mix seeds, 64 requests each                     (configs[3])
    cfg5  one chain of L = 1e5 stages x W = 1e7 budget columns        (configs[4])

Device calibration follows the reference acceptance suite: client 7.727 s and
server 0.0979 s for bert-12 at 4096 tokens (`test_acceptance.py:23-52`).
"""

from __future__ import annotations

import math

import numpy as np

from . import cost_model as cm
from .cost_model import LayerKind, LayerSpec

CLIENT_S, SERVER_S = 7.727, 0.0979
PROP_S = 0.01
SOURCE_CLIENT = 2  # sp_request_flags SP_REQ_SOURCE_CLIENT


def calibrated_rates() -> tuple[float, float]:
    """cost_model.calibrate on bert-12 @ 4096 (cost_model.py:294-302)."""
    ref = cm.build_preset("bert-12", 4096)
    return (cm.calibrate(ref, 4096, CLIENT_S).flops_per_s,
            cm.calibrate(ref, 4096, SERVER_S).flops_per_s)


def llama2_7b_layers() -> tuple[LayerSpec, ...]:
    """Llama-2-7B-like chain from the reference's layer kinds (L = 130):
    embedding, 32 x (attention, norm, feed-forward, norm), classifier."""
    d, h, f, v = 4096, 32, 11008, 32000
    block = [LayerSpec(LayerKind.ATTENTION, d, heads=h), LayerSpec(LayerKind.LAYER_NORM, d),
             LayerSpec(LayerKind.FEED_FORWARD, d, ffn_dim=f), LayerSpec(LayerKind.LAYER_NORM, d)]
    return (LayerSpec(LayerKind.EMBEDDING, d, out_dim=v), *[x for _ in range(32) for x in block],
            LayerSpec(LayerKind.CLASSIFIER, d, out_dim=v))


def model_layers(name: str):
    if name == "llama2-7b":
        return llama2_7b_layers()
    return cm.build_preset(name, 128).layers


def _total_flops(layers, seq_len: int) -> int:
    return sum(cm.flop_of_layer(l, int(seq_len)) for l in layers)


def _total_flops_many(layers, seqs) -> np.ndarray:
    """float(_total_flops(layers, s)) for every s in `seqs`: the closed forms
    of cost_model.flop_of_layer in exact int64 arithmetic (every term and sum
    stays far below 2^63 for these models), one numpy pass per layer; models
    with custom (possibly float) entries take the scalar path."""
    seqs = np.asarray(seqs, dtype=np.int64)
    if any(l.kind is cm.LayerKind.CUSTOM for l in layers):
        return np.array([_total_flops(layers, int(x)) for x in seqs], dtype=float)
    tot = np.zeros(seqs.shape, dtype=np.int64)
    for l in layers:
        s, d = np.maximum(1, seqs // l.seq_divisor), int(l.hidden_dim)
        k = l.kind
        if k is cm.LayerKind.ATTENTION:
            tot += 8 * s * d * d + 4 * s * s * d + cm.SOFTMAX_FLOPS_PER_SCORE * s * s * int(l.heads)
        elif k is cm.LayerKind.FEED_FORWARD:
            tot += 4 * s * d * int(l.ffn_dim)
        elif k is cm.LayerKind.LAYER_NORM:
            tot += 5 * s * d
        elif k is cm.LayerKind.EMBEDDING:
            tot += 2 * s * d
        else:  # classifier
            tot += 2 * s * d * int(l.out_dim)
    return tot.astype(np.float64)


def _requests(model, seq, cfps, sfps, up, down, deadline, unit, flags=SOURCE_CLIENT) -> dict:
    n = len(seq)
    full = lambda v: np.full(n, v, dtype=np.float64) if np.isscalar(v) else np.asarray(v, np.float64)
    return dict(model=np.asarray(model, np.int32), seq_len=np.asarray(seq, np.int64),
                client_fps=full(cfps), server_fps=full(sfps), uplink_bps=full(up),
                downlink_bps=full(down), propagation_s=full(PROP_S), deadline_s=full(deadline),
                unit_s=full(unit), flags=np.full(n, flags, np.uint8))


def cfg1(seed: int = 1) -> tuple[dict, list]:
    """100 bert-12 requests (seq = round(2^U(7,11))) x deadlines {1, 1/2, 1/4, 1/8}
    of the request's all-client time x links {3e7, 2e8, 1e9} bit/s; unit 1 ms."""
    cfps, sfps = calibrated_rates()
    layers = model_layers("bert-12")
    rng = np.random.default_rng(seed)
    seqs = np.rint(2.0 ** rng.uniform(7, 11, 100)).astype(np.int64)
    rows = []
    for s in seqs:
        t_client = _total_flops(layers, s) / cfps
        for frac in (1.0, 0.5, 0.25, 0.125):
            for bw in (3e7, 2e8, 1e9):
                rows.append((s, frac * t_client, bw))
    seq, dl, bw = (np.array(c) for c in zip(*rows))
    return _requests(np.zeros(len(seq)), seq, cfps, sfps, bw, bw, dl, 1e-3), [layers]


def cfg2(n: int = 10_000, seed: int = 2) -> tuple[dict, list]:
    """gpt2-24, seq ~ U{128..2048}, symmetric links log-U[3e7, 1e9], deadline =
    f x all-client time (f ~ U(0.05, 1)), unit = deadline / 1e5 -> W = 1e5."""
    cfps, sfps = calibrated_rates()
    layers = model_layers("gpt2-24")
    rng = np.random.default_rng(seed)
    seq = rng.integers(128, 2049, n)
    bw = np.exp(rng.uniform(math.log(3e7), math.log(1e9), n))
    f = rng.uniform(0.05, 1.0, n)
    flops = np.array([_total_flops(layers, s) for s in seq], dtype=float)
    deadline = f * flops / cfps
    return _requests(np.zeros(n), seq, cfps, sfps, bw, bw.copy(), deadline, deadline / 1e5), [layers]


def cfg3(n: int = 1_000_000, seed: int = 3) -> tuple[dict, list]:
    """Llama-2-7B-like, seq = round(2^U(9,15)) (<= 32,768), up = down log-U[1e7,
    1e10], deadline uniform between the all-server and all-client latencies,
    unit = deadline / 1e4 -> W = 1e4."""
    cfps, sfps = calibrated_rates()
    layers = model_layers("llama2-7b")
    rng = np.random.default_rng(seed)
    seq = np.rint(2.0 ** rng.uniform(9, 15, n)).astype(np.int64)
    bw = np.exp(rng.uniform(math.log(1e7), math.log(1e10), n))
    u = rng.uniform(0.0, 1.0, n)
    uniq, inv = np.unique(seq, return_inverse=True)
    flops = np.array([_total_flops(layers, s) for s in uniq], dtype=float)[inv]
    t_client = flops / cfps
    # all-server: raw input (4 B/token) up the link, then every layer on the server
    t_server = flops / sfps + 8.0 * 4.0 * seq / bw + PROP_S
    lo, hi = np.minimum(t_server, t_client), np.maximum(t_server, t_client)
    deadline = lo + u * (hi - lo)
    return _requests(np.zeros(n), seq, cfps, sfps, bw, bw.copy(), deadline, deadline / 1e4), [layers]


CFG4_MODELS = ("bert-12", "gpt2-24", "vanilla-6x6")
CFG4_SCALES = 2.0 ** np.linspace(-3.0, 0.0, 16)           # deadline / all-client time
CFG4_BANDWIDTHS = np.exp(np.linspace(math.log(3e7), math.log(1e9), 16))
CFG4_MIXES = 256
CFG4_REQUESTS = 64


def cfg4_scenario(sid: int) -> tuple[int, int, int]:
    """scenario id -> (deadline-scale index, bandwidth index, workload-mix seed)."""
    return (sid // 16) % 16, sid % 16, sid // 256


def _cfg4_mix(mix: int):
    rng = np.random.default_rng(1_000_003 * mix + 4)
    m = rng.integers(0, len(CFG4_MODELS), CFG4_REQUESTS)
    s = np.rint(2.0 ** rng.uniform(7, 12, CFG4_REQUESTS)).astype(np.int64)
    return m, s


def cfg4(scenarios=None) -> tuple[dict, list, np.ndarray]:
    """Requests of the Monte-Carlo grid: scenario sid has 64 requests, model
    uniform over bert-12 / gpt2-24 / vanilla-6x6, seq = round(2^U(7,12)),
    deadline = scale x the request's all-client time, symmetric bandwidth, unit
    1 ms.  The workload mix depends only on the mix seed, so the 256 mixes are
    drawn once and broadcast over the SLA x bandwidth grid.  Returns
    (requests, model layer lists, scenario offsets [S+1])."""
    cfps, sfps = calibrated_rates()
    sids = np.arange(16 * 16 * CFG4_MIXES) if scenarios is None else np.asarray(scenarios, dtype=np.int64)
    layer_lists = [model_layers(m) for m in CFG4_MODELS]
    a, b, mix = (sids // 16) % 16, sids % 16, sids // 256
    uniq, inv = np.unique(mix, return_inverse=True)
    drawn = [_cfg4_mix(int(x)) for x in uniq]
    um, us = np.stack([d[0] for d in drawn]), np.stack([d[1] for d in drawn])
    # total FLOPs of every (model, seq) pair the mixes draw, once per pair
    uf = np.empty(um.shape)
    for mi in range(len(CFG4_MODELS)):
        sel = um == mi
        vals, back = np.unique(us[sel], return_inverse=True)
        uf[sel] = _total_flops_many(layer_lists[mi], vals)[back]
    M, S, F = um[inv], us[inv], uf[inv]
    dl = CFG4_SCALES[a][:, None] * F / cfps
    bw = np.repeat(CFG4_BANDWIDTHS[b], CFG4_REQUESTS)
    off = np.arange(len(sids) + 1, dtype=np.int64) * CFG4_REQUESTS
    return (_requests(M.ravel(), S.ravel(), cfps, sfps, bw, bw.copy(), dl.ravel(), 1e-3), layer_lists,
            off)


def cfg4_device(scenarios, device):
    """cfg4 built on `device`: the 256 workload mixes are drawn on the host
    (numpy, as `cfg4`), the grid's 4.2M requests are expanded from them on the
    device -- the same values bit for bit (the deadline is the same IEEE
    product and quotient).  Returns (RequestBatch on `device`, model layer
    lists, scenario offsets [S+1] on the host)."""
    import torch
    from . import _native as N
    from .requests import RequestBatch, _req_layout
    cfps, sfps = calibrated_rates()
    sids = np.asarray(scenarios, dtype=np.int64)
    layer_lists = [model_layers(m) for m in CFG4_MODELS]
    a, b, mix = (sids // 16) % 16, sids % 16, sids // 256
    uniq, inv = np.unique(mix, return_inverse=True)
    drawn = [_cfg4_mix(int(x)) for x in uniq]
    um, us = np.stack([d[0] for d in drawn]), np.stack([d[1] for d in drawn])
    uf = np.empty(um.shape)
    for mi in range(len(CFG4_MODELS)):
        sel = um == mi
        vals, back = np.unique(us[sel], return_inverse=True)
        uf[sel] = _total_flops_many(layer_lists[mi], vals)[back]
    dev = torch.device(device)
    t = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x)).to(dev, dt)
    inv_d = t(inv.astype(np.int64), torch.int64)
    n = len(sids) * CFG4_REQUESTS
    _buf, v = N.packed(_req_layout(n), dev)
    v["model"].view(-1, CFG4_REQUESTS).copy_(t(um, torch.int32)[inv_d])
    v["seq_len"].view(-1, CFG4_REQUESTS).copy_(t(us, torch.int64)[inv_d])
    # (the divisor as a device tensor: PyTorch's CUDA division by a Python
    # scalar multiplies by its reciprocal, which is not numpy's quotient)
    prod = t(CFG4_SCALES, torch.float64)[t(a, torch.int64)][:, None] * t(uf, torch.float64)[inv_d]
    torch.div(prod, torch.full((1, 1), cfps, dtype=torch.float64, device=dev).expand_as(prod),
              out=v["deadline_s"].view(-1, CFG4_REQUESTS))
    bw = t(CFG4_BANDWIDTHS, torch.float64)[t(b, torch.int64)][:, None].expand(-1, CFG4_REQUESTS)
    v["uplink_bps"].view(-1, CFG4_REQUESTS).copy_(bw)
    v["downlink_bps"].view(-1, CFG4_REQUESTS).copy_(bw)
    for k, val in (("client_fps", cfps), ("server_fps", sfps), ("propagation_s", PROP_S), ("unit_s", 1e-3),
                   ("flags", SOURCE_CLIENT)):
        v[k].fill_(val)
    req = RequestBatch(**v)
    req._buf = _buf
    off = np.arange(len(sids) + 1, dtype=np.int64) * CFG4_REQUESTS
    return req, layer_lists, off


def cfg5(L: int = 100_000, W: int = 10_000_000, seed: int = 5) -> dict:
    """configs[4]: one huge chain via PlanProblem.from_costs (problem.py:179-185):
    i, s, u, d ~ U{0..200}, r ~ U{0..100} (integral floats), source at the
    client, budget W.  The worst path exceeds W, so W_eff = W.  Returns the
    CSR instance arrays of `batch.InstanceBatch.from_arrays`."""
    rng = np.random.default_rng(seed)
    i, s, u, d = (rng.integers(0, 201, L) for _ in range(4))
    r = rng.integers(0, 101, L).astype(np.float64)
    return dict(layer_off=np.array([0, L], dtype=np.int64), i=i, s=s, u=u, d=d, r=r,
                budget=np.array([W], dtype=np.int64), sac=np.array([1], dtype=np.uint8))
