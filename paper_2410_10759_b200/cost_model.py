"""Analytic per-layer cost model -- drop-in for `splitplan.cost_model`.

`profile()` (cost_model.py:305-329), the per-(request, layer) hot loop, runs
in the K1 cost-table kernel; the scalar helpers below (`flop_of_layer`,
`memory_of_layer`, `output_bytes`, `model_flops`, `calibrate`) are exact
Python-int API conveniences used for device calibration and by callers that
inspect single layers.  The closed forms are those of cost_model.py:137-192.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from enum import Enum
from pathlib import Path
from typing import Sequence

import numpy as np
import torch

from . import _native as N

BYTES_PER_ELEMENT = 4
SOFTMAX_FLOPS_PER_SCORE = 5

__all__ = ["LayerKind", "LayerSpec", "ModelSpec", "DeviceSpec", "LayerProfile", "PRESET_NAMES",
           "build_preset", "flop_of_layer", "memory_of_layer", "output_bytes", "raw_input_bytes",
           "model_flops", "profile", "profile_many", "calibrate", "profile_to_dict",
           "profile_from_dict", "save_profile", "load_profile", "load_model_spec",
           "encode_models"]


class LayerKind(str, Enum):
    EMBEDDING = "embedding"
    ATTENTION = "attention"
    FEED_FORWARD = "feed_forward"
    LAYER_NORM = "layer_norm"
    CLASSIFIER = "classifier"
    CUSTOM = "custom"


@dataclass(frozen=True)
class LayerSpec:
    """One splittable model entry (cost_model.py:52-86).  Custom entries carry
    (quad, lin, const) polynomials in the effective sequence length."""

    kind: LayerKind
    hidden_dim: int
    heads: int = 1
    ffn_dim: int = 0
    out_dim: int = 0
    seq_divisor: int = 1
    flop_coeffs: tuple[float, float, float] | None = None
    mem_coeffs: tuple[float, float, float] | None = None
    out_bytes_per_token: float | None = None

    def __post_init__(self):
        problems = [
            (self.hidden_dim <= 0, f"hidden_dim must be positive, got {self.hidden_dim}"),
            (self.heads <= 0 or self.seq_divisor <= 0, "heads and seq_divisor must be positive"),
            (self.kind is LayerKind.FEED_FORWARD and self.ffn_dim <= 0,
             "feed_forward layers need a positive ffn_dim"),
            (self.kind is LayerKind.CLASSIFIER and self.out_dim <= 0,
             "classifier layers need a positive out_dim"),
            (self.kind is LayerKind.CUSTOM and self.flop_coeffs is None,
             "custom layers must supply flop_coeffs"),
        ]
        for bad, msg in problems:
            if bad:
                raise ValueError(msg)


@dataclass(frozen=True)
class ModelSpec:
    name: str
    layers: tuple[LayerSpec, ...]
    seq_len: int

    def __post_init__(self):
        if not self.layers:
            raise ValueError("model must have at least one layer")
        if self.seq_len < 1:
            raise ValueError(f"seq_len must be >= 1, got {self.seq_len}")
        object.__setattr__(self, "layers", tuple(self.layers))

    @property
    def attention_count(self) -> int:
        return sum(l.kind is LayerKind.ATTENTION for l in self.layers)


@dataclass(frozen=True)
class DeviceSpec:
    name: str
    flops_per_s: float

    def __post_init__(self):
        if not self.flops_per_s > 0:
            raise ValueError(f"throughput must be positive, got {self.flops_per_s}")


@dataclass(frozen=True)
class LayerProfile:
    """Cost metric r, device times and input-tensor bytes of one layer."""

    index: int
    kind: str
    r: float
    client_time_s: float
    server_time_s: float
    tau_bytes: float


# ---------------------------------------------------------------------------
# scalar closed forms (exact Python ints for the derived kinds)


def _s_eff(layer: LayerSpec, seq_len: int) -> int:
    return max(1, seq_len // layer.seq_divisor)


def _quadratic(coeffs, s):
    a, b, c = coeffs
    return a * s * s + b * s + c


def flop_of_layer(layer: LayerSpec, seq_len: int):
    s, d = _s_eff(layer, seq_len), layer.hidden_dim
    k = layer.kind
    if k is LayerKind.ATTENTION:
        return 8 * s * d * d + 4 * s * s * d + SOFTMAX_FLOPS_PER_SCORE * s * s * layer.heads
    if k is LayerKind.FEED_FORWARD:
        return 4 * s * d * layer.ffn_dim
    if k is LayerKind.LAYER_NORM:
        return 5 * s * d
    if k is LayerKind.EMBEDDING:
        return 2 * s * d
    if k is LayerKind.CLASSIFIER:
        return 2 * s * d * layer.out_dim
    return _quadratic(layer.flop_coeffs, s)


def memory_of_layer(layer: LayerSpec, seq_len: int):
    s = _s_eff(layer, seq_len)
    if layer.kind is LayerKind.CUSTOM:
        return _quadratic(layer.mem_coeffs or (0.0, BYTES_PER_ELEMENT * layer.hidden_dim, 0.0), s)
    extra = s * s * layer.heads * BYTES_PER_ELEMENT if layer.kind is LayerKind.ATTENTION else 0
    return s * layer.hidden_dim * BYTES_PER_ELEMENT + extra


def output_bytes(layer: LayerSpec, seq_len: int):
    s = _s_eff(layer, seq_len)
    if layer.kind is LayerKind.CLASSIFIER:
        return layer.out_dim * BYTES_PER_ELEMENT
    if layer.kind is LayerKind.CUSTOM and layer.out_bytes_per_token is not None:
        return layer.out_bytes_per_token * s
    return s * layer.hidden_dim * BYTES_PER_ELEMENT


def raw_input_bytes(spec: ModelSpec) -> int:
    return spec.seq_len * BYTES_PER_ELEMENT


def model_flops(spec: ModelSpec, seq_len: int | None = None):
    s = spec.seq_len if seq_len is None else seq_len
    return sum(flop_of_layer(l, s) for l in spec.layers)


# ---------------------------------------------------------------------------
# presets (cost_model.py:204-287)

_PRESET_DIMS = {  # d, heads, d_ff, vocab, encoder blocks
    "bert-12": (768, 12, 3072, 30522, 12),
    "gpt2-24": (1024, 16, 4096, 50257, 24),
}


def _block(d, h, f, div=1, decoder=False):
    A = lambda: LayerSpec(LayerKind.ATTENTION, d, heads=h, seq_divisor=div)
    LN = lambda: LayerSpec(LayerKind.LAYER_NORM, d, seq_divisor=div)
    FF = LayerSpec(LayerKind.FEED_FORWARD, d, ffn_dim=f, seq_divisor=div)
    if decoder:  # self-attention, cross-attention, feed-forward, each + norm
        return [A(), LN(), A(), LN(), FF, LN()]
    return [A(), LN(), FF, LN()]


def _encoder_only(name):
    d, h, f, v, nb = _PRESET_DIMS[name]
    body = [x for _ in range(nb) for x in _block(d, h, f)]
    return [LayerSpec(LayerKind.EMBEDDING, d, out_dim=v), *body,
            LayerSpec(LayerKind.CLASSIFIER, d, out_dim=v)]


def _vanilla():
    d, h, f, v = 512, 8, 2048, 32000
    enc = [x for _ in range(6) for x in _block(d, h, f)]
    dec = [x for _ in range(6) for x in _block(d, h, f, decoder=True)]
    return [LayerSpec(LayerKind.EMBEDDING, d, out_dim=v), *enc, *dec,
            LayerSpec(LayerKind.CLASSIFIER, d, out_dim=v)]


def _cmt():
    out = [LayerSpec(LayerKind.EMBEDDING, 64)]
    for stage, (d, h) in enumerate(((64, 1), (128, 2), (256, 4), (512, 8))):
        div = 4 ** stage
        if stage:
            out.append(LayerSpec(LayerKind.EMBEDDING, d, seq_divisor=div))
        out += _block(d, h, 4 * d, div) + _block(d, h, 4 * d, div)
    out.append(LayerSpec(LayerKind.CLASSIFIER, 512, out_dim=1000, seq_divisor=64))
    return out


_PRESETS = {"vanilla-6x6": _vanilla, "bert-12": lambda: _encoder_only("bert-12"),
            "gpt2-24": lambda: _encoder_only("gpt2-24"), "cmt-like": _cmt}
PRESET_NAMES = tuple(sorted(_PRESETS))


def build_preset(name: str, seq_len: int) -> ModelSpec:
    if name not in _PRESETS:
        raise ValueError(f"unknown preset {name!r}; known: {', '.join(PRESET_NAMES)}")
    if seq_len < 1:
        raise ValueError(f"seq_len must be >= 1, got {seq_len}")
    return ModelSpec(name, tuple(_PRESETS[name]()), seq_len)


def calibrate(spec: ModelSpec, seq_len: int, target_total_time_s: float,
              name: str = "calibrated") -> DeviceSpec:
    """Device rate that makes the whole model take the target time (cost_model.py:294-302)."""
    if target_total_time_s <= 0:
        raise ValueError("target_total_time_s must be positive")
    total = model_flops(spec, seq_len)
    if total <= 0:
        raise ValueError(f"model {spec.name!r} has zero total FLOPs; cannot calibrate")
    return DeviceSpec(name, total / target_total_time_s)


# ---------------------------------------------------------------------------
# GPU encoding + profile


def encode_models(layer_lists: Sequence[Sequence[LayerSpec]], dev=None) -> tuple[N.SpModels, dict]:
    """CSR encoding of model layer lists for the K1 kernel (sp_models)."""
    dev = dev or N.device()
    flat = [l for layers in layer_lists for l in layers]
    off = np.zeros(len(layer_lists) + 1, dtype=np.int64)
    np.cumsum([len(x) for x in layer_lists], out=off[1:])
    col = lambda f, dt: N.to_dev(np.array([f(l) for l in flat], dtype=dt), _TORCH[dt], dev)
    coef = lambda c: [float(v) for v in c] if c is not None else [0.0, 0.0, 0.0]
    t = dict(
        off=N.to_dev(off, torch.int64, dev),
        kind=col(lambda l: N.KIND_CODE[LayerKind(l.kind).value], np.int32),
        d=col(lambda l: l.hidden_dim, np.int64), h=col(lambda l: l.heads, np.int64),
        f=col(lambda l: l.ffn_dim, np.int64), v=col(lambda l: l.out_dim, np.int64),
        div=col(lambda l: l.seq_divisor, np.int64),
        fc=N.to_dev(np.array([coef(l.flop_coeffs) for l in flat], dtype=np.float64).ravel(),
                    torch.float64, dev),
        mc=N.to_dev(np.array([coef(l.mem_coeffs) for l in flat], dtype=np.float64).ravel(),
                    torch.float64, dev),
        hm=col(lambda l: l.mem_coeffs is not None, np.uint8),
        ob=col(lambda l: float(l.out_bytes_per_token or 0.0), np.float64),
        ho=col(lambda l: l.out_bytes_per_token is not None, np.uint8),
    )
    s = N.SpModels(len(layer_lists), *[N.ptr(t[k]).value for k in
                                       ("off", "kind", "d", "h", "f", "v", "div", "fc", "mc",
                                        "hm", "ob", "ho")])
    return s, t


_TORCH = {np.int32: torch.int32, np.int64: torch.int64, np.float64: torch.float64,
          np.uint8: torch.uint8}


def profile_many(specs: Sequence[ModelSpec], clients: Sequence[DeviceSpec],
                 servers: Sequence[DeviceSpec], metric: str = "flop") -> list[list[LayerProfile]]:
    """Batched `profile`: one K1 launch for many (model, seq_len, devices)."""
    if metric not in ("flop", "memory"):
        raise ValueError(f"metric must be 'flop' or 'memory', got {metric!r}")
    dev = N.device()
    n = len(specs)
    models, keep = encode_models([s.layers for s in specs], dev)
    f64 = lambda vals: N.to_dev(np.asarray(vals, dtype=np.float64), torch.float64, dev)
    req_t = dict(model=N.to_dev(np.arange(n, dtype=np.int32), torch.int32, dev),
                 seq=N.to_dev(np.array([s.seq_len for s in specs], np.int64), torch.int64, dev),
                 cf=f64([c.flops_per_s for c in clients]), sf=f64([c.flops_per_s for c in servers]),
                 fl=N.to_dev(np.full(n, N.SP_REQ_METRIC_MEMORY if metric == "memory" else 0,
                                     np.uint8), torch.uint8, dev))
    req = N.SpRequests(n, N.ptr(req_t["model"]).value, N.ptr(req_t["seq"]).value,
                       N.ptr(req_t["cf"]).value, N.ptr(req_t["sf"]).value, None, None, None, None,
                       None, N.ptr(req_t["fl"]).value)
    off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    N.check(N.library().sp_request_layer_offsets(models, req, N.ptr(off), N.stream_ptr()),
            "sp_request_layer_offsets")
    total = sum(len(s.layers) for s in specs)
    o = {k: torch.empty(total, dtype=torch.float64, device=dev) for k in ("r", "c", "s", "t")}
    tab = N.SpCostTable(N.ptr(off).value, total, N.ptr(o["r"]).value, N.ptr(o["c"]).value,
                        N.ptr(o["s"]).value, N.ptr(o["t"]).value, None, None, None, None, None,
                        None, None, None, None, None)
    N.check(N.library().sp_build_cost_table(models, req, 0, tab, N.stream_ptr()),
            "sp_build_cost_table")
    h = {k: v.cpu().numpy() for k, v in o.items()}
    offs = off.cpu().numpy()
    out = []
    for m, spec in enumerate(specs):
        a = offs[m]
        out.append([LayerProfile(index=k, kind=spec.layers[k].kind.value, r=float(h["r"][a + k]),
                                 client_time_s=float(h["c"][a + k]),
                                 server_time_s=float(h["s"][a + k]),
                                 tau_bytes=float(h["t"][a + k]))
                    for k in range(len(spec.layers))])
    del keep
    return out


def profile(spec: ModelSpec, client: DeviceSpec, server: DeviceSpec,
            metric: str = "flop") -> list[LayerProfile]:
    """Per-layer r, device times and input bytes (cost_model.py:305-329), on the GPU."""
    return profile_many([spec], [client], [server], metric)[0]


# ---------------------------------------------------------------------------
# serialization (cost_model.py:336-401)


def profile_to_dict(spec: ModelSpec, layers: Sequence[LayerProfile], metric: str) -> dict:
    keys = ("index", "kind", "r", "client_time_s", "server_time_s", "tau_bytes")
    return {"model": spec.name, "seq_len": spec.seq_len, "metric": metric,
            "layers": [{k: getattr(p, k) for k in keys} for p in layers]}


def profile_from_dict(doc: dict) -> list[LayerProfile]:
    return [LayerProfile(int(e["index"]), str(e["kind"]), float(e["r"]), float(e["client_time_s"]),
                         float(e["server_time_s"]), float(e["tau_bytes"])) for e in doc["layers"]]


def save_profile(path, spec: ModelSpec, layers: Sequence[LayerProfile], metric: str) -> None:
    Path(path).write_text(json.dumps(profile_to_dict(spec, layers, metric), indent=2,
                                     sort_keys=True) + "\n")


def load_profile(path) -> tuple[dict, list[LayerProfile]]:
    doc = json.loads(Path(path).read_text())
    return doc, profile_from_dict(doc)


def load_model_spec(source: str, seq_len: int) -> ModelSpec:
    """A preset name or a model-spec JSON file -> ModelSpec."""
    if source in _PRESETS:
        return build_preset(source, seq_len)
    path = Path(source)
    if not path.exists():
        raise ValueError(f"{source!r} is neither a preset nor a model-spec file")
    doc = json.loads(path.read_text())
    layers = []
    for entry in doc["layers"]:
        kw = dict(entry)
        kind = LayerKind(kw.pop("kind"))
        for key in ("flop_coeffs", "mem_coeffs"):
            if kw.get(key) is not None:
                kw[key] = tuple(float(v) for v in kw[key])
        layers.append(LayerSpec(kind=kind, **kw))
    return ModelSpec(str(doc.get("name", path.stem)), tuple(layers), seq_len)
