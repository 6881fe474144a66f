"""Model configs, FTCN weight files, models and run reports.

Mirrors the reference's on-disk and wire formats so a user of the reference can bring
their files unchanged:

* model config JSON -- ``parse_model_config`` / ``load_model_config``
  (model.hpp:12-44, model_io.cpp:14-76): same fields, defaults and validation
  (element type, non-empty, groups divide channels/kernels, integral extents, layer
  chain E_k == H_{k+1}, M_k == Ch_{k+1}, equal batch), ConfigError / IoError;
* FTCN weight files -- ``save_weights`` / ``load_weights`` (model_io.cpp:78-174):
  magic "FTCN", version 1, layer count, then per layer {M, Ckw, R, R, bias} u32 LE and
  the FP32 LE kernels then bias; byte-identical to the reference's writer, and the same
  truncation / magic / dims / non-finite checks on read;
* ``random_weights`` (model_io.cpp:176-192) and ``random_input`` (Tensor4::random,
  tensor.hpp:57-66) -- std::mt19937_64 + uniform_real_distribution<double> inside the
  library, so seeded weights and inputs are the reference's bit for bit;
* ``build_model`` (model.hpp:81-117) -> :class:`Model`, one :class:`ProtectedConv` per
  layer (golden weights uploaded and their kernel checksums precomputed on device);
* run reports -- ``report_to_json`` for protected runs and campaigns
  (serialize.cpp:157-193; keys sorted, 2-space indent, trailing newline).

The element type is FP32 on this engine; an "f64" model parses (it is a valid
reference config) but ``build_model`` refuses it with ConfigError.
"""
from __future__ import annotations

import json
import math
import re
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from .campaign import Model as _ChainModel
from .ftconv import ConfigError, ConvParams, IoError, ShapeError

MAGIC = b"FTCN"
VERSION = 1


def default_tau(f64: bool) -> float:
    """workflow.hpp:19"""
    return 1e-10 if f64 else 1e-4


# ----------------------------------------------------------------------------- configs
@dataclass
class LayerConfig:
    """model.hpp:14-33"""
    name: str = ""
    batch: int = 1
    channels: int = 1
    height: int = 1
    kernels: int = 1
    kernel_size: int = 1
    stride: int = 1
    pad: int = 0
    groups: int = 1
    bias: bool = False

    def params(self) -> ConvParams:
        return ConvParams(stride=self.stride, pad=self.pad, groups=self.groups, bias_enabled=self.bias)

    @property
    def ckw(self) -> int:
        return self.channels // self.groups


@dataclass
class ModelConfig:
    """model.hpp:36-41"""
    name: str = "model"
    element_type: str = "f32"
    tau: float = 0.0
    layers: list = field(default_factory=list)


def _size(v, what):
    # nlohmann get<std::size_t>(): integers (floats truncate); strings, bools, null throw
    if isinstance(v, bool) or not isinstance(v, (int, float)):
        raise ConfigError(f"malformed config: {what} must be a number")
    if isinstance(v, float):
        if not math.isfinite(v):
            raise ConfigError(f"malformed config: {what} must be finite")
        v = int(v)
    if v < 0:
        raise ConfigError(f"malformed config: {what} must be non-negative")
    return v


def _extent(H: int, R: int, stride: int, pad: int) -> int:
    """tensor.hpp:100-107 (ConfigError unless a positive integer)."""
    Hp = H + 2 * pad
    if stride == 0:
        raise ConfigError("stride must be positive")
    if Hp < R:
        raise ConfigError("kernel larger than padded input")
    if (Hp - R) % stride:
        raise ConfigError("output extent (H+2p-R+U)/U is not an integer")
    return (Hp - R) // stride + 1


def _parse_layer(j) -> LayerConfig:
    """model_io.cpp:14-27"""
    if not isinstance(j, dict):
        raise ConfigError("malformed config: layer is not an object")
    try:
        name = j["name"]
        if not isinstance(name, str):
            raise ConfigError("malformed config: layer name must be a string")
        lc = LayerConfig(name=name,
                         batch=_size(j["batch"], "batch"), channels=_size(j["channels"], "channels"),
                         height=_size(j["height"], "height"), kernels=_size(j["kernels"], "kernels"),
                         kernel_size=_size(j["kernel_size"], "kernel_size"),
                         stride=_size(j.get("stride", 1), "stride"), pad=_size(j.get("pad", 0), "pad"),
                         groups=_size(j.get("groups", 1), "groups"))
    except KeyError as e:
        raise ConfigError(f"malformed config: key {e} not found")
    bias = j.get("bias", False)
    if not isinstance(bias, bool):
        raise ConfigError("malformed config: bias must be a boolean")
    lc.bias = bias
    return lc


def parse_model_config(text: str) -> ModelConfig:
    """model_io.cpp:29-69"""
    try:
        j = json.loads(text)
    except (ValueError, TypeError) as e:
        raise ConfigError(f"config is not valid JSON: {e}")
    if not isinstance(j, dict):
        raise ConfigError("malformed config: not an object")
    cfg = ModelConfig()
    name, et, tau = j.get("name", "model"), j.get("element_type", "f32"), j.get("tau", 0.0)
    if not isinstance(name, str) or not isinstance(et, str):
        raise ConfigError("malformed config: name / element_type must be strings")
    if isinstance(tau, bool) or not isinstance(tau, (int, float)):
        raise ConfigError("malformed config: tau must be a number")
    cfg.name, cfg.element_type, cfg.tau = name, et, float(tau)
    if "layers" not in j:
        raise ConfigError("malformed config: key 'layers' not found")
    if not isinstance(j["layers"], list):
        raise ConfigError("malformed config: layers must be an array")
    cfg.layers = [_parse_layer(lj) for lj in j["layers"]]
    if cfg.element_type not in ("f32", "f64"):
        raise ConfigError("element_type must be f32 or f64")
    if not cfg.layers:
        raise ConfigError("config has no layers")
    for i, lc in enumerate(cfg.layers):
        if lc.groups == 0 or lc.channels % lc.groups or lc.kernels % lc.groups:
            raise ConfigError(f"groups must divide channels and kernels in {lc.name}")
        E = _extent(lc.height, lc.kernel_size, lc.stride, lc.pad)
        if i + 1 < len(cfg.layers):
            nx = cfg.layers[i + 1]
            if E != nx.height:
                raise ConfigError(f"layer chain broken: extent of {lc.name} does not match height of {nx.name}")
            if lc.kernels != nx.channels:
                raise ConfigError(f"layer chain broken: kernels of {lc.name} do not match channels of {nx.name}")
            if lc.batch != nx.batch:
                raise ConfigError(f"layer chain broken: batch mismatch at {nx.name}")
    return cfg


def load_model_config(path: str) -> ModelConfig:
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise IoError(f"cannot open config file: {path}")
    return parse_model_config(text)


# ----------------------------------------------------------------------------- weights
@dataclass
class RawLayerWeights:
    """model.hpp:45-48: FP32 kernels (M*Ckw*R*R) and bias (M or empty)."""
    kernel: np.ndarray
    bias: np.ndarray


def mt64_uniform(seed: int, n: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """std::mt19937_64(seed) + uniform_real_distribution<double>(lo, hi), n draws."""
    out = np.empty(n, np.float64)
    st = _abi.lib().ftc_mt64_uniform(seed & 0xFFFFFFFFFFFFFFFF, lo, hi, n, out.ctypes.data if n else None)
    if st:
        raise ConfigError("mt64_uniform: bad arguments")
    return out


def random_weights(cfg: ModelConfig, seed: int) -> list:
    """model_io.cpp:176-192: one generator over all layers, kernels then bias."""
    sizes = []
    for lc in cfg.layers:
        sizes.append((lc.kernels * lc.ckw * lc.kernel_size ** 2, lc.kernels if lc.bias else 0))
    draws = mt64_uniform(seed, sum(a + b for a, b in sizes)).astype(np.float32)
    out, o = [], 0
    for nk, nb in sizes:
        out.append(RawLayerWeights(draws[o:o + nk].copy(), draws[o + nk:o + nk + nb].copy()))
        o += nk + nb
    return out


def random_input(lc: LayerConfig, seed: int) -> np.ndarray:
    """Tensor4<float>::random(batch, channels, height, height, seed) (tensor.hpp:57-66)."""
    shape = (lc.batch, lc.channels, lc.height, lc.height)
    return mt64_uniform(seed, int(np.prod(shape))).astype(np.float32).reshape(shape)


def weights_to_bytes(cfg: ModelConfig, w: list) -> bytes:
    """model_io.cpp:105-131"""
    if len(w) != len(cfg.layers):
        raise ConfigError("weight layer count does not match config")
    parts = [MAGIC, struct.pack("<II", VERSION, len(cfg.layers))]
    for lc, lw in zip(cfg.layers, w):
        parts.append(struct.pack("<5I", lc.kernels, lc.ckw, lc.kernel_size, lc.kernel_size, 1 if lc.bias else 0))
        k = np.ascontiguousarray(lw.kernel, np.float32).reshape(-1)
        b = np.ascontiguousarray(lw.bias, np.float32).reshape(-1)
        if k.size != lc.kernels * lc.ckw * lc.kernel_size ** 2:
            raise ConfigError(f"kernel element count mismatch in layer {lc.name}")
        if b.size != (lc.kernels if lc.bias else 0):
            raise ConfigError(f"bias element count mismatch in layer {lc.name}")
        parts.append(k.astype("<f4").tobytes())
        parts.append(b.astype("<f4").tobytes())
    return b"".join(parts)


def save_weights(path: str, cfg: ModelConfig, w: list) -> None:
    blob = weights_to_bytes(cfg, w)
    try:
        with open(path, "wb") as f:
            f.write(blob)
    except OSError:
        raise IoError(f"cannot open weight file for writing: {path}")


def weights_from_bytes(blob: bytes, cfg: ModelConfig, path: str = "<bytes>") -> list:
    """model_io.cpp:133-174"""
    if len(blob) < 4 or blob[:4] != MAGIC:
        raise IoError(f"bad weight file magic (expected FTCN): {path}")
    o = 4

    def u32():
        nonlocal o
        if o + 4 > len(blob):
            raise IoError("weight file truncated while reading header")
        v = struct.unpack_from("<I", blob, o)[0]
        o += 4
        return v

    if u32() != VERSION:
        raise IoError("unsupported weight file version")
    layers = u32()
    if layers != len(cfg.layers):
        raise ConfigError(f"weight file holds {layers} layers, config expects {len(cfg.layers)}")
    out = []
    for lc in cfg.layers:
        M, ckw, r0, r1, bias = (u32() for _ in range(5))
        if M != lc.kernels or ckw != lc.ckw or r0 != lc.kernel_size or r1 != lc.kernel_size or (bias != 0) != lc.bias:
            raise ConfigError(f"weight file dims disagree with config at layer {lc.name}")
        nk, nb = M * ckw * r0 * r1, (M if bias else 0)
        nbytes = (nk + nb) * 4
        if o + nbytes > len(blob):
            raise IoError(f"weight file truncated: expected {nbytes} more bytes in layer {lc.name}")
        vals = np.frombuffer(blob, "<f4", nk + nb, o).astype(np.float32)
        o += nbytes
        k, b = vals[:nk].copy(), vals[nk:].copy()
        if not np.isfinite(k).all():
            raise ConfigError(f"non-finite kernel value in {lc.name}")
        if not np.isfinite(b).all():
            raise ConfigError(f"non-finite bias value in {lc.name}")
        out.append(RawLayerWeights(k, b))
    return out


def load_weights(path: str, cfg: ModelConfig) -> list:
    try:
        with open(path, "rb") as f:
            blob = f.read()
    except OSError:
        raise IoError(f"cannot open weight file: {path}")
    return weights_from_bytes(blob, cfg, path)


# ----------------------------------------------------------------------------- models
class Model(_ChainModel):
    """model.hpp:50-117: golden weights per layer on the device (kernel checksums
    precomputed by each layer handle, model.hpp:104), tau = config tau or the default.
    A chain of ProtectedConv layers (campaign.Model), so run_campaign takes it as is."""

    def __init__(self, cfg: ModelConfig, raw: list):
        if len(raw) != len(cfg.layers):
            raise ConfigError("weight file layer count does not match config")
        if cfg.element_type != "f32":
            raise ConfigError("element_type f64 is not supported by the B200 engine (FP32 tensor cores)")
        self.cfg = cfg
        self.tau = cfg.tau if cfg.tau > 0 else default_tau(cfg.element_type == "f64")
        specs, self.extents = [], []
        for lc, rw in zip(cfg.layers, raw):
            k = np.ascontiguousarray(rw.kernel, np.float32)
            if k.size != lc.kernels * lc.ckw * lc.kernel_size ** 2:
                raise ConfigError(f"kernel element count mismatch in layer {lc.name}")
            b = None
            if lc.bias:
                b = np.ascontiguousarray(rw.bias, np.float32)
                if b.size != lc.kernels:
                    raise ConfigError(f"bias element count mismatch in layer {lc.name}")
            if not np.isfinite(k).all() or (b is not None and not np.isfinite(b).all()):
                raise ConfigError(f"non-finite weights in layer {lc.name}")
            specs.append((k.reshape(lc.kernels, lc.ckw, lc.kernel_size, lc.kernel_size), b, lc.params()))
            self.extents.append(_extent(lc.height, lc.kernel_size, lc.stride, lc.pad))
        l0 = cfg.layers[0]
        super().__init__(specs, l0.batch, l0.height)
        self.names = [lc.name for lc in cfg.layers]


def build_model(cfg: ModelConfig, raw: list) -> Model:
    return Model(cfg, raw)


# ----------------------------------------------------------------------------- reports
# nlohmann's dump(2) prints each corrected block -- pushed as a 2-element initializer
# list (serialize.cpp:163) -- on one line, "[i,j]"; json.dumps would expand it
_BLK = "@@ftc-block@@"
_BLK_RE = re.compile(r'"' + _BLK + r'(\[\d+,\d+\])' + _BLK + '"')


def _dump(obj) -> str:
    return _BLK_RE.sub(r"\1", json.dumps(obj, indent=2, sort_keys=True)) + "\n"


def _layer_report_obj(r, timings: bool) -> dict:
    """serialize.cpp:157-172"""
    j = {"layer": r.layer, "detected": bool(r.detected), "stage": r.stage,
         "weights_reloaded": bool(r.weights_reloaded), "recomputed": bool(r.recomputed),
         "corrected_blocks": [f"{_BLK}[{int(b[0])},{int(b[1])}]{_BLK}" for b in r.corrected_blocks],
         "stages_attempted": list(r.stages_attempted)}
    if timings:
        j["timings"] = {k: float(v) for k, v in r.timings.items()}
    return j


def report_to_json(reports, timings: bool = False) -> str:
    """serialize.cpp:174-180: {"layers": [...]}"""
    return _dump({"layers": [_layer_report_obj(r, timings) for r in reports]})


def campaign_report_to_json(rep, timings: bool = False) -> str:
    """serialize.cpp:182-193"""
    j = {"runs": rep.runs, "detected": rep.detected, "above_threshold": rep.above_threshold,
         "recovered": rep.recovered, "ground_truth_mismatches": rep.ground_truth_mismatches,
         "integrity_fatals": rep.integrity_fatals, "by_stage": dict(rep.by_stage),
         "entries": [_layer_report_obj(e, timings) for e in rep.entries]}
    return _dump(j)


__all__ = ["LayerConfig", "ModelConfig", "RawLayerWeights", "Model", "parse_model_config", "load_model_config",
           "save_weights", "load_weights", "weights_to_bytes", "weights_from_bytes", "random_weights",
           "random_input", "mt64_uniform", "build_model", "report_to_json", "campaign_report_to_json",
           "default_tau", "ShapeError"]
