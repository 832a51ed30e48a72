"""Model configuration and parameters in the reference layout.

`GnnConfig` mirrors model.hpp:19-27 (presets model.cpp:17-41). Parameters are
one flat fp64 vector in ModelParams::for_each order (model.cpp:124-135); the
MP-layer block is what the device engine consumes.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N


@dataclass
class GnnConfig:
    name: str = "custom"
    hidden_dim: int = 8
    num_mp_layers: int = 4
    mlp_hidden_layers: int = 2
    in_node_dim: int = 3
    in_edge_dim: int = 7
    out_dim: int = 3
    mode: str = "na2a"

    @staticmethod
    def small_model(mode: str = "na2a") -> "GnnConfig":
        return GnnConfig("small", 8, 4, 2, mode=mode)

    @staticmethod
    def large_model(mode: str = "na2a") -> "GnnConfig":
        return GnnConfig("large", 32, 4, 5, mode=mode)

    def dims(self):
        return (self.hidden_dim, self.num_mp_layers, self.mlp_hidden_layers, self.in_node_dim, self.in_edge_dim,
                self.out_dim)


def param_count(cfg: GnnConfig) -> int:
    n = N.LIB.hgnn_param_count(*cfg.dims())
    if n < 0:
        N.check(2)
    return n


def init_params(cfg: GnnConfig, seed: int) -> np.ndarray:
    """init_params(config, seed) (model.cpp:105-122), for_each order, fp64."""
    out = np.empty(param_count(cfg), dtype=np.float64)
    N.check(N.LIB.hgnn_init_params(*cfg.dims(), seed, out.ctypes.data_as(N.f64p)))
    return out


def mp_param_range(cfg: GnnConfig) -> tuple[int, int]:
    off, cnt = C.c_int64(), C.c_int64()
    N.check(N.LIB.hgnn_mp_param_range(cfg.hidden_dim, cfg.num_mp_layers, cfg.mlp_hidden_layers, cfg.in_node_dim,
                                      cfg.in_edge_dim, C.byref(off), C.byref(cnt)))
    return off.value, cnt.value


def mp_params(cfg: GnnConfig, full: np.ndarray) -> np.ndarray:
    off, cnt = mp_param_range(cfg)
    return np.ascontiguousarray(full[off:off + cnt])


def mlp_param_count(in_dim: int, hidden: int, k: int) -> int:
    """Processor-MLP size (nn.cpp:28-36, no skip / output LN)."""
    return in_dim * hidden + hidden + k * (hidden * hidden + hidden) + hidden * hidden + hidden


def mp_layer_slices(cfg: GnnConfig):
    """(name, start, stop) of every MP tensor inside the MP block, for_each order."""
    H, k = cfg.hidden_dim, cfg.mlp_hidden_layers
    out, off = [], 0
    for m in range(cfg.num_mp_layers):
        for which, in_dim in (("edge_update", 3 * H), ("node_update", 2 * H)):
            for l in range(k + 2):
                rows = in_dim if l == 0 else H
                out.append((f"layer{m}.{which}.w{l}", off, off + rows * H))
                off += rows * H
                out.append((f"layer{m}.{which}.b{l}", off, off + H))
                off += H
    return out


def model_slices(cfg: "GnnConfig"):
    """(name, start, stop) of every tensor of the full ModelParams::for_each
    vector (model.cpp:124-135, nn.cpp:38-46): encoders (+ skip, ln_g, ln_b),
    MP layers, decoder (+ skip)."""
    H, k = cfg.hidden_dim, cfg.mlp_hidden_layers
    out, off = [], 0

    def mlp(prefix, in_dim, out_dim, skip, ln):
        nonlocal off
        for l in range(k + 2):
            rows = in_dim if l == 0 else H
            cols = out_dim if l == k + 1 else H
            out.append((f"{prefix}.w{l}", off, off + rows * cols))
            off += rows * cols
            out.append((f"{prefix}.b{l}", off, off + cols))
            off += cols
        if skip:
            out.append((f"{prefix}.skip", off, off + in_dim * out_dim))
            off += in_dim * out_dim
        if ln:
            out.append((f"{prefix}.ln_g", off, off + out_dim))
            off += out_dim
            out.append((f"{prefix}.ln_b", off, off + out_dim))
            off += out_dim

    mlp("node_encoder", cfg.in_node_dim, H, True, True)
    mlp("edge_encoder", cfg.in_edge_dim, H, True, True)
    for m in range(cfg.num_mp_layers):
        mlp(f"layer{m}.edge_update", 3 * H, H, False, False)
        mlp(f"layer{m}.node_update", 2 * H, H, False, False)
    mlp("node_decoder", H, cfg.out_dim, True, False)
    return out
