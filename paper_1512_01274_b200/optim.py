"""Momentum SGD on device (optim.py:1-78 in the reference).

    v <- momentum * v - eta * (g + weight_decay * w);  w <- w + v

as five separately rounded fp32 steps in the reference's order:
tmp = g + w*wd; v = v*mom; v = v + tmp*(-eta); w = w + v*1.
``sgd_step`` is the tensor path (one fused kernel, ``mgx_sgd_step``);
``make_sgd_updater`` returns the KVStore updater, which the store recognises
and fuses into its reduce kernel (identical float sequence, so server-side
and local updates agree bit for bit).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Dict

import numpy as np

from . import _lib as L
from .errors import ArgumentError
from .tensor import Tensor


@dataclass(frozen=True)
class SGDConfig:
    eta: float
    momentum: float = 0.0
    weight_decay: float = 0.0

    def __post_init__(self):
        if not self.eta > 0:
            raise ArgumentError("learning rate must be > 0")
        if not 0 <= self.momentum < 1:
            raise ArgumentError("momentum must be in [0, 1)")
        if self.weight_decay < 0:
            raise ArgumentError("weight decay must be >= 0")


def _f32(x: float) -> float:
    return float(np.float32(x))


def sgd_step(w: Tensor, g: Tensor, v: Tensor, tmp: Tensor, cfg: SGDConfig) -> None:
    """Enqueue one update.  ``tmp`` is accepted for API compatibility
    (optim.py:39-50); the fused kernel keeps the scratch in registers."""
    for t in (g, v, tmp):
        if t.shape != w.shape:
            raise ArgumentError("sgd_step: all tensors must share one shape")
    eng = w.engine
    eng.push(lambda: L.call("mgx_sgd_step", w.ptr, g.ptr, v.ptr, w.size, _f32(cfg.eta),
                            _f32(cfg.momentum), _f32(cfg.weight_decay), eng.stream_handle),
             reads=[g.tag], writes=[w.tag, v.tag], label="sgd")


def sgd_arrays(w, g, v, cfg: SGDConfig) -> None:
    """Device-array mirror (optim.py:53-61): w, g, v are fp32 CUDA torch
    tensors; same float sequence as ``sgd_step``."""
    from .engine import current_stream
    L.call("mgx_sgd_step", w.data_ptr(), g.data_ptr(), v.data_ptr(), w.numel(), _f32(cfg.eta),
           _f32(cfg.momentum), _f32(cfg.weight_decay), current_stream())


def make_sgd_updater(cfg: SGDConfig, scale: int = 1):
    """KVStore updater: g = incoming * f32(1/scale), then the SGD sequence
    with per-key momentum (optim.py:64-78).  Carries ``_mgx_sgd`` so the
    device store runs it inside the fused reduce kernel."""
    state: Dict[int, object] = {}

    def updater(key: int, stored, incoming) -> None:
        import torch
        from .engine import current_stream
        v = state.get(key)
        if v is None:
            v = state[key] = torch.zeros_like(stored)
        g = torch.empty_like(incoming)
        L.call("mgx_scalar_op", 1, incoming.data_ptr(), _f32(1.0 / scale), g.data_ptr(),
               g.numel(), current_stream())
        sgd_arrays(stored, g, v, cfg)

    updater._mgx_sgd = (cfg, scale)
    return updater
