"""Adam on the device — lseforge::AdamState (adam.hpp:11-49, adam.cpp:8-55):
the optimizer that consumes dE (and the encoder's gradients) after the loss.

Float parameters, double moments, the reference's update arithmetic rounded
once per operation in its order (lf_adam_step), so parameters match the
reference bit for bit after any number of steps.  ``step`` can also refresh a
bf16 shadow of a parameter (the E the next CCE call reads) in the same pass.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import torch

from . import _capi
from .cce import _stream


@dataclass
class AdamConfig:
    """adam.hpp:11-16."""
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8


_SHADOW = {torch.bfloat16: _capi.LF_BF16, torch.float32: _capi.LF_F32}
_GRAD = {torch.float32: _capi.LF_F32, torch.float64: _capi.LF_F64}


class DeviceAdam:
    """AdamState over a list of float32 CUDA parameter tensors (any layout;
    the update is elementwise)."""

    def __init__(self, params: Sequence[torch.Tensor], cfg: AdamConfig = AdamConfig()):
        if not params or any(p.numel() == 0 for p in params):  # adam.cpp:11-13
            raise ValueError("adam: catalog and hidden must be >= 1")
        if not (0.0 <= cfg.beta1 < 1.0 and 0.0 <= cfg.beta2 < 1.0):  # adam.cpp:14-16
            raise ValueError("adam: betas must lie in [0, 1)")
        if not cfg.eps > 0.0:  # adam.cpp:17-19
            raise ValueError("adam: eps must be positive")
        for p in params:
            if not (p.is_cuda and p.dtype == torch.float32 and p.is_contiguous()):
                raise ValueError("adam: parameters must be contiguous float32 CUDA tensors")
        self.params = list(params)
        self.cfg = cfg
        self.t = 0
        self.m = [torch.zeros(p.shape, dtype=torch.float64, device=p.device) for p in self.params]
        self.v = [torch.zeros(p.shape, dtype=torch.float64, device=p.device) for p in self.params]

    @property
    def steps_taken(self) -> int:
        return self.t

    def step(self, grads: Sequence[torch.Tensor],
             shadows: Optional[Sequence[Optional[torch.Tensor]]] = None) -> None:
        """adam.cpp:38-55: one update from the batch gradients (f32 or f64,
        same shapes as the parameters)."""
        if len(grads) != len(self.params) or any(g.shape != p.shape for g, p in zip(grads, self.params)):
            raise ValueError("adam: gradient shapes do not match the optimizer state")
        self.t += 1
        shadows = shadows if shadows is not None else [None] * len(self.params)
        L = _capi.lib()
        for p, g, m, v, sh in zip(self.params, grads, self.m, self.v, shadows):
            g = g.contiguous()
            if g.dtype not in _GRAD:
                raise ValueError("adam: gradients must be float32 or float64")
            sp, sd = None, -1
            if sh is not None:
                if sh.shape != p.shape or sh.dtype not in _SHADOW or not sh.is_contiguous():
                    raise ValueError("adam: shadow must match the parameter (bfloat16 or float32)")
                sp, sd = sh.data_ptr(), _SHADOW[sh.dtype]
            _capi.check(L.lf_adam_step(p.data_ptr(), g.data_ptr(), _GRAD[g.dtype], m.data_ptr(),
                                       v.data_ptr(), p.numel(), self.cfg.lr, self.cfg.beta1,
                                       self.cfg.beta2, self.cfg.eps, self.t, sp, sd, _stream(p)))
