"""CCE- (negative-sampled fused CE) — B200 drop-in for lseforge::ccem_forward /
ccem_backward / ccem_backward_rows / estimate_flops
(proj/include/lseforge/ccem.hpp:19-49, proj/src/ccem.cpp).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass
from typing import Optional

import torch

from . import _capi
from .accountant import MemAccountant, ScalarKind
from .cce import CceConfig, _charge_scratch, _reset_peak, _stream
from .losses import GradPair, LossOutput, check_device_matrix, grad_dtype, lf_dtype


class Backend(enum.IntEnum):  # backend.hpp:10-16
    kCe = 0
    kCem = 1
    kCce = 2
    kCcem = 3
    kBce = 4


def backend_is_sampled(b: Backend) -> bool:  # backend.hpp:22
    return b in (Backend.kCem, Backend.kCcem)


@dataclass
class FlopEstimate:  # ccem.hpp:43-46
    forward: int = 0
    backward: int = 0


def estimate_flops(n: int, d: int, v: int, ns: int, backend: Backend) -> FlopEstimate:
    """ccem.cpp:207-235 (multiply-accumulate counts), via the C-ABI."""
    f, b = C.c_uint64(), C.c_uint64()
    _capi.check(_capi.lib().lf_estimate_flops(n, d, v, ns, int(backend), C.byref(f), C.byref(b)))
    return FlopEstimate(int(f.value), int(b.value))


def _validate_sampled(X: torch.Tensor, E: torch.Tensor, inds: torch.Tensor, validate: bool):
    """ccem.cpp:16-31."""
    check_device_matrix("hidden states", X)
    check_device_matrix("item embeddings", E)
    if inds.dim() != 2 or inds.dtype != torch.int64 or not inds.is_cuda or not inds.is_contiguous():
        raise ValueError("fused sampled loss: inds must be a contiguous [n, 1+ns] int64 CUDA tensor")
    if inds.shape[0] != X.shape[0]:
        raise ValueError(f"fused sampled loss: {inds.shape[0]} candidate rows for {X.shape[0]} "
                         "embedding rows")
    if X.shape[0] == 0:
        raise ValueError("fused sampled loss: zero rows; the mean loss is undefined")
    if X.shape[1] != E.shape[1]:
        raise ValueError(f"fused sampled loss: embedding width {X.shape[1]} does not match "
                         f"classifier height {E.shape[1]}")
    if X.dtype != E.dtype:
        raise ValueError(f"fused sampled loss: X is {X.dtype} but E is {E.dtype}")
    if inds.shape[1] == 0:
        raise ValueError("NegIndexMatrix: width must be at least 1 (the positive slot)")
    if validate:
        _capi.check(_capi.lib().lf_validate_inds(inds.data_ptr(), inds.shape[0], inds.shape[1],
                                                 E.shape[0], _stream(X)))


def ccem_forward(X: torch.Tensor, E: torch.Tensor, inds: torch.Tensor,
                 cfg: CceConfig = CceConfig(), acct: Optional[MemAccountant] = None,
                 validate: bool = True) -> LossOutput:
    """ccem.cpp:48-105 (paper Alg. 1)."""
    _validate_sampled(X, E, inds, validate)
    if cfg.row_block < 1:
        raise ValueError("CceConfig: row_block must be >= 1")
    n, d = X.shape
    v = E.shape[0]
    w = inds.shape[1]
    if acct is not None:  # ccem.cpp:63-68
        acct.record_ensure("retained/ccem/pos_logits", n)
        acct.record_ensure("retained/ccem/lse", n)
        acct.record_ensure("retained/ccem/inds", n * w, ScalarKind.kIndex)
    base = _reset_peak() if acct is not None else 0
    lse = torch.empty(n, dtype=torch.float64, device=X.device)
    pos = torch.empty(n, dtype=torch.float64, device=X.device)
    loss = torch.empty((), dtype=torch.float64, device=X.device)
    c = cfg.to_c(lf_dtype(X))
    _capi.check(_capi.lib().lf_ccem_forward(X.data_ptr(), E.data_ptr(), inds.data_ptr(), n, d, v,
                                            w, C.byref(c), lse.data_ptr(), pos.data_ptr(),
                                            loss.data_ptr(), _stream(X)))
    _charge_scratch(acct, "scratch/ccem/forward", base)
    return LossOutput(loss, pos, lse)


def ccem_backward_rows(X: torch.Tensor, E: torch.Tensor, inds: torch.Tensor, lse: torch.Tensor,
                       row_upstream: Optional[torch.Tensor], cfg: CceConfig = CceConfig(),
                       acct: Optional[MemAccountant] = None, validate: bool = True,
                       upstream: float = 1.0) -> GradPair:
    """ccem.cpp:107-194 (paper Alg. 2); row_upstream[i] = d objective / d loss_i.
    Filtering never applies here (ccem.hpp:22-26)."""
    _validate_sampled(X, E, inds, validate)
    if cfg.row_block < 1:
        raise ValueError("CceConfig: row_block must be >= 1")
    n, d = X.shape
    v = E.shape[0]
    w = inds.shape[1]
    if lse.numel() != n:  # ccem.cpp:116-119
        raise ValueError(f"ccem_backward: LSE vector has {lse.numel()} entries for {n} rows")
    if row_upstream is not None and row_upstream.numel() != n:  # ccem.cpp:120-124
        raise ValueError(f"ccem_backward: upstream vector has {row_upstream.numel()} entries "
                         f"for {n} rows")
    lse = lse.to(dtype=torch.float64).contiguous()
    if row_upstream is not None:
        row_upstream = row_upstream.to(device=X.device, dtype=torch.float64).contiguous()
    if acct is not None:  # ccem.cpp:132-137
        acct.record_ensure("retained/ccem/lse", n)
        acct.record_ensure("retained/ccem/inds", n * w, ScalarKind.kIndex)
    base = _reset_peak() if acct is not None else 0
    gd = grad_dtype(X)
    dX = torch.empty((n, d), dtype=gd, device=X.device)
    dE = torch.empty((v, d), dtype=gd, device=X.device)
    c = cfg.to_c(lf_dtype(X))
    _capi.check(_capi.lib().lf_ccem_backward(
        X.data_ptr(), E.data_ptr(), inds.data_ptr(), lse.data_ptr(),
        row_upstream.data_ptr() if row_upstream is not None else None, float(upstream), n, d, v,
        w, C.byref(c), dX.data_ptr(), dE.data_ptr(), _stream(X)))
    _charge_scratch(acct, "scratch/ccem/backward", base)
    return GradPair(dX, dE)


def ccem_backward(X: torch.Tensor, E: torch.Tensor, inds: torch.Tensor, lse: torch.Tensor,
                  upstream: float = 1.0, cfg: CceConfig = CceConfig(),
                  acct: Optional[MemAccountant] = None, validate: bool = True) -> GradPair:
    """ccem.cpp:196-205: row_upstream[i] = upstream / n."""
    if X.shape[0] == 0:
        raise ValueError("fused sampled loss: zero rows; the mean loss is undefined")
    return ccem_backward_rows(X, E, inds, lse, None, cfg, acct, validate, upstream=upstream)


def ccem_forward_backward(X: torch.Tensor, E: torch.Tensor, inds: torch.Tensor,
                          upstream: float = 1.0, cfg: CceConfig = CceConfig(),
                          row_upstream: Optional[torch.Tensor] = None,
                          acct: Optional[MemAccountant] = None,
                          validate: bool = True) -> tuple[LossOutput, GradPair]:
    """ccem_forward then ccem_backward[_rows] on the same inputs (the
    trainer's pairing, trainer.cpp:71-77) through lf_ccem_forward_backward:
    one gather pass over the candidates gives lse, pos, dX and the entries'
    logits (bf16 / f32, d in {64, 128, 256}, ordered dE); otherwise the two
    calls run in sequence.  Same outputs and tolerances as the two calls."""
    _validate_sampled(X, E, inds, validate)
    if cfg.row_block < 1:
        raise ValueError("CceConfig: row_block must be >= 1")
    n, d = X.shape
    v = E.shape[0]
    w = inds.shape[1]
    if row_upstream is not None:
        if row_upstream.numel() != n:  # ccem.cpp:120-124
            raise ValueError(f"ccem_backward: upstream vector has {row_upstream.numel()} entries "
                             f"for {n} rows")
        row_upstream = row_upstream.to(device=X.device, dtype=torch.float64).contiguous()
    if acct is not None:  # ccem.cpp:63-68, 132-137
        acct.record_ensure("retained/ccem/pos_logits", n)
        acct.record_ensure("retained/ccem/lse", n)
        acct.record_ensure("retained/ccem/inds", n * w, ScalarKind.kIndex)
    base = _reset_peak() if acct is not None else 0
    lse = torch.empty(n, dtype=torch.float64, device=X.device)
    pos = torch.empty(n, dtype=torch.float64, device=X.device)
    loss = torch.empty((), dtype=torch.float64, device=X.device)
    gd = grad_dtype(X)
    dX = torch.empty((n, d), dtype=gd, device=X.device)
    dE = torch.empty((v, d), dtype=gd, device=X.device)
    c = cfg.to_c(lf_dtype(X))
    _capi.check(_capi.lib().lf_ccem_forward_backward(
        X.data_ptr(), E.data_ptr(), inds.data_ptr(), n, d, v, w,
        row_upstream.data_ptr() if row_upstream is not None else None, float(upstream), C.byref(c),
        lse.data_ptr(), pos.data_ptr(), loss.data_ptr(), dX.data_ptr(), dE.data_ptr(), _stream(X)))
    _charge_scratch(acct, "scratch/ccem/forward_backward", base)
    return LossOutput(loss, pos, lse), GradPair(dX, dE)
